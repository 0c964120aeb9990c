"""Synthetic sharded state: the reference's layout generator and the configs of
BASELINE.json, as recipes (host descriptors only; payload bytes are produced on
the GPU by the pattern kernel).

Reference: model.cpp:17-193 (generate_layout, ZeRO-1 sharding, pattern spaces),
model.cpp:206-231 (metadata object). The hand-built ZeRO-3 configs follow the
same conventions: every raw object is a window of a pattern space, shards of
one tensor share the space and differ by offset.

Recipe text format (shared with oracle/ref_driver.cpp):
    checkpoint <ckpt_id> <iteration>
    pattern_iteration <it>
    layout <n_params> <layers> <hidden> <tp> <pp> <dp> <zero1> <seed> <metadata_bytes>
  or hand-built ranks:
    rank <rank_id> <tp_idx> <pp_idx> <dp_idx> <seed> <metadata_bytes>
    raw <oid> <file_id> <precision> <tier> <size> <space> <offset>
    meta <oid> <file_id>
    tmeta <oid> <file_id> <name> <dtype> <numel> <shard_off> <shard_len>
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

ROLE_PARAM, ROLE_OPT, ROLE_META = 1, 2, 3  # model.cpp:13-15
ROLE_EXP_AVG, ROLE_EXP_AVG_SQ = 4, 5       # extra roles of the hand-built ZeRO-3 states
FILE_METADATA, FILE_PARAMS, FILE_OPTIMIZER = 0, 1, 2  # model.hpp:28-30
FP16, FP32, OPAQUE = 0, 1, 2
DEVICE, HOST, PERSISTENT = 0, 1, 2


def pack_space(role: int, layer: int, tp_idx: int) -> int:
    """model.cpp:17-19."""
    return (role << 56) | (layer << 16) | tp_idx


def share_of(total: int, parts: int, idx: int) -> int:
    """model.cpp:22-26 (remainder to index 0)."""
    return total // parts + (total % parts if idx == 0 else 0)


def share_offset(total: int, parts: int, idx: int) -> int:
    """model.cpp:28-32."""
    return 0 if idx == 0 else total % parts + (total // parts) * idx


@dataclass
class ObjSpec:
    object_id: int
    kind: int          # 0 raw, 1 structured
    tier: int
    precision: int
    file_id: int
    size: int = 0
    space: int = 0
    offset: int = 0
    meta: Optional[Tuple] = None  # ("meta",) | ("tmeta", name, dtype, numel, off, len)
    align: int = 256   # device allocation alignment used by the harness (not part of the format)


@dataclass
class RankSpec:
    rank_id: int
    tp_idx: int = 0
    pp_idx: int = 0
    dp_idx: int = 0
    seed: int = 0
    metadata_bytes: int = 0
    objects: List[ObjSpec] = field(default_factory=list)

    @property
    def raw_bytes(self) -> int:
        return sum(o.size for o in self.objects if o.kind == 0)


@dataclass
class Recipe:
    name: str = "custom"
    ckpt_id: int = 1
    iteration: int = 1
    pattern_iteration: Optional[int] = None
    layout: Optional[Tuple[int, ...]] = None
    ranks: List[RankSpec] = field(default_factory=list)

    @property
    def pit(self) -> int:
        return self.iteration if self.pattern_iteration is None else self.pattern_iteration

    def manifest_echo(self):
        """engine.cpp:35-66."""
        if self.layout is None:
            return None
        n, layers, _h, tp, pp, dp, z, seed, meta = self.layout
        return dict(tp=tp, pp=pp, dp=dp, zero1=1 if z else 0, seed=seed, n_params=n, layers=layers,
                    metadata_bytes=meta)

    def to_text(self, ranks: Optional[List[int]] = None) -> str:
        out = [f"checkpoint {self.ckpt_id} {self.iteration}"]
        if self.pattern_iteration is not None:
            out.append(f"pattern_iteration {self.pattern_iteration}")
        if self.layout is not None and ranks is None:
            out.append("layout " + " ".join(str(int(x)) for x in self.layout))
            return "\n".join(out) + "\n"
        for r in self.ranks:
            if ranks is not None and r.rank_id not in ranks:
                continue
            out.append(f"rank {r.rank_id} {r.tp_idx} {r.pp_idx} {r.dp_idx} {r.seed} {r.metadata_bytes}")
            for o in r.objects:
                if o.kind == 0:
                    out.append(f"raw {o.object_id} {o.file_id} {o.precision} {o.tier} {o.size} {o.space} {o.offset}")
                elif o.meta[0] == "meta":
                    out.append(f"meta {o.object_id} {o.file_id}")
                else:
                    _, name, dtype, numel, off, ln = o.meta
                    out.append(f"tmeta {o.object_id} {o.file_id} {name} {dtype} {numel} {off} {ln}")
        return "\n".join(out) + "\n"


def generate_layout(n_params: int, layers: int, hidden: int, tp: int, pp: int, dp: int, zero1: bool,
                    seed: int, metadata_bytes: int = 2 << 20) -> List[RankSpec]:
    """model.cpp:92-193: 2 B/param params + 12 B/param optimizer state, layers over
    PP, bytes over TP, optimizer over DP under ZeRO-1, params written by dp 0 only,
    one structured metadata object per rank, global object ids."""
    if tp < 1 or pp < 1 or dp < 1:
        raise ValueError("layout: tp, pp, dp must be >= 1")
    if layers < pp:
        raise ValueError("layout: insufficient layers for pipeline stages")
    ptot, otot = 2 * n_params, 12 * n_params
    ranks, nid, rid = [], 1, 0
    for d in range(dp):
        for s in range(pp):
            for t in range(tp):
                r = RankSpec(rid, t, s, d, seed, metadata_bytes)
                rid += 1
                first, nl = share_offset(layers, pp, s), share_of(layers, pp, s)
                for l in range(first, first + nl):
                    pslice = share_of(share_of(ptot, layers, l), tp, t)
                    oslice = share_of(share_of(otot, layers, l), tp, t)
                    if pslice == 0 or oslice == 0:
                        raise ValueError("layout: zero share")
                    if d == 0:
                        r.objects.append(ObjSpec(nid, 0, DEVICE, FP16, FILE_PARAMS, pslice,
                                                 pack_space(ROLE_PARAM, l, t), 0))
                        nid += 1
                    if zero1 or d == 0:
                        shard = share_of(oslice, dp, d) if zero1 else oslice
                        off = share_offset(oslice, dp, d) if zero1 else 0
                        r.objects.append(ObjSpec(nid, 0, DEVICE, FP32, FILE_OPTIMIZER, shard,
                                                 pack_space(ROLE_OPT, l, t), off))
                        nid += 1
                r.objects.append(ObjSpec(nid, 1, HOST, OPAQUE, FILE_METADATA, 0,
                                         pack_space(ROLE_META, r.rank_id, 0), 0, ("meta",)))
                nid += 1
                ranks.append(r)
    return ranks


def layout_recipe(name, n_params, layers, hidden, tp, pp, dp, zero1, seed, metadata_bytes,
                  ckpt_id=1, iteration=1, pattern_iteration=None) -> Recipe:
    rec = Recipe(name, ckpt_id, iteration, pattern_iteration,
                 (n_params, layers, hidden, tp, pp, dp, int(bool(zero1)), seed, metadata_bytes))
    rec.ranks = generate_layout(n_params, layers, hidden, tp, pp, dp, zero1, seed, metadata_bytes)
    return rec


# ---------------------------------------------------------------------------
# Transformer tensor lists for the hand-built configs.


def gpt2_small_tensors():
    """GPT-2 small (124M): 148 tensors (BASELINE.json configs[0])."""
    d, v, ctx = 768, 50257, 1024
    ts = [("wte", (v, d)), ("wpe", (ctx, d))]
    for i in range(12):
        p = f"h.{i}."
        ts += [(p + "ln_1.weight", (d,)), (p + "ln_1.bias", (d,)),
               (p + "attn.c_attn.weight", (d, 3 * d)), (p + "attn.c_attn.bias", (3 * d,)),
               (p + "attn.c_proj.weight", (d, d)), (p + "attn.c_proj.bias", (d,)),
               (p + "ln_2.weight", (d,)), (p + "ln_2.bias", (d,)),
               (p + "mlp.c_fc.weight", (d, 4 * d)), (p + "mlp.c_fc.bias", (4 * d,)),
               (p + "mlp.c_proj.weight", (4 * d, d)), (p + "mlp.c_proj.bias", (d,))]
    ts += [("ln_f.weight", (d,)), ("ln_f.bias", (d,))]
    return ts


def llama_tensors(hidden, inter, layers, vocab=32000, kv_hidden=None):
    """Llama-2 parameter list: per layer q,k,v,o, gate, up, down, 2 norms; plus
    embed_tokens, norm, lm_head (13B: 363 tensors, 70B: 723)."""
    kv = kv_hidden or hidden
    ts = [("model.embed_tokens.weight", (vocab, hidden))]
    for i in range(layers):
        p = f"model.layers.{i}."
        ts += [(p + "self_attn.q_proj.weight", (hidden, hidden)), (p + "self_attn.k_proj.weight", (kv, hidden)),
               (p + "self_attn.v_proj.weight", (kv, hidden)), (p + "self_attn.o_proj.weight", (hidden, hidden)),
               (p + "mlp.gate_proj.weight", (inter, hidden)), (p + "mlp.up_proj.weight", (inter, hidden)),
               (p + "mlp.down_proj.weight", (hidden, inter)),
               (p + "input_layernorm.weight", (hidden,)), (p + "post_attention_layernorm.weight", (hidden,))]
    ts += [("model.norm.weight", (hidden,)), ("lm_head.weight", (vocab, hidden))]
    return ts


def numel(shape) -> int:
    n = 1
    for s in shape:
        n *= s
    return n


def gpt2_adam_recipe(seed=42, metadata_bytes=2 << 20, iteration=1, pattern_iteration=0) -> Recipe:
    """cfg1 (ii): one rank, 148 GPT-2 tensors x {fp32 param, exp_avg, exp_avg_sq}
    = 444 raw objects (params in file 1, moments in file 2) + rank metadata."""
    rec = Recipe("gpt2_adam", 1, iteration, pattern_iteration)
    r = RankSpec(0, 0, 0, 0, seed, metadata_bytes)
    nid = 1
    for ti, (name, shape) in enumerate(gpt2_small_tensors()):
        b = 4 * numel(shape)
        r.objects.append(ObjSpec(nid, 0, DEVICE, FP32, FILE_PARAMS, b, pack_space(ROLE_PARAM, ti, 0), 0))
        r.objects.append(ObjSpec(nid + 1, 0, DEVICE, FP32, FILE_OPTIMIZER, b, pack_space(ROLE_EXP_AVG, ti, 0), 0))
        r.objects.append(ObjSpec(nid + 2, 0, DEVICE, FP32, FILE_OPTIMIZER, b, pack_space(ROLE_EXP_AVG_SQ, ti, 0), 0))
        nid += 3
    r.objects.append(ObjSpec(nid, 1, HOST, OPAQUE, FILE_METADATA, meta=("meta",),
                             space=pack_space(ROLE_META, 0, 0)))
    rec.ranks = [r]
    return rec


def zero3_recipe(name, tensors, world: int, ranks: Optional[List[int]] = None, seed=42,
                 metadata_bytes=2 << 20, iteration=1, pattern_iteration=None, tensor_meta=True) -> Recipe:
    """ZeRO-3 state (configs 3 and 4): every tensor flat-partitioned over `world`
    ranks (remainder to rank 0, model.cpp:22-32 convention). Per rank and tensor:
    bf16 param shard (file 1), fp32 master / exp_avg / exp_avg_sq shards (file 2),
    optionally one small structured tensor descriptor (file 0), plus the rank
    metadata object. Object ids are global (exclusive scan over ranks, as
    model.cpp:108 numbers them). fp32 shards are carved out of flat buffers at
    4-byte granularity (alignment recorded for the harness)."""
    rec = Recipe(name, 1, iteration, pattern_iteration)
    per_rank = len(tensors) * (5 if tensor_meta else 4) + 1
    for r in range(world):
        if ranks is not None and r not in ranks:
            continue
        rs = RankSpec(r, 0, 0, r, seed, metadata_bytes)
        nid = 1 + r * per_rank
        for ti, (tname, shape) in enumerate(tensors):
            n = numel(shape)
            cnt, off = share_of(n, world, r), share_offset(n, world, r)
            rs.objects.append(ObjSpec(nid, 0, DEVICE, FP16, FILE_PARAMS, 2 * cnt,
                                      pack_space(ROLE_PARAM, ti, 0), 2 * off, align=2))
            rs.objects.append(ObjSpec(nid + 1, 0, DEVICE, FP32, FILE_OPTIMIZER, 4 * cnt,
                                      pack_space(ROLE_OPT, ti, 0), 4 * off, align=4))
            rs.objects.append(ObjSpec(nid + 2, 0, DEVICE, FP32, FILE_OPTIMIZER, 4 * cnt,
                                      pack_space(ROLE_EXP_AVG, ti, 0), 4 * off, align=4))
            rs.objects.append(ObjSpec(nid + 3, 0, DEVICE, FP32, FILE_OPTIMIZER, 4 * cnt,
                                      pack_space(ROLE_EXP_AVG_SQ, ti, 0), 4 * off, align=4))
            nid += 4
            if tensor_meta:
                rs.objects.append(ObjSpec(nid, 1, HOST, OPAQUE, FILE_METADATA,
                                          meta=("tmeta", tname, "bf16", n, off, cnt)))
                nid += 1
        rs.objects.append(ObjSpec(nid, 1, HOST, OPAQUE, FILE_METADATA, meta=("meta",),
                                  space=pack_space(ROLE_META, r, 0)))
        rec.ranks.append(rs)
    return rec


LLAMA2_7B = dict(n_params=6_738_415_616, layers=32, hidden=4096)


def config_recipe(cfg: str, rank: int = 0, **kw) -> Recipe:
    """Named configs of BASELINE.json (one rank's state)."""
    if cfg == "cfg1":  # GPT-2 small generate_layout, SURVEY §8c pinned outputs
        return layout_recipe("cfg1", 124_439_808, 12, 768, 1, 1, 1, False, 42, 2 << 20,
                             iteration=1, pattern_iteration=0)
    if cfg == "cfg1b":
        return gpt2_adam_recipe()
    if cfg == "cfg2":  # Llama-2 7B ZeRO-1 over 8 ranks; one rank's shard
        full = layout_recipe("cfg2", LLAMA2_7B["n_params"], 32, 4096, 1, 1, 8, True, 42, 2 << 20)
        rec = Recipe("cfg2", 1, 1, None, None, [r for r in full.ranks if r.rank_id == rank])
        rec.full_layout = full.layout  # type: ignore[attr-defined]
        return rec
    if cfg == "cfg3":
        return zero3_recipe("cfg3", llama_tensors(5120, 13824, 40), 8, ranks=[rank], **kw)
    if cfg == "cfg4":
        return zero3_recipe("cfg4", llama_tensors(8192, 28672, 80, kv_hidden=1024), 8, ranks=[rank],
                            tensor_meta=kw.pop("tensor_meta", True), **kw)
    raise ValueError(cfg)


def load_recipe(path: str) -> Recipe:
    rec = Recipe(name=path)
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].split()
            if not line:
                continue
            kw, a = line[0], line[1:]
            if kw == "checkpoint":
                rec.ckpt_id, rec.iteration = int(a[0]), int(a[1])
            elif kw == "pattern_iteration":
                rec.pattern_iteration = int(a[0])
            elif kw == "layout":
                v = [int(x) for x in a]
                rec.layout = tuple(v)
                rec.ranks = generate_layout(v[0], v[1], v[2], v[3], v[4], v[5], bool(v[6]), v[7], v[8])
            elif kw == "rank":
                rid, tp, pp, dp, seed, meta = (int(x) for x in a)
                rec.ranks.append(RankSpec(rid, tp, pp, dp, seed, meta))
            elif kw == "raw":
                oid, fid, prec, tr, size, space, off = (int(x) for x in a)
                rec.ranks[-1].objects.append(ObjSpec(oid, 0, tr, prec, fid, size, space, off))
            elif kw == "meta":
                rec.ranks[-1].objects.append(ObjSpec(int(a[0]), 1, HOST, OPAQUE, int(a[1]), meta=("meta",)))
            elif kw == "tmeta":
                rec.ranks[-1].objects.append(ObjSpec(int(a[0]), 1, HOST, OPAQUE, int(a[1]),
                                                     meta=("tmeta", a[2], a[3], int(a[4]), int(a[5]), int(a[6]))))
            else:
                raise ValueError(f"unknown recipe keyword {kw}")
    return rec
