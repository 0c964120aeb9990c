"""The C-ABI library: loads, exports every symbol include/ts_b200.h declares, and
its host-only functions (TLV, planner, FNV, metadata, manifest assembly) agree
with the oracle. No compute calls: engine creation must fail loudly without a GPU."""
import os
import random
import re

import numpy as np
import pytest
import torch

from conftest import ROOT


def header_symbols():
    with open(os.path.join(ROOT, "include", "ts_b200.h")) as f:
        src = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)
    return sorted(set(re.findall(r"\b(ts_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol(native):
    syms = header_symbols()
    assert len(syms) > 50
    missing = [s for s in syms if not hasattr(native.lib, s)]
    assert not missing, missing
    assert native.lib.ts_abi_version() == 1


def rand_value(rng, depth=0):
    t = rng.randrange(7 if depth < 3 else 5)
    if t == 0:
        return None
    if t == 1:
        return rng.randrange(-2**63, 2**63)
    if t == 2:
        return rng.choice([0.0, -1.5, 1e300, float(rng.random())])
    if t == 3:
        return "".join(rng.choice(["a", "é", "∑", "😀", "z"]) for _ in range(rng.randrange(6)))
    if t == 4:
        return bytes(rng.randrange(256) for _ in range(rng.randrange(10)))
    if t == 5:
        return [rand_value(rng, depth + 1) for _ in range(rng.randrange(4))]
    return {rand_value(rng, 4) or "k" + str(i) if False else "k%d" % rng.randrange(100):
            rand_value(rng, depth + 1) for i in range(rng.randrange(4))}


def test_tlv_matches_oracle(native, oracle):
    from paper_2601_16956_b200 import api

    rng = random.Random(1)
    for _ in range(300):
        v = rand_value(rng)
        enc = api.tlv_encode(v)
        assert enc == oracle.tlv_encode(v)
        assert api.tlv_decode(enc) == oracle.tlv_decode(enc)


def test_tlv_strict_decoder(native):
    from paper_2601_16956_b200 import api

    good = api.tlv_encode({"a": [1, "x"]})
    for bad in (good[:-1], good + b"\x00", b"\x07", b"\x03\x02\x00\x00\x00\x00\x00\x00\x00\xff\xfe",
                b"\x06\x01" + b"\x00" * 7 + b"\x01" + b"\x00" * 8 + b"\x00"):
        with pytest.raises(api.TlvError):
            api.tlv_decode(bad)


def test_metadata_value_matches_oracle(native, oracle):
    from paper_2601_16956_b200 import api

    for (rid, tp, pp, dp, seed, mb, it) in [(0, 0, 0, 0, 42, 2 << 20, 0), (5, 1, 2, 3, 2**64 - 1, 100, 7),
                                             (3, 1, 0, 1, 99, (1 << 20) + 300_000, 2)]:
        enc = api.Value.metadata(rid, tp, pp, dp, seed, mb, it).encode()
        ref = oracle.tlv_encode(oracle.make_metadata_value(oracle.Rank(rid, tp, pp, dp, seed, mb), it))
        assert enc == ref


def test_fnv_matches_oracle(native, oracle):
    from paper_2601_16956_b200 import api

    data = np.random.default_rng(0).integers(0, 256, 100_000, dtype=np.uint8).tobytes()
    assert api.fnv1a64(data) == oracle.fnv1a64(data)
    assert api.fnv1a64(data[500:], api.fnv1a64(data[:500])) == oracle.fnv1a64(data)


def plan_native(native, objs):
    import ctypes as C

    arr = (native.ObjectDesc * max(1, len(objs)))()
    for i, o in enumerate(objs):
        arr[i].object_id, arr[i].kind, arr[i].file_id, arr[i].size_bytes = o.object_id, o.kind, o.file_id, o.size
    n = len(objs)
    files = (C.c_uint32 * max(1, n))()
    ends = (C.c_uint64 * max(1, n))()
    fixed = (native.FixedAssignment * max(1, n))()
    ffile = (C.c_uint32 * max(1, n))()
    nf, nx, h = C.c_size_t(), C.c_size_t(), C.c_uint64()
    native.call(native.lib.ts_plan_layout, arr, n, 4096, files, ends, C.byref(nf), fixed, ffile,
                C.byref(nx), C.byref(h))
    return ({files[i]: ends[i] for i in range(nf.value)},
            [(ffile[i], fixed[i].object_id, fixed[i].file_offset, fixed[i].length) for i in range(nx.value)],
            h.value)


def test_plan_layout_matches_oracle(native, oracle):
    rng = random.Random(7)
    for trial in range(200):
        n = rng.randrange(0, 40)
        ids = rng.sample(range(1, 10_000), n)
        objs = []
        for oid in ids:
            kind = 1 if rng.random() < 0.2 else 0
            size = rng.choice([1, 4095, 4096, 4097, rng.randrange(1, 1 << 22), 7777]) if kind == 0 else 0
            objs.append(oracle.Obj(oid, kind, 0, 0, rng.choice([0, 1, 2, 9]), size))
        ends, fixed, h = plan_native(native, objs)
        plan = oracle.plan_layout(objs)
        assert ends == {f: p.tensor_region_end for f, p in plan.items()}
        assert fixed == [(f, oid, off, ln) for f, p in plan.items() for oid, off, ln in p.fixed]
        assert h == oracle.plan_hash(plan)


def test_plan_layout_errors(native, oracle):
    with pytest.raises(native.TsError, match="duplicate object id"):
        plan_native(native, [oracle.Obj(1, 0, 0, 0, 1, 5), oracle.Obj(1, 0, 0, 0, 1, 5)])
    with pytest.raises(native.TsError, match="raw buffer without a known size"):
        plan_native(native, [oracle.Obj(1, 0, 0, 0, 1, 0)])


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback(native):
    from paper_2601_16956_b200 import api

    with pytest.raises(api.CudaError):
        api.CheckpointEngine(api.EngineConfig())
    import ctypes as C

    d = (native.PatternDesc * 1)()
    with pytest.raises(api.CudaError):
        native.call(native.lib.ts_pattern_fill, d, 1, 1, 1, None)


def test_session_manifest_matches_oracle(native, oracle, tmp_path):
    """Manifest assembly (register + persisted, manifest-last) byte-equal to the
    reference's MANIFEST.tlv for every golden tree."""
    from paper_2601_16956_b200 import api
    from paper_2601_16956_b200 import synthetic as S
    from conftest import GOLDEN, golden_recipes

    for name in golden_recipes():
        rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
        d = str(tmp_path / name)
        s = api.CheckpointSession(d, rec.ckpt_id, rec.iteration, rec.manifest_echo(), n_ranks=len(rec.ranks))
        for r in reversed(rec.ranks):  # any order: ranks are sorted at commit
            rs = api.RankState(r.rank_id, r.tp_idx, r.pp_idx, r.dp_idx,
                               objects=[api.StateObject(o.object_id, o.kind, o.tier, o.precision, o.file_id, o.size)
                                        for o in r.objects])
            s.register_rank(rs)
        for r in rec.ranks:
            assert not s.complete
            s.rank_persisted(r.rank_id)
        s.wait_complete(10)
        with open(os.path.join(d, "MANIFEST.tlv"), "rb") as f, \
                open(os.path.join(GOLDEN, "trees", name, "MANIFEST.tlv"), "rb") as g:
            assert f.read() == g.read(), name


def test_capi_caller_compiles_against_header(native, tmp_path):
    """include/ts_b200.h is enough to build a C++ caller (tests/capi/capi_checkpoint.cpp)
    that links the library; run on a GPU by tests/test_gpu_capi.py."""
    import subprocess

    from paper_2601_16956_b200 import build as B

    lib = B.build()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "capi_checkpoint")
    subprocess.run(["g++", "-O2", "-std=c++17", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                    "-I", "/usr/local/cuda/include", os.path.join(root, "tests", "capi", "capi_checkpoint.cpp"),
                    "-o", exe, "-L", os.path.dirname(lib), "-lts_b200", "-L", "/usr/local/cuda/lib64",
                    "-lcudart_static", "-ldl", "-lrt", "-lpthread"], check=True)
    assert os.path.getsize(exe) > 0
