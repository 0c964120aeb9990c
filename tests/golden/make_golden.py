"""Generates the golden fixtures from the compiled REFERENCE (oracle/_ref/ts_ref_driver).

    python tests/golden/make_golden.py            # small trees + KATs
    python tests/golden/make_golden.py --digests  # + large-config digests (minutes)

Outputs (all committed):
  kat.json                      known-answer values printed by the reference
  recipes/<name>.recipe         the state descriptions
  trees/<name>/...              complete checkpoint trees written by the reference
                                in canonical mode (lazy, flush_workers=1)
  digests/<name>.json           per-file size + sha256 + footer summary of large
                                configs (trees too big to commit)
Needs /root/reference (this container only); the GPU box only reads the outputs.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import struct
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_2601_16956_b200 import synthetic as S  # noqa: E402

DRIVER = os.path.join(ROOT, "oracle", "_ref", "ts_ref_driver")


def hand_mixed() -> S.Recipe:
    """One hand-built rank covering the edge cases of the format: 1-byte and
    unaligned sizes, equal sizes (id tie-break), several files incl. a sparse
    file id, host-tier raw objects, pattern offsets, tensor descriptors and a
    metadata object larger than one 1 MiB append chunk."""
    r = S.RankSpec(3, 1, 0, 1, 99, (1 << 20) + 300_000)
    sizes = [1, 17, 4095, 4096, 4097, 100_000, 3 * 65536 + 5, 4096, 12_345]
    files = [1, 1, 2, 2, 5, 1, 2, 2, 1]
    tiers = [0, 0, 0, 1, 0, 0, 0, 0, 1]
    oid = 10
    for i, (sz, f, t) in enumerate(zip(sizes, files, tiers)):
        r.objects.append(S.ObjSpec(oid, 0, t, i % 3, f, sz, S.pack_space(1 + (i % 2), i, 0), 7 * i))
        oid += 1
    r.objects.insert(3, S.ObjSpec(oid, 1, 1, 2, 5, meta=("tmeta", "w.0", "bf16", 123, 0, 123)))
    r.objects.append(S.ObjSpec(oid + 1, 1, 1, 2, 0, meta=("meta",)))
    r.objects.append(S.ObjSpec(oid + 2, 1, 1, 2, 0, meta=("tmeta", "b.ü", "fp32", 7, 3, 4)))
    return S.Recipe("hand_mixed", 4, 9, 2, None, [r])


def two_ranks() -> S.Recipe:
    a = S.RankSpec(0, 0, 0, 0, 5, 600)
    a.objects = [S.ObjSpec(1, 0, 0, 0, 1, 5000, S.pack_space(1, 0, 0), 0),
                 S.ObjSpec(2, 0, 0, 1, 2, 7000, S.pack_space(2, 0, 0), 0),
                 S.ObjSpec(3, 1, 1, 2, 0, meta=("meta",))]
    b = S.RankSpec(1, 0, 0, 1, 5, 600)
    b.objects = [S.ObjSpec(4, 0, 0, 1, 2, 7001, S.pack_space(2, 0, 0), 7000),
                 S.ObjSpec(5, 1, 1, 2, 0, meta=("meta",))]
    return S.Recipe("two_ranks", 2, 3, None, None, [a, b])


def structured_only() -> S.Recipe:
    r = S.RankSpec(0, 0, 0, 0, 1, 100)
    r.objects = [S.ObjSpec(1, 1, 1, 2, 0, meta=("meta",)),
                 S.ObjSpec(2, 1, 1, 2, 3, meta=("tmeta", "x", "fp16", 1, 0, 1))]
    return S.Recipe("structured_only", 1, 1, None, None, [r])


def small_recipes():
    return [
        S.layout_recipe("tiny_layout", 65536, 4, 64, 2, 2, 2, True, 7, 4096, ckpt_id=1, iteration=1),
        S.layout_recipe("odd_layout", 100003, 3, 0, 1, 1, 3, True, 42, 1000, ckpt_id=3, iteration=6,
                        pattern_iteration=5),
        S.layout_recipe("nozero_dp2", 50001, 2, 0, 1, 1, 2, False, 5, 300, ckpt_id=1, iteration=2),
        hand_mixed(),
        two_ranks(),
        structured_only(),
        S.zero3_recipe("zero3_tiny", S.llama_tensors(64, 160, 2, vocab=100), 4, seed=11,
                       metadata_bytes=1000, iteration=2),
    ]


def run_driver(recipe_path: str, out_dir: str, workers: int = 1):
    r = subprocess.run([DRIVER, "write", recipe_path, out_dir, "--workers", str(workers)],
                       capture_output=True, text=True, check=True)
    return json.loads(r.stdout)


def footer_summary(path: str):
    with open(path, "rb") as f:
        f.seek(-8, 2)
        blob_len = struct.unpack("<Q", f.read(8))[0]
        f.seek(-8 - blob_len, 2)
        blob = f.read(blob_len)
    n = struct.unpack("<Q", blob[:8])[0]
    ents = []
    for i in range(n):
        e = blob[8 + 41 * i: 8 + 41 * (i + 1)]
        oid = struct.unpack("<Q", e[:8])[0]
        foff, ln, base, ck = struct.unpack("<QQQQ", e[9:41])
        ents.append([oid, e[8], foff, ln, base, "%016x" % ck])
    return ents


def sha256_file(path: str) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as f:
        while True:
            b = f.read(64 << 20)
            if not b:
                break
            h.update(b)
    return h.hexdigest()


def tree_digest(root: str, with_manifest: bool = True) -> dict:
    out = {}
    for dp, _, fs in os.walk(root):
        for fn in sorted(fs):
            p = os.path.join(dp, fn)
            rel = os.path.relpath(p, root)
            if fn == "MANIFEST.tlv" and not with_manifest:
                continue
            d = {"size": os.path.getsize(p), "sha256": sha256_file(p)}
            if fn.endswith(".bin"):
                d["footer"] = footer_summary(p)
            out[rel] = d
    return dict(sorted(out.items()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--digests", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, stdout=subprocess.DEVNULL)
    kat = subprocess.run([DRIVER, "kat"], capture_output=True, text=True, check=True).stdout
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        f.write(kat)
    os.makedirs(os.path.join(HERE, "recipes"), exist_ok=True)
    for rec in small_recipes():
        if args.only and rec.name != args.only:
            continue
        rp = os.path.join(HERE, "recipes", rec.name + ".recipe")
        with open(rp, "w") as f:
            f.write(rec.to_text())
        dst = os.path.join(HERE, "trees", rec.name)
        shutil.rmtree(dst, ignore_errors=True)
        run_driver(rp, dst)
        print("tree", rec.name, sum(os.path.getsize(os.path.join(d, x)) for d, _, fs in os.walk(dst) for x in fs))
    if not args.digests:
        return
    os.makedirs(os.path.join(HERE, "digests"), exist_ok=True)
    big = [("cfg1", S.config_recipe("cfg1"), None, True),
           ("cfg1b", S.config_recipe("cfg1b"), None, True),
           ("cfg2_rank0", S.config_recipe("cfg2", 0), [0], False),
           ("cfg3_rank0", S.config_recipe("cfg3", 0), [0], False)]
    # cfg2 ranks 1-7 (ZeRO-1 optimizer shards only, 10.1 GB each; the params
    # are written by dp 0, model.cpp:124)
    big += [(f"cfg2_rank{r}", S.config_recipe("cfg2", r), [r], False) for r in range(1, 8)]
    for name, rec, ranks, with_manifest in big:
        if args.only and name != args.only:
            continue
        rp = os.path.join(HERE, "recipes", name + ".recipe")
        with open(rp, "w") as f:
            f.write(rec.to_text(ranks=ranks))
        with tempfile.TemporaryDirectory(dir=os.environ.get("GOLDEN_TMP", "/root")) as td:
            t = run_driver(rp, td, workers=1)
            d = {"recipe": name, "timing_ref": t, "files": tree_digest(td, with_manifest)}
        with open(os.path.join(HERE, "digests", name + ".json"), "w") as f:
            json.dump(d, f, indent=1)
        print("digest", name, t)


if __name__ == "__main__":
    main()
