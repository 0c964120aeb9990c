"""Digests of full-size configs too large for the compiled reference to write in
this container's RAM (cfg4: 120.7 GB per rank), computed by the PINNED oracle
restatement (oracle/tso.py `rank_digest`: plan, header, footer tables with
per-object FNV-1a of the pattern bytes, append-region sha256, manifest sha256).

    python tests/golden/make_oracle_digests.py [--only cfg4_rank0]

Before writing anything, the restatement is re-pinned against every digest the
compiled reference wrote (tests/golden/digests/cfg*_rank*.json, cfg1, cfg1b):
the footers (hence every object's checksum) and file sizes must agree.
Outputs: tests/golden/digests/<name>.json + recipes/<name>.recipe (committed).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import tso  # noqa: E402

from paper_2601_16956_b200 import synthetic as S  # noqa: E402


def oracle_digest(rec: "tso.Recipe", with_manifest: bool) -> dict:
    files, infos = {}, []
    for r in rec.ranks:
        f, info = tso.rank_digest(r, rec.pit)
        files.update(f)
        infos.append(info)
    if with_manifest:
        m = tso.tlv_encode(tso.manifest_value(rec.ckpt_id, rec.iteration, rec.manifest_echo(), infos))
        files["MANIFEST.tlv"] = {"size": len(m), "sha256": hashlib.sha256(m).hexdigest()}
    return dict(sorted(files.items()))


def pin_against_reference():
    """Every reference-written digest must be reproduced by the restatement."""
    d = os.path.join(HERE, "digests")
    for fn in sorted(os.listdir(d)):
        with open(os.path.join(d, fn)) as f:
            ref = json.load(f)
        if ref.get("source", "reference") != "reference":
            continue
        rec = tso.load_recipe(os.path.join(HERE, "recipes", ref["recipe"] + ".recipe"))
        got = oracle_digest(rec, "MANIFEST.tlv" in ref["files"])
        for rel, g in ref["files"].items():
            assert got[rel]["size"] == g["size"], (fn, rel)
            if "footer" in g:
                assert got[rel]["footer"] == g["footer"], (fn, rel)
            if rel == "MANIFEST.tlv":
                assert got[rel]["sha256"] == g["sha256"], (fn, rel)
        print("pinned", fn)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--no-pin", action="store_true")
    args = ap.parse_args()
    if not args.no_pin:
        pin_against_reference()
    for name, rec, with_manifest in [("cfg4_rank0", S.config_recipe("cfg4", 0), True)]:
        if args.only and name != args.only:
            continue
        rp = os.path.join(HERE, "recipes", name + ".recipe")
        with open(rp, "w") as f:
            f.write(rec.to_text())
        t0 = time.time()
        dig = oracle_digest(tso.load_recipe(rp), with_manifest)
        out = {"recipe": name, "source": "oracle restatement (oracle/tso.py rank_digest), pinned against "
                                         "every reference-written digest by this script",
               "oracle_s": round(time.time() - t0, 1), "files": dig}
        with open(os.path.join(HERE, "digests", name + ".json"), "w") as f:
            json.dump(out, f, indent=1)
        print("digest", name, out["oracle_s"], "s")


if __name__ == "__main__":
    main()
