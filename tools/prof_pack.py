"""One lazy checkpoint of a bounded sample of a config (for ncu captures).

    python tools/prof_pack.py [cfg2|cfg3] [n_raw] [mode]
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_16956_b200 import api
from paper_2601_16956_b200 import synthetic as S

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n_raw = int(sys.argv[2]) if len(sys.argv) > 2 else 8
mode = sys.argv[3] if len(sys.argv) > 3 else "ring"
rec = S.config_recipe(cfg, 0)
spec = rec.ranks[0]
raws = [o for o in spec.objects if o.kind == 0][:n_raw]
if cfg == "cfg3":
    for o in raws:
        o.align = 2 if o.precision == 0 else 4
spec.objects = raws + [o for o in spec.objects if o.kind == 1 and o.meta[0] == "meta"]
st = api.materialize_payloads(spec, 0, 1)
need = spec.raw_bytes
ec = api.EngineConfig(d2h_mode=mode, staging_capacity_bytes=(need + (256 << 20)) // (2 << 20) * (2 << 20),
                      raw_chunk_bytes=64 << 20, device_staging_bytes=need + (64 << 20), write_files=False,
                      flush_workers=16)
eng = api.CheckpointEngine(ec, 0, 0)
for it in (2, 3):
    api.mutate_update_step(st, it)
    sess = api.CheckpointSession("", it, it, None, 1, writes_manifest=False)
    t = eng.issue_checkpoint(sess, st, it)
    t.wait_persisted()
    s = t.stats()
    print({k: s[k] for k in ("image_bytes", "pack_ms", "d2h_ms", "t_captured_ns", "t_snapshot_ns", "t_persisted_ns",
                             "kernel_launches")})
eng.shutdown()
