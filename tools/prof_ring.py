"""One rank of a config checkpointed twice through the production RING path
(no device shadow: a multi-slot HBM ring sized like bench.py's, warp pack),
snapshot only — for ncu counters of the ring-mode pack launches:

    ncu --replay-mode application --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        -k regex:'(^|:)pack_kernel' --csv python tools/prof_ring.py cfg4
"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_16956_b200 import api
from paper_2601_16956_b200 import synthetic as S

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
mode = sys.argv[2] if len(sys.argv) > 2 else "ring"  # "hybrid": only the last ring-full is packed
spec = S.config_recipe(cfg, 0).ranks[0]
st = api.materialize_payloads(spec, 0, 1)
free, _ = torch.cuda.mem_get_info(0)
ring = max(8 << 30, free - (26 << 30))
ec = api.EngineConfig(d2h_mode=mode, staging_capacity_bytes=4 << 30, raw_chunk_bytes=64 << 20, device_staging_bytes=ring,
                      write_files=False, flush_workers=16)
eng = api.CheckpointEngine(ec, 0, 0)
for it in (2, 3):
    api.mutate_update_step(st, it)
    sess = api.CheckpointSession("", it, it, None, 1, writes_manifest=False)
    t = eng.issue_checkpoint(sess, st, it)
    t.wait_persisted()
    s = t.stats()
    print(json.dumps({"config": cfg, "mode": mode, "packed_bytes": s["packed_bytes"], "ring_bytes": ring, "image_bytes": s["image_bytes"], "raw_bytes": spec.raw_bytes,
                      "pack_ms": s["pack_ms"], "kernel_launches": s["kernel_launches"]}), flush=True)
eng.shutdown()
