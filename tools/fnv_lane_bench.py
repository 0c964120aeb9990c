"""Lane-serial vs segment-parallel FNV on the cfg4 rank shard's object sizes
(2,892 device objects, 120.7 GB; here scaled to fit beside nothing else):
wall time of each kernel path through the C-ABI, per-lane rate, and the
SM-time each needs (lanes: ~7 integer ops/byte on a few warps; segments:
~26 ops/byte on every SM). Prints one JSON line per path."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2601_16956_b200 import api  # noqa: E402
from paper_2601_16956_b200 import synthetic as S  # noqa: E402

scale = float(os.environ.get("SCALE", "1.0"))
rec = S.config_recipe("cfg4", 0)
sizes = sorted((o.size for o in rec.ranks[0].objects if o.kind == 0), reverse=True)
sizes = [max(1, int(s * scale)) for s in sizes]
total = sum(sizes)
buf = torch.randint(0, 256, (total + 4096 * len(sizes),), dtype=torch.uint8, device="cuda")
views, off = [], 0
for s in sizes:
    views.append(buf[off:off + s])
    off = (off + s + 4095) // 4096 * 4096
ref = None
for name, lanes in (("segments", False), ("lanes", True)):
    r = api.fnv1a64_device(views[:64], lanes=lanes)  # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = api.fnv1a64_device(views, lanes=lanes)
    dt = time.perf_counter() - t
    if ref is None:
        ref = r
    print(json.dumps({"path": name, "objects": len(sizes), "bytes": total, "max_object": sizes[0],
                      "wall_s": round(dt, 4), "gbps": round(total / dt / 1e9, 2),
                      "largest_lane_mbps": round(sizes[0] / dt / 1e6, 1) if lanes else None,
                      "identical": r == ref}), flush=True)
