"""Isolated kernel runs for ncu (no copy-engine traffic in flight, so DRAM
counters belong to the kernel): the scatter-unpack kernel and the FNV-1a
kernel chain over a config's rank shard layout (cfg2 rank 0: 65 objects,
23.6 GB, the raw shards at their ZeRO alignments).

    python tools/prof_kernels.py [cfg2] [unpack|fnv|pack|all] [reps]

Under ncu:  ncu --set full -k regex:"unpack_kernel|fnv_pass_c" -c 2 ...
Outside ncu it prints CUDA-event times and the achieved algorithmic GB/s.
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_16956_b200 import api
from paper_2601_16956_b200 import synthetic as S

N = api.N


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    what = sys.argv[2] if len(sys.argv) > 2 else "all"
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    spec = S.config_recipe(cfg, 0).ranks[0]
    spec.objects = [o for o in spec.objects if o.kind == 0]
    st = api.materialize_payloads(spec, 0, 1)
    objs = [o for o in st.objects if o.is_raw()]
    n = len(objs)
    sizes = (C.c_uint64 * n)(*[o.size_bytes for o in objs])
    offs, pos = [], 0
    for o in objs:  # image: every object 16-B aligned (the engine's layout rule)
        pos = (pos + 4095) // 4096 * 4096
        offs.append(pos)
        pos += o.size_bytes
    img_len = pos
    doffs = (C.c_uint64 * n)(*offs)
    ptrs = (C.c_void_p * n)(*[o.payload.data_ptr() for o in objs])
    img = torch.empty(img_len, dtype=torch.uint8, device="cuda")
    raw = sum(o.size_bytes for o in objs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {"config": cfg, "objects": n, "raw_bytes": raw}

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts)

    sh = torch.cuda.current_stream().cuda_stream
    if what in ("pack", "unpack", "all"):
        N.call(N.lib.ts_pack, ptrs, sizes, doffs, n, img.data_ptr(), img_len, 0, 0, C.c_void_p(sh))
    if what in ("pack", "all"):
        ms = timed(lambda: N.call(N.lib.ts_pack, ptrs, sizes, doffs, n, img.data_ptr(), img_len, 0, 0,
                                  C.c_void_p(sh)))
        out["pack_ms"] = round(ms, 3)
        out["pack_gbps"] = round((raw + img_len) / ms / 1e6, 1)
    if what in ("unpack", "all"):
        ms = timed(lambda: N.call(N.lib.ts_unpack, img.data_ptr(), doffs, ptrs, sizes, n, 0, 0, C.c_void_p(sh)))
        out["unpack_ms"] = round(ms, 3)
        out["unpack_gbps"] = round(2 * raw / ms / 1e6, 1)  # reads the image pieces, writes the shards
    if what in ("fnv", "all"):
        views = [o.payload for o in objs]
        ms = timed(lambda: api.fnv1a64_device(views))
        out["fnv_ms"] = round(ms, 3)
        out["fnv_gbps"] = round(raw / ms / 1e6, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
