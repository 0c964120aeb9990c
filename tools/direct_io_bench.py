"""Disk flush A/B: page-cache flush (flush_mmap=1, default) vs O_DIRECT flush
(flush_mmap=2) of one rank's state to a disk filesystem. Reports the time to
"persisted" (files + footers + manifest written) and to persisted + sync(2)
(bytes on the device), per mode, alternating modes. Mode 3: O_DIRECT through
io_uring.

  python tools/direct_io_bench.py [--gb 8] [--root /var/tmp] [--reps 2]
"""
import argparse
import json
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_16956_b200 import api  # noqa: E402


def drop_caches() -> bool:
    os.sync()
    try:
        with open("/proc/sys/vm/drop_caches", "w") as f:
            f.write("3\n")
        return True
    except OSError:
        return False


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=8.0)
    ap.add_argument("--root", default="/var/tmp")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--objects", type=int, default=16)
    ap.add_argument("--modes", default="1,2")
    ap.add_argument("--workers", type=int, default=0, help="flush workers (0: engine default)")
    ap.add_argument("--window-mb", type=int, default=0, help="D2H window MiB (0: engine default)")
    ap.add_argument("--restore", action="store_true",
                    help="also time cold restores (caches dropped) with pread and with O_DIRECT reads")
    a = ap.parse_args()
    per = int(a.gb * 1e9 / a.objects) // 4096 * 4096
    objs = [api.StateObject(i + 1, file_id=i % 4, size_bytes=per,
                            payload=torch.randint(0, 255, (per,), dtype=torch.uint8, device="cuda"))
            for i in range(a.objects)]
    st = api.RankState(objects=objs)
    total = per * a.objects
    for rep in range(a.reps):
        for mode in [int(m) for m in a.modes.split(",")]:
            d = os.path.join(a.root, f"dio_bench_{os.getpid()}_{rep}_{mode}")
            cfg = api.EngineConfig(flush_mmap=mode, staging_capacity_bytes=min(total + (64 << 20), 24 << 30),
                                   file_dma=False)
            if a.workers:
                cfg.flush_workers = a.workers
            if a.window_mb:
                cfg.raw_chunk_bytes = a.window_mb << 20
            eng = api.CheckpointEngine(cfg, 0, 0)
            os.sync()
            t0 = time.perf_counter()
            sess = api.CheckpointSession(d, 1, 1, None, n_ranks=1)
            t = eng.issue_checkpoint(sess, st, 1)
            eng.pre_update_barrier(t)
            t.wait_persisted()
            sess.wait_complete(600)
            t1 = time.perf_counter()
            os.sync()
            t2 = time.perf_counter()
            s = t.stats()
            print(json.dumps({"mode": {1: "page-cache", 2: "O_DIRECT", 3: "O_DIRECT+io_uring"}[mode], "rep": rep, "gb": round(total / 1e9, 2),
                              "persisted_gbps": round(total / (t1 - t0) / 1e9, 2),
                              "synced_gbps": round(total / (t2 - t0) / 1e9, 2),
                              "sync_s": round(t2 - t1, 2),
                              "direct_io_frac": round(s["direct_io_bytes"] / total, 3),
                              "workers": cfg.flush_workers, "window_mb": cfg.raw_chunk_bytes >> 20}), flush=True)
            eng.shutdown()
            if a.restore:
                for dio, cold in ((False, True), (True, True), ("uring", True), (None, True), (None, False)):
                    dropped = drop_caches() if cold else False
                    r = api.Restorer(os.path.join(d, "MANIFEST.tlv"), direct_io=dio)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    rs = r.restore_rank(0)
                    torch.cuda.synchronize()
                    dt = time.perf_counter() - t0
                    ok = all(torch.equal(o.payload, so.payload) for o, so in zip(rs.objects, objs))
                    print(json.dumps({"restore": {False: "pread", True: "O_DIRECT", "uring": "O_DIRECT+io_uring",
                                                  None: "auto"}[dio],
                                      "written_by": mode,
                                      "caches_dropped": dropped, "gbps": round(total / dt / 1e9, 2),
                                      "direct_io_frac": round(r.last_stats["direct_io_bytes"] / total, 3),
                                      "bit_exact": ok}), flush=True)
                    del rs, r
            shutil.rmtree(d, ignore_errors=True)
            os.sync()


if __name__ == "__main__":
    main()
