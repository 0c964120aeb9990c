"""Issue latency on the training thread for a config's object list (default cfg4:
3,616 objects), raw sizes shrunk so the probe takes seconds: engine-side
issue_block_ns vs the whole Python call, with rotation (spare files) like
bench.py's training phase. TS_TRACE=1 prints the engine's per-phase split.

    python tools/issue_latency.py [--config cfg4] [--iters 20] [--max-obj 65536]
"""
import argparse
import json
import os
import shutil
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--max-obj", type=int, default=64 << 10)
    ap.add_argument("--values", action="store_true", help="structured objects pre-built as Values")
    args = ap.parse_args()
    import torch

    from paper_2601_16956_b200 import api
    from paper_2601_16956_b200 import synthetic as S

    rec = S.config_recipe(args.config, 0)
    spec = rec.ranks[0]
    for o in spec.objects:
        if o.kind == 0:
            o.size = min(o.size, args.max_obj)
    st = api.materialize_payloads(spec, 0, 0)
    if args.values:
        for o in st.objects:
            if not o.is_raw() and not isinstance(o.structured, api.Value):
                o.structured = api.Value.from_py(o.structured)
    tdir = "/dev/shm/ts_issue_probe"
    shutil.rmtree(tdir, ignore_errors=True)
    os.makedirs(tdir)
    spare = os.path.join(tdir, ".spare")
    cfg = api.EngineConfig(staging_capacity_bytes=256 << 20, raw_chunk_bytes=16 << 20,
                           device_staging_bytes=1 << 30, flush_workers=8)
    eng = api.CheckpointEngine(cfg, 0, 0)
    eng.set_spare_dir(spare)
    comp = torch.cuda.current_stream()
    eng_ms, py_ms, desc_ms = [], [], []
    prev = []
    for it in range(1, args.iters + 1):
        while prev:
            d0, t0, s0 = prev.pop(0)
            t0.wait_persisted()
            s0.wait_complete(60)  # (the manifest is committed after persist)
            api.retire_checkpoint(d0, spare)
        d = os.path.join(tdir, f"ckpt_{it:06d}")
        sess = api.CheckpointSession(d, it, it, None, 1, writes_manifest=True)
        keep = []
        ta = time.perf_counter()
        api._desc_array(st, keep)
        desc_ms.append(1e3 * (time.perf_counter() - ta))
        torch.cuda.synchronize()
        tb = time.perf_counter()
        t = eng.issue_checkpoint(sess, st, it, producer_stream=comp)
        py_ms.append(1e3 * (time.perf_counter() - tb))
        t.wait_snapshot()
        eng_ms.append(t.stats()["issue_block_ns"] / 1e6)
        prev.append((d, t, sess))
    for d0, t0, s0 in prev:
        t0.wait_persisted()
        s0.wait_complete(60)
    eng.shutdown()
    shutil.rmtree(tdir, ignore_errors=True)
    k = args.iters // 2
    print(json.dumps({"config": args.config, "objects": len(spec.objects), "values_prebuilt": args.values,
                      "engine_issue_ms_median": round(statistics.median(eng_ms[k:]), 3),
                      "python_call_ms_median": round(statistics.median(py_ms[k:]), 3),
                      "desc_array_ms_median": round(statistics.median(desc_ms[k:]), 3),
                      "engine_issue_ms": [round(x, 3) for x in eng_ms]}))


if __name__ == "__main__":
    main()
