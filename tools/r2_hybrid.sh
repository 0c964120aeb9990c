# HYBRID D2H (head by copy-engine DMA from the state, last ring-full packed): parity + cfg4 A/B vs RING.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_snapshot.py -q -x -m gpu > gpurun_out/hy_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hy_tests.log
tail -2 gpurun_out/hy_tests.log
python -m pytest tests/test_gpu_large.py -q -x -m gpu -k "cfg4 and hybrid" > gpurun_out/hy_large.log 2>&1; echo "rc=$?" >> gpurun_out/hy_large.log
tail -2 gpurun_out/hy_large.log
for a in "--mode ring" "--mode hybrid" "--mode ring" "--mode hybrid" "--mode ring" "--mode hybrid"; do
  timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline $a > gpurun_out/hy.tmp 2> gpurun_out/hy.err; cp gpurun_out/hy.tmp gpurun_out/hy_last.json
  python - "$a" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/hy.tmp").read().strip().splitlines()[-1])
b = d["blocked"]; e = d["e2e"]
print(json.dumps({"args": sys.argv[1], "value": d["value"], "e2e": e["value"], "slowdown_pct": b["slowdown_pct"],
                  "blocked_ms": b["blocked_ms_per_ckpt"], "fwd_bwd_gpu_ms": b["fwd_bwd_gpu_ms"], "host_ck": b["host_checksum_frac"],
                  "roofline": d["roofline"], "d2h_gbps": d["d2h_gbps"], "restore": e["restore_gbps"], "clocks": b["clocks"]}))
PY
  cat gpurun_out/hy.tmp >> gpurun_out/hy_full.jsonl
done | tee gpurun_out/hy_ab.jsonl
