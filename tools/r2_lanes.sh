# Lane-serial FNV: parity, kernel rate, and the cfg4 bench A/B (auto lanes vs off, host share auto vs 0).
mkdir -p gpurun_out
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_snapshot.py -q -x -k "lane or fnv" > gpurun_out/lanes_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lanes_tests.log
tail -3 gpurun_out/lanes_tests.log
timeout 600 python tools/fnv_lane_bench.py > gpurun_out/lanes_kernel.jsonl 2> gpurun_out/lanes_kernel.err; cat gpurun_out/lanes_kernel.jsonl
for a in "--lane-max-mb -1" "--lane-max-mb 0" "--lane-max-mb -1 --ck-host-frac 0" "--lane-max-mb 0"; do
  timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline $a > gpurun_out/lanes_bench.tmp 2> gpurun_out/lanes_bench.err
  python - "$a" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/lanes_bench.tmp").read().strip().splitlines()[-1])
b = d["blocked"]; e = d["engine"]
print(json.dumps({"args": sys.argv[1], "value": d["value"], "slowdown_pct": b["slowdown_pct"], "blocked_ms": b["blocked_ms_per_ckpt"],
                  "fwd_bwd_gpu_ms": b["fwd_bwd_gpu_ms"], "host_ck": b["host_checksum_frac"], "lane_ck": b.get("lane_checksum_frac"),
                  "lane_ms": e.get("lane_ms"), "pack_frac": d["roofline"]["frac"], "e2e": d["e2e"]["value"],
                  "clocks": b["clocks"]}))
PY
  cat gpurun_out/lanes_bench.tmp >> gpurun_out/lanes_bench_full.jsonl
done | tee gpurun_out/lanes_bench.jsonl
