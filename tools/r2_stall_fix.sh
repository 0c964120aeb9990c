mkdir -p gpurun_out
python -m pytest tests/test_gpu_snapshot.py tests/test_gpu_stress.py tests/test_gpu_fuzz.py tests/test_gpu_filedma.py tests/test_gpu_errors.py -q -x -m gpu > gpurun_out/sf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sf_tests.log
tail -2 gpurun_out/sf_tests.log
for k in 1 2; do
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/sf_bench_$k.json 2> gpurun_out/sf_bench_$k.err
python - $k <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/sf_bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
b = d["blocked"]; e = d["e2e"]
print(json.dumps({"value": d["value"], "e2e": e["value"], "pack_frac": d["roofline"]["frac"], "traffic": d["roofline"]["traffic"],
  "restore": e["restore_gbps"], "restore_warm": e["restore_warm_gbps"], "slowdown": b["slowdown_pct"], "blocked": b["blocked_ms_per_ckpt"],
  "ev_rec_max": b["phase_ms_max"]["lazy"]["fwd_bwd_event_record"], "ev_rec": b["fwd_bwd_event_record_ms_per_step"]["lazy"]}))
PY
done
