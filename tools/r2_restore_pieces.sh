# Restore through pinned pieces: parity (restore / O_DIRECT / large / fuzz tests), probe over knobs, default bench.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_restore.py tests/test_gpu_direct_io.py tests/test_gpu_capi.py tests/test_gpu_fuzz.py tests/test_gpu_filedma.py -q -x -m gpu > gpurun_out/rp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rp_tests.log
tail -2 gpurun_out/rp_tests.log
python -m pytest tests/test_gpu_large.py -q -x -m gpu -k "restore" > gpurun_out/rp_large.log 2>&1; echo "rc=$?" >> gpurun_out/rp_large.log
tail -2 gpurun_out/rp_large.log
: > gpurun_out/rp_knobs.log
for cfg in "4 32" "2 32" "4 16" "8 16" "4 64"; do
  set -- $cfg
  echo "== R=$1 P=$2" >> gpurun_out/rp_knobs.log
  TS_RESTORE_READ_MB=$1 TS_RESTORE_PIECES=$2 timeout 600 python tools/restore_probe.py cfg2 2>&1 | grep "^restore" >> gpurun_out/rp_knobs.log
done
cat gpurun_out/rp_knobs.log | cut -c1-200
timeout 1200 python bench.py --steps 6 --warmup 3 > gpurun_out/rp_bench.json 2> gpurun_out/rp_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/rp_bench.json").read().strip().splitlines()[-1])
e = d["e2e"]
print(json.dumps({"value": d["value"], "e2e": e["value"], "restore_gbps": e["restore_gbps"], "restore_warm_gbps": e["restore_warm_gbps"],
                  "restore_bit_exact": e["restore_bit_exact"], "restore_stats": e["restore_stats"], "unpack": e["unpack_roofline"],
                  "slowdown": d["blocked"]["slowdown_pct"]}))
PY
