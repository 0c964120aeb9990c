#!/bin/bash
# cfg4 training-interference noise study: repeated default runs vs all-GPU
# checksums vs lowest-priority host workers.
mkdir -p gpurun_out
for v in "" "--ck-host-frac 0" "--worker-nice 19" "" "--ck-host-frac 0" "--worker-nice 19"; do
  echo "== $v" >> gpurun_out/r2_noise.log
  timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline $v 2>&1 | tail -1 >> gpurun_out/r2_noise.log
done
g++ -O3 -pthread tools/host_fnv_probe.cpp -o tools/host_fnv_probe 2>/dev/null && ./tools/host_fnv_probe 64 > gpurun_out/r2_host_fnv.jsonl
