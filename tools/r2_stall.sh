#!/bin/bash
# Where does the training thread's CUDA-call stall come from? Full bench
# (snapshot + e2e + restore + training) vs training right after the snapshot
# phase (--e2e-steps 0), back to back.
mkdir -p gpurun_out
for v in "" "--e2e-steps 0" ""; do
  echo "== $v" >> gpurun_out/r2_stall.log
  timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $v 2>&1 | tail -1 >> gpurun_out/r2_stall.log
done
