#!/bin/bash
# Host cost of the copier's D2H enqueues: windows landing in page-locked file
# pages (file_dma) vs the cudaHostAlloc'd pool (--no-train-files).
mkdir -p gpurun_out
for v in "" "--no-train-files"; do
  echo "== $v" >> gpurun_out/r2_copytrace.log
  TS_TRACE_COPIES=1 timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline $v \
    > gpurun_out/r2_copytrace_out.tmp 2> gpurun_out/r2_copytrace_err.tmp
  grep "run_job" gpurun_out/r2_copytrace_err.tmp >> gpurun_out/r2_copytrace.log
  tail -1 gpurun_out/r2_copytrace_out.tmp >> gpurun_out/r2_copytrace.log
done
