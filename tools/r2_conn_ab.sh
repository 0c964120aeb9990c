#!/bin/bash
# cfg4 training: hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS 8 default vs 32)
mkdir -p gpurun_out
for c in 8 32 8 32; do
  echo "== CUDA_DEVICE_MAX_CONNECTIONS=$c" >> gpurun_out/r2_conn_ab.log
  CUDA_DEVICE_MAX_CONNECTIONS=$c TS_TRACE_COPIES=1 timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    2> gpurun_out/r2_conn_err.tmp | tail -1 >> gpurun_out/r2_conn_ab.log
  grep run_job gpurun_out/r2_conn_err.tmp | head -3 >> gpurun_out/r2_conn_ab.log
done
