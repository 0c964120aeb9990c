#!/bin/bash
# cfg4 training: deferred host hashing (default) vs hashing as windows land.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_filedma.py tests/test_gpu_snapshot.py tests/test_gpu_stress.py -x -q > gpurun_out/t17.log 2>&1; echo rc=$? >> gpurun_out/t17.log
for v in D N D N D N; do
  echo "== $v" >> gpurun_out/r2_defer_ab.log
  if [ $v = N ]; then export TS_HOST_CK_NODEFER=1; else unset TS_HOST_CK_NODEFER; fi
  timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 >> gpurun_out/r2_defer_ab.log
done
