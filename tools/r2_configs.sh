#!/bin/bash
# Other BASELINE configs with the round-2 engine, and fresh-file e2e.
mkdir -p gpurun_out
for c in cfg2 cfg3 cfg1; do
  echo "== $c" >> gpurun_out/r2_configs.log
  timeout 1200 python bench.py --config $c --steps 10 --warmup 3 --keep 2 2>&1 | tail -1 >> gpurun_out/r2_configs.log
done
echo "== cfg2 fresh files" >> gpurun_out/r2_configs.log
timeout 900 python bench.py --config cfg2 --steps 3 --warmup 3 --train-steps 0 --fresh-files --no-cpu-baseline 2>&1 | tail -1 >> gpurun_out/r2_configs.log
