#!/bin/bash
# D2H mechanism comparison (north_star item 2) on cfg2 / cfg3, plus cfg4 (70B ZeRO-3 shard).
out=gpurun_out/sweep_r1.jsonl
: > $out
for cfg in cfg2 cfg3; do
  for mode in ring direct zerocopy; do
    timeout 400 python bench.py --config $cfg --mode $mode --steps 3 --warmup 2 --e2e-steps 0 --train-steps 0 \
      --no-cpu-baseline 2>gpurun_out/sweep_${cfg}_${mode}.err | tail -1 >> $out
  done
done
timeout 900 python bench.py --config cfg4 --mode ring --steps 2 --warmup 1 --e2e-steps 0 --train-steps 0 \
  --no-cpu-baseline --pool-gb 16 2>gpurun_out/sweep_cfg4.err | tail -1 >> $out
