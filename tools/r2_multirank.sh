#!/bin/bash
# N>1 code paths on a 1-GPU box: bench.py --gpus 2 spawns two ranks itself
# (they share the device: gloo, TS_BENCH_SHARE_GPU semantics), and the
# reference arm runs two reference processes on disjoint core sets.
mkdir -p gpurun_out
timeout 1200 python bench.py --gpus 2 --config cfg2 --steps 3 --warmup 3 --train-steps 2 --no-cpu-baseline \
  > gpurun_out/r2_two_ranks.log 2>&1; echo rc=$? >> gpurun_out/r2_two_ranks.log
timeout 900 python bench.py --impl reference --gpus 2 --config cfg2 --steps 2 --warmup 1 --ref-budget-s 60 \
  > gpurun_out/r2_two_ranks_ref.log 2>&1; echo rc=$? >> gpurun_out/r2_two_ranks_ref.log
