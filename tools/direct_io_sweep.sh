#!/bin/bash
# O_DIRECT flush sweep on the box's disk (/var/tmp): workers x window size.
mkdir -p gpurun_out
for w in 0 16 32; do for mb in 16 64; do
  timeout 300 python tools/direct_io_bench.py --gb 8 --reps 1 --modes 2 --workers $w --window-mb $mb >> gpurun_out/dio_sweep.jsonl 2>>gpurun_out/dio_sweep.err
done; done
timeout 300 python tools/direct_io_bench.py --gb 8 --reps 1 --modes 1 --workers 16 >> gpurun_out/dio_sweep.jsonl 2>>gpurun_out/dio_sweep.err
