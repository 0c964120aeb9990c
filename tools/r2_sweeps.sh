#!/bin/bash
# Round-2 measurement sweeps (one gpurun call): cfg4 interference vs HBM ring
# size, strategy comparison (blocked ms / slowdown) on cfg2 and cfg4, host
# memory bandwidth, disk flush/restore with io_uring.
mkdir -p gpurun_out
g++ -O2 -pthread tools/membw_probe.cpp -o tools/membw_probe 2>/dev/null && ./tools/membw_probe 8 > gpurun_out/r2_membw.jsonl
for r in 8 16 0; do
  echo "== ring_gb=$r" >> gpurun_out/r2_ring_sweep.log
  timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --ring-gb $r 2>&1 | tail -1 >> gpurun_out/r2_ring_sweep.log
done
for c in cfg2 cfg4; do for s in lazy lazy_old two_phase sync; do
  echo "== $c $s" >> gpurun_out/r2_strategies.log
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --strategy $s 2>&1 | tail -1 >> gpurun_out/r2_strategies.log
done; done
timeout 900 python tools/direct_io_bench.py --gb 8 --reps 2 --modes 2,3 --workers 16 --window-mb 64 --restore > gpurun_out/r2_uring_disk.jsonl 2> gpurun_out/r2_uring_disk.err
