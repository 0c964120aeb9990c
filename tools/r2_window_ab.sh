#!/bin/bash
# cfg4 training interference vs D2H window size: thousands of queued 64 MiB
# window copies per checkpoint vs a few hundred 512 MiB ones (host-side stalls
# of the training thread's CUDA calls: phase fwd_bwd_event_record).
mkdir -p gpurun_out
for v in "--window-mb 64" "--window-mb 512" "--window-mb 64" "--window-mb 512"; do
  echo "== $v" >> gpurun_out/r2_window_ab.log
  timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline $v 2>&1 | tail -1 >> gpurun_out/r2_window_ab.log
done
