#!/bin/bash
# Page-cache restore path (cfg2 rank 0 on /dev/shm, fresh files: not page-locked):
# ring depth x pread piece.
mkdir -p gpurun_out
for k in 4 8; do for mb in 16 64; do
  echo "== windows=$k read_mb=$mb" >> gpurun_out/r2_restore_knobs.log
  TS_RESTORE_WINDOWS=$k TS_RESTORE_READ_MB=$mb timeout 600 python tools/restore_probe.py cfg2 2>&1 | grep "^restore" >> gpurun_out/r2_restore_knobs.log
done; done
