#!/bin/bash
# ncu of the HYBRID pack launches on cfg4 (only the last ring-full is packed):
# DRAM bytes + time of every pack launch of two checkpoints (application replay).
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --replay-mode application --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k "regex:(^|:)pack_kernel" --csv --log-file gpurun_out/r2_cfg4_hybrid_pack_launches.csv \
  python tools/prof_ring.py cfg4 hybrid > gpurun_out/r2_cfg4_hybrid_pack_launches.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/r2_cfg4_hybrid_pack_launches.log
