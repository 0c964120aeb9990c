#!/bin/bash
# ncu of the ring-mode warp pack on cfg4 (70B shard, ~37 GiB HBM ring of 6.5 GiB
# slots): (1) every pack launch of two checkpoints, DRAM bytes + time
# (application replay: the counters fit one pass); (2) one launch --set full.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --replay-mode application --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k "regex:(^|:)pack_kernel" --csv --log-file gpurun_out/r2_cfg4_ring_pack_launches.csv \
  python tools/prof_ring.py cfg4 > gpurun_out/r2_cfg4_ring_pack_launches.log 2>&1
timeout 2400 $NCU --set full --replay-mode application --clock-control none --import-source on \
  -k "regex:(^|:)pack_kernel" -s 3 -c 1 -o gpurun_out/r2_cfg4_ring_pack_full -f \
  python tools/prof_ring.py cfg4 > gpurun_out/r2_cfg4_ring_pack_full.log 2>&1
$NCU -i gpurun_out/r2_cfg4_ring_pack_full.ncu-rep --page raw --csv > gpurun_out/r2_cfg4_ring_pack_full_raw.csv 2>&1
