#!/bin/bash
# Round-2 isolated kernel captures (no concurrent DMA): unpack_kernel and the
# FNV passes over cfg2 rank 0's shards, and the warp pack for reference.
mkdir -p gpurun_out
lscpu > gpurun_out/r2_lscpu.txt 2>&1
timeout 300 python tools/prof_kernels.py cfg2 all 3 > gpurun_out/r2_kernels_plain.jsonl 2>&1
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active
for spec in "unpack:unpack_kernel:1" "fnv:regex:fnv_pass_:3" "pack:regex:(^|:)pack_kernel:1"; do
  what=${spec%%:*}; rest=${spec#*:}; k=${rest%:*}; c=${rest##*:}
  timeout 900 $NCU --set full --clock-control none --import-source on -k $k -c $c \
    -o gpurun_out/r2_isolated_$what -f python tools/prof_kernels.py cfg2 $what 1 > gpurun_out/r2_ncu_$what.log 2>&1
  $NCU -i gpurun_out/r2_isolated_$what.ncu-rep --page raw --csv --metrics $M > gpurun_out/r2_isolated_${what}_raw.csv 2>&1
done
