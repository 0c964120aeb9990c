#!/bin/bash
# cfg2 e2e to the box's ext4 disk: page-cache flush vs O_DIRECT flush.
mkdir -p gpurun_out /var/tmp/ts_disk
timeout 900 python bench.py --ckpt-root /var/tmp/ts_disk --keep 1 --no-train-files --steps 3 > gpurun_out/disk_pc.json 2> gpurun_out/disk_pc.err
rm -rf /var/tmp/ts_disk/*; sync
timeout 900 python bench.py --ckpt-root /var/tmp/ts_disk --keep 1 --no-train-files --steps 3 --flush-direct > gpurun_out/disk_dio.json 2> gpurun_out/disk_dio.err
rm -rf /var/tmp/ts_disk
