#!/bin/bash
# cfg4 training interference: host checksum budget (slack vs slack + D2H time), nice 19.
mkdir -p gpurun_out
for v in "A" "B" "A" "B" "A" "B"; do
  echo "== $v" >> gpurun_out/r2_hostck.log
  if [ $v = B ]; then export TS_HOST_CK_D2H=1; else unset TS_HOST_CK_D2H; fi
  timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 >> gpurun_out/r2_hostck.log
done
