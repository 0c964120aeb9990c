#!/bin/bash
# Pack kernel A/B: warp gather kernel vs TMA bulk (cp.async.bulk) for large fragments.
for cfg in cfg2 cfg3; do
  for k in warp bulk warp bulk; do
    timeout 600 python bench.py --config $cfg --train-steps 0 --e2e-steps 0 --no-cpu-baseline --pack-kernel $k 2>/dev/null |
      tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', '$k', r['achieved'], r['frac'], r['launch_ms'], d['gpu_launches'])"
  done
done
