#!/bin/bash
# cfg4 training interference with and without the e2e + restore phase before it.
for e in 0 2; do
  timeout 1500 python bench.py --config cfg4 --steps 2 --warmup 3 --e2e-steps $e --keep 1 --pool-gb 8 --train-steps 5 \
    --ckpt-interval 2 --no-cpu-baseline 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['blocked']; print('e2e_steps', $e, b['slowdown_pct'], b['blocked_ms_per_ckpt'], b['host_checksum_frac'], b['phase_ms']['lazy']['barrier'])"
done
