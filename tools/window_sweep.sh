#!/bin/bash
# D2H window size (raw_chunk_bytes) sweep on the default config, snapshot only.
for w in 64 256 16; do
  for r in 1 2; do
    timeout 600 python bench.py --train-steps 0 --e2e-steps 0 --no-cpu-baseline --window-mb $w 2>/dev/null | tail -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('window_mb', $w, d['value'], d['d2h_gbps'])"
  done
done
