#!/bin/bash
# Training interference of the lazy snapshot under checksum placement.
# One JSON line each in gpurun_out/interference.jsonl; summary on stdout.
out=gpurun_out/interference.jsonl
: > $out
run() {
  timeout 600 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --train-steps 5 --no-cpu-baseline "$@" \
    2>>gpurun_out/interference.err | tail -1 >> $out
}
for a in "$@"; do run $a; done
python - <<'PY'
import json
for l in open("gpurun_out/interference.jsonl"):
    d = json.loads(l); b = d["blocked"]; c = d["config"]
    print(c["workload"][:5], b.get("fwd_bwd_launch"), c.get("checksum_host_frac"), "interval", b["ckpt_interval"],
          "slowdown %", b["slowdown_pct"], "blocked ms", b["blocked_ms_per_ckpt"], "host frac", b.get("host_checksum_frac"),
          "off", b["step_ms_no_ckpt"], "lazy", b["step_ms_lazy_ckpt"])
PY
