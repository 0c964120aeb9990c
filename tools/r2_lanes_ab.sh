# cfg4 training interference: lane-serial checksums (auto cap) vs off, interleaved.
mkdir -p gpurun_out
for a in "--lane-max-mb 0" "--lane-max-mb -1" "--lane-max-mb 0" "--lane-max-mb -1"; do
  timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline $a > gpurun_out/lanes_ab.tmp 2> gpurun_out/lanes_ab.err
  python - "$a" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/lanes_ab.tmp").read().strip().splitlines()[-1])
b = d["blocked"]; e = d["engine"]
print(json.dumps({"args": sys.argv[1], "value": d["value"], "slowdown_pct": b["slowdown_pct"], "blocked_ms": b["blocked_ms_per_ckpt"],
                  "fwd_bwd_gpu_ms": b["fwd_bwd_gpu_ms"], "host_ck": b["host_checksum_frac"], "lane_ck": b.get("lane_checksum_frac"),
                  "lane_ms": e.get("lane_ms"), "lane_ck_snapshot": e.get("lane_checksum_frac"), "pack_frac": d["roofline"]["frac"],
                  "e2e": d["e2e"]["value"], "clocks": b["clocks"]}))
PY
  cat gpurun_out/lanes_ab.tmp >> gpurun_out/lanes_ab_full.jsonl
done | tee gpurun_out/lanes_ab.jsonl
