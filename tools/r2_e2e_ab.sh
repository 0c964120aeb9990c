# e2e (issue -> files + footers + MANIFEST on /dev/shm) RING vs HYBRID, interleaved, no training phase.
mkdir -p gpurun_out
for a in "--mode ring" "--mode hybrid" "--mode ring" "--mode hybrid" "--mode ring" "--mode hybrid"; do
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --train-steps 0 --e2e-steps 4 $a > gpurun_out/e2e.tmp 2> gpurun_out/e2e.err
  python - "$a" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/e2e.tmp").read().strip().splitlines()[-1])
e = d["e2e"]
print(json.dumps({"args": sys.argv[1], "value": d["value"], "d2h_gbps": d["d2h_gbps"], "e2e": e["value"],
                  "persist_ms_last": e["persist_ms_last"], "snapshot_ms_last": e["snapshot_ms_last"],
                  "restore": e["restore_gbps"], "restore_warm": e["restore_warm_gbps"]}))
PY
done | tee gpurun_out/e2e_ab.jsonl
