"""Checkpoint one cfg2 rank-0 state to /dev/shm and time restores (TS_TRACE=1 for phases)."""
import os, sys, time, shutil
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_16956_b200 import api, synthetic as S
rec = S.config_recipe(sys.argv[1] if len(sys.argv) > 1 else "cfg2", 0)
spec = rec.ranks[0]
st = api.materialize_payloads(spec, 0, 1)
need = spec.raw_bytes
eng = api.CheckpointEngine(api.EngineConfig(staging_capacity_bytes=(need + (256 << 20)) // (2 << 20) * (2 << 20),
                                            raw_chunk_bytes=64 << 20, device_staging_bytes=need + (64 << 20),
                                            flush_workers=16), 0, 0)
d = "/dev/shm/rp"
shutil.rmtree(d, ignore_errors=True)
sess = api.CheckpointSession(d, 1, 1, None, 1)
t = eng.issue_checkpoint(sess, st, 1)
t.wait_persisted(); sess.wait_complete(600); eng.shutdown()
for i in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    r = api.Restorer(d + "/MANIFEST.tlv"); r.restore_rank(0, 0, into=st); torch.cuda.synchronize()
    print("restore", i, round(time.time() - t0, 3), "s", {k: round(v, 3) if isinstance(v, float) else v for k, v in r.last_stats.items()}, flush=True)
shutil.rmtree(d, ignore_errors=True)
