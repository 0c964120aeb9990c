"""Helpers for the GPU parity tests: drive the B200 engine through the Python
mirror of the reference API exactly as the reference's run loop does."""
import os

from paper_2601_16956_b200 import api
from paper_2601_16956_b200 import synthetic as S


def checkpoint_recipe(rec: S.Recipe, out_dir: str, cfg: api.EngineConfig, device: int = 0,
                      states=None, keep_engines=False):
    """Materialize every rank of `rec` on the GPU at its pattern iteration and take
    one lazy checkpoint of all ranks into `out_dir` (ranks as engines of one
    process sharing one session, like the reference's run_training)."""
    session = api.CheckpointSession(out_dir, rec.ckpt_id, rec.iteration, rec.manifest_echo(),
                                    n_ranks=len(rec.ranks))
    if states is None:
        states = [api.materialize_payloads(r, device, rec.pit) for r in rec.ranks]
    engines = [api.CheckpointEngine(cfg, r.rank_id, device) for r in rec.ranks]
    tickets = [e.issue_checkpoint(session, s, rec.iteration) for e, s in zip(engines, states)]
    for t in tickets:
        t.wait_persisted()
    session.wait_complete(120)
    stats = [t.stats() for t in tickets]
    if not keep_engines:
        for e in engines:
            e.shutdown()
        engines = None
    return session, states, stats, engines


def tree_bytes(root):
    out = {}
    for dp, _, fs in os.walk(root):
        for fn in fs:
            p = os.path.join(dp, fn)
            with open(p, "rb") as f:
                out[os.path.relpath(p, root)] = f.read()
    return out
