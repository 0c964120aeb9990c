"""Stress of the asynchronous machinery: a lazy training loop (update -> issue
-> barrier -> update ...) over several checkpoints with rotation, random
checksum placement, helper-GPU windows, host/device tiers and random engine
configurations. Every checkpoint must restore bit-exactly to the state it was
issued from (pattern iteration) and pass verify; the barrier contract is what
makes that hold while the state keeps changing."""
import os
import random
import shutil
import tempfile

import pytest

from paper_2601_16956_b200 import api

pytestmark = pytest.mark.gpu


@pytest.fixture
def shm():
    base = "/dev/shm" if os.path.isdir("/dev/shm") else None
    d = tempfile.mkdtemp(dir=base, prefix="ts_stress_")
    yield d
    shutil.rmtree(d, ignore_errors=True)
    api.file_cache_release_all()


@pytest.mark.parametrize("seed", range(16))
def test_lazy_loop_rotation_stress(gpu, shm, seed):
    from test_gpu_fuzz import random_cfg, random_recipe

    rng = random.Random(9000 + seed)
    rec = random_recipe(rng)
    rec.ranks = rec.ranks[:1]
    spec = rec.ranks[0]
    cfg = random_cfg(rng)
    cfg.checksum_host_frac = rng.choice([-1.0, 0.0, 0.5, 1.0])
    if cfg.d2h_mode in ("ring", "hybrid") and rng.random() < 0.5:
        cfg.helper_devices, cfg.helper_share = (0,), rng.choice([0.25, 0.75])
    keep = rng.choice([1, 2])
    spare = os.path.join(shm, "spare")
    eng = api.CheckpointEngine(cfg, spec.rank_id, 0)
    eng.set_spare_dir(spare)
    state = api.materialize_payloads(spec, 0, 1)
    kept, it = [], 1
    for step in range(7):
        while len(kept) >= keep:
            d0, t0 = kept.pop(0)
            t0.wait_persisted()
            api.retire_checkpoint(d0, spare)
        d = os.path.join(shm, f"c{step}")
        sess = api.CheckpointSession(d, step + 1, it, None, 1, writes_manifest=True)
        ticket = eng.issue_checkpoint(sess, state, it)
        kept.append((d, ticket))
        # lazy: the next optimizer update may only run after the barrier, and
        # then rewrites every state byte while the snapshot is still in flight
        eng.pre_update_barrier(ticket, host_block=rng.choice([0, 1, 2]))  # 0: stream wait
        api.mutate_update_step(state, it + 1)
        ticket.wait_persisted()
        sess.wait_complete(60)
        man = os.path.join(d, "MANIFEST.tlv")
        assert api.verify_checkpoint(man).ok
        rs = api.restore_checkpoint(man)[0]
        for o, so in zip(rs.objects, spec.objects):
            o.pattern_space, o.pattern_offset = so.space, so.offset
        rs.seed = spec.seed
        assert api.pattern_mismatches(rs, it) == 0, (seed, step, cfg)
        it += 1
    eng.shutdown()


@pytest.mark.parametrize("seed", range(8))
def test_lazy_loop_multirank_stress(gpu, shm, seed):
    """Same loop with every rank of a random multi-rank state: engines of one
    process sharing each checkpoint's session (the reference's run_training
    shape), manifest committed once all ranks persisted."""
    from test_gpu_fuzz import random_cfg, random_recipe

    rng = random.Random(19000 + seed)
    rec = random_recipe(rng)
    while len(rec.ranks) < 2:
        rec = random_recipe(rng)
    cfg = random_cfg(rng)
    cfg.checksum_host_frac = rng.choice([-1.0, 0.0, 1.0])
    spare = os.path.join(shm, "spare")
    engines = [api.CheckpointEngine(cfg, r.rank_id, 0) for r in rec.ranks]
    for e in engines:
        e.set_spare_dir(spare)
    states = [api.materialize_payloads(r, 0, 1) for r in rec.ranks]
    kept, it = [], 1
    for step in range(5):
        while len(kept) >= 2:
            d0, ts0 = kept.pop(0)
            for t in ts0:
                t.wait_persisted()
            api.retire_checkpoint(d0, spare)
        d = os.path.join(shm, f"c{step}")
        sess = api.CheckpointSession(d, step + 1, it, None, len(rec.ranks), writes_manifest=True)
        tickets = [e.issue_checkpoint(sess, s, it) for e, s in zip(engines, states)]
        kept.append((d, tickets))
        for e, t, s in zip(engines, tickets, states):
            e.pre_update_barrier(t, host_block=rng.choice([0, 1, 2]))
            api.mutate_update_step(s, it + 1)
        for t in tickets:
            t.wait_persisted()
        sess.wait_complete(60)
        man = os.path.join(d, "MANIFEST.tlv")
        assert api.verify_checkpoint(man).ok
        for rs, spec in zip(api.restore_checkpoint(man), rec.ranks):
            for o, so in zip(rs.objects, spec.objects):
                o.pattern_space, o.pattern_offset = so.space, so.offset
            rs.seed = spec.seed
            assert api.pattern_mismatches(rs, it) == 0, (seed, step, cfg)
        it += 1
    for e in engines:
        e.shutdown()
