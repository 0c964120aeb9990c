"""Direct D2H into page-locked checkpoint files (file_dma, csrc/filereg.hpp).

With checkpoint rotation, a finalized file's fixed region is page-locked in the
background; when the file is recycled for a later checkpoint of the same
layout, the copy engines write the D2H windows straight into its page-cache
pages. Every case must stay byte-identical to the reference's trees, and a
registration must never be used for a file that changed behind our back."""
import os
import shutil
import tempfile

import pytest

from conftest import GOLDEN, read_tree
from gpu_helpers import checkpoint_recipe
from paper_2601_16956_b200 import api
from paper_2601_16956_b200 import synthetic as S

pytestmark = pytest.mark.gpu


@pytest.fixture
def shm():
    if not os.path.isdir("/dev/shm"):
        pytest.skip("needs tmpfs /dev/shm")
    d = tempfile.mkdtemp(dir="/dev/shm", prefix="ts_filedma_")
    yield d
    shutil.rmtree(d, ignore_errors=True)
    api.file_cache_release_all()


def cfg_for(mode, **kw):
    extra = {}
    if mode == "ring-bulk":
        # (a full device shadow: the bulk path is used for one-pack images only)
        mode, extra = "ring", dict(pack_kernel="bulk", bulk_min_bytes=32768, device_staging_bytes=256 << 20)
    base = dict(d2h_mode=mode, raw_chunk_bytes=64 << 10, staging_capacity_bytes=1 << 20,
                device_staging_bytes=256 << 10, flush_workers=3)
    base.update(extra)
    base.update(kw)
    return api.EngineConfig(**base)


def fixed_bytes(rec, tso):
    """Σ fixed-region bytes [4096, tensor_region_end) over every rank file
    (plan from the oracle's restatement: test-side checker only)."""
    tot = 0
    for r in rec.ranks:
        objs = [tso.Obj(o.object_id, o.kind, o.tier, o.precision, o.file_id, o.size) for o in r.objects]
        tot += sum(fp.tensor_region_end - 4096 for fp in tso.plan_layout(objs).values())
    return tot


def rotate(rec, shm, cfg, rounds=3, tamper=None):
    """`rounds` checkpoints of the same state, each new one recycling the files
    of the one before (retired into a spare directory); engines are recreated
    per checkpoint, so their shutdown waits for the background page locking."""
    spare = os.path.join(shm, "spare")
    stats = []
    prev = None
    for k in range(rounds):
        if prev:
            api.retire_checkpoint(prev, spare)
            if tamper:
                tamper(spare)
        out = os.path.join(shm, f"c{k}")
        session = api.CheckpointSession(out, rec.ckpt_id, rec.iteration, rec.manifest_echo(),
                                        n_ranks=len(rec.ranks))
        states = [api.materialize_payloads(r, 0, rec.pit) for r in rec.ranks]
        engines = [api.CheckpointEngine(cfg, r.rank_id, 0) for r in rec.ranks]
        for e in engines:
            e.set_spare_dir(spare)
        tickets = [e.issue_checkpoint(session, s, rec.iteration) for e, s in zip(engines, states)]
        for t in tickets:
            t.wait_persisted()
        session.wait_complete(120)
        stats.append([t.stats() for t in tickets])
        for e in engines:
            e.shutdown()
        assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", rec_name(rec))), f"checkpoint {k}"
        prev = out
    return stats


def rec_name(rec):
    return rec._golden_name


def load(name):
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    rec._golden_name = name
    return rec


@pytest.mark.parametrize("mode", ["ring", "direct", "zerocopy", "ring-bulk"])
@pytest.mark.parametrize("name", ["hand_mixed", "odd_layout", "zero3_tiny", "two_ranks"])
def test_recycled_files_take_direct_dma(gpu, shm, oracle, name, mode):
    rec = load(name)
    stats = rotate(rec, shm, cfg_for(mode))
    dma0 = sum(s["file_dma_bytes"] for s in stats[0])
    dma1 = sum(s["file_dma_bytes"] for s in stats[1])
    dma2 = sum(s["file_dma_bytes"] for s in stats[2])
    assert dma0 == 0  # fresh files: pool + flush
    assert dma1 == dma2 == fixed_bytes(rec, oracle) > 0  # every fixed-region byte straight into the file


@pytest.mark.parametrize("mode", ["ring", "direct"])
def test_direct_dma_host_checksums(gpu, shm, oracle, mode):
    """checksum_on_gpu=0: host FNV workers hash the pieces in the file pages."""
    rec = load("hand_mixed")
    stats = rotate(rec, shm, cfg_for(mode, checksum_on_gpu=False))
    assert sum(s["file_dma_bytes"] for s in stats[1]) == fixed_bytes(rec, oracle)


def test_file_dma_off_uses_pool(gpu, shm):
    rec = load("odd_layout")
    stats = rotate(rec, shm, cfg_for("ring", file_dma=False))
    assert all(s["file_dma_bytes"] == 0 for ss in stats for s in ss)
    assert api.file_cache_bytes() == 0


def test_tampered_file_is_not_trusted(gpu, shm):
    """A recycled file truncated behind the registry's back (size/mtime stamp
    changed) is not written through its stale locked pages."""
    rec = load("odd_layout")

    def tamper(spare):
        for f in sorted(os.listdir(spare)):
            p = os.path.join(spare, f)
            sz = os.path.getsize(p)
            if sz > 8192:
                os.truncate(p, 4096)
                os.truncate(p, sz)
                with open(p, "r+b") as fh:
                    fh.seek(5000)
                    fh.write(b"x")

    stats = rotate(rec, shm, cfg_for("ring"), rounds=2, tamper=tamper)
    assert sum(s["file_dma_bytes"] for s in stats[1]) == 0


def test_layout_change_drops_registration(gpu, shm):
    """Files recycled for a different layout (other tensor_region_end) fall back
    to the pool path, and the bytes stay identical."""
    a, b = load("tiny_layout"), load("two_ranks")
    for r, o in zip(b.ranks, a.ranks):
        o.rank_id = r.rank_id
    a.ranks = a.ranks[:len(b.ranks)]
    spare = os.path.join(shm, "spare")
    cfg = cfg_for("ring")
    old = os.path.join(shm, "old")
    sess = api.CheckpointSession(old, a.ckpt_id, a.iteration, a.manifest_echo(), n_ranks=len(a.ranks))
    engines = [api.CheckpointEngine(cfg, r.rank_id, 0) for r in a.ranks]
    for e in engines:
        e.set_spare_dir(spare)
    states = [api.materialize_payloads(r, 0, a.pit) for r in a.ranks]
    for t in [e.issue_checkpoint(sess, s, a.iteration) for e, s in zip(engines, states)]:
        t.wait_persisted()
    sess.wait_complete(60)
    for e in engines:
        e.shutdown()
    assert api.file_cache_bytes() > 0
    api.retire_checkpoint(old, spare)
    new = os.path.join(shm, "new")
    sess = api.CheckpointSession(new, b.ckpt_id, b.iteration, b.manifest_echo(), n_ranks=len(b.ranks))
    engines = [api.CheckpointEngine(cfg, r.rank_id, 0) for r in b.ranks]
    for e in engines:
        e.set_spare_dir(spare)
    states = [api.materialize_payloads(r, 0, b.pit) for r in b.ranks]
    tickets = [e.issue_checkpoint(sess, s, b.iteration) for e, s in zip(engines, states)]
    for t in tickets:
        t.wait_persisted()
    sess.wait_complete(60)
    assert all(t.stats()["file_dma_bytes"] == 0 for t in tickets)
    for e in engines:
        e.shutdown()
    assert read_tree(new) == read_tree(os.path.join(GOLDEN, "trees", "two_ranks"))


def test_deleted_files_are_unlocked(gpu, shm):
    rec = load("hand_mixed")
    rotate(rec, shm, cfg_for("ring"), rounds=2)
    assert api.file_cache_bytes() > 0
    for d in os.listdir(shm):
        shutil.rmtree(os.path.join(shm, d))
    # the next issue sweeps registrations of unlinked files
    out = os.path.join(shm, "after")
    checkpoint_recipe(rec, out, cfg_for("ring"))
    assert api.file_cache_bytes() == 0


@pytest.mark.parametrize("use_cache", [True, False])
def test_restore_from_locked_files(gpu, shm, use_cache):
    """Restore of a checkpoint whose files this process page-locked: the copy
    engines read them straight from the page cache (or pread when disabled);
    bit-exact either way."""
    rec = load("hand_mixed")
    rotate(rec, shm, cfg_for("ring"), rounds=2)
    man = os.path.join(shm, "c1", "MANIFEST.tlv")
    r = api.Restorer(man, use_file_cache=use_cache)
    direct = 0
    for i, spec in enumerate(rec.ranks):
        rs = r.restore_rank(i, 0)
        direct += r.last_stats["direct_bytes"]
        for o, so in zip(rs.objects, spec.objects):
            o.pattern_space, o.pattern_offset = so.space, so.offset
        rs.seed = spec.seed
        assert api.pattern_mismatches(rs, rec.pit) == 0
    assert (direct > 0) == use_cache


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_rotation_parity(gpu, shm, oracle, seed):
    """Random states and engine configs, checkpointed with rotation: each round
    recycles the previous round's files (page-locked when the layout matches,
    dropped when it does not) and must equal the oracle's canonical tree."""
    import random

    from test_gpu_fuzz import random_cfg, random_recipe

    rng = random.Random(5000 + seed)
    recs = [random_recipe(rng)]
    # rounds 2-3: the same state again (same layout: direct DMA), then another
    # random state with the same rank ids (other layout: pool path)
    recs.append(recs[0])
    other = random_recipe(rng)
    other.ranks = other.ranks[:len(recs[0].ranks)]
    for r, o in zip(recs[0].ranks, other.ranks):
        o.rank_id = r.rank_id
    recs.append(other)
    cfg = random_cfg(rng)
    spare = os.path.join(shm, "spare")
    prev = None
    for k, rec in enumerate(recs):
        if prev:
            api.retire_checkpoint(prev, spare)
        out = os.path.join(shm, f"c{k}")
        session = api.CheckpointSession(out, rec.ckpt_id, rec.iteration, rec.manifest_echo(), n_ranks=len(rec.ranks))
        states = [api.materialize_payloads(r, 0, rec.pit) for r in rec.ranks]
        engines = [api.CheckpointEngine(cfg, r.rank_id, 0) for r in rec.ranks]
        for e in engines:
            e.set_spare_dir(spare)
        tickets = [e.issue_checkpoint(session, s, rec.iteration) for e, s in zip(engines, states)]
        for t in tickets:
            t.wait_persisted()
        session.wait_complete(120)
        for e in engines:
            e.shutdown()
        ref = os.path.join(shm, f"ref{k}")
        orec = oracle.load_recipe_text(rec.to_text())
        oracle.write_checkpoint(orec, ref, ser_chunk=min(cfg.serialized_chunk_bytes, cfg.staging_capacity_bytes))
        assert read_tree(out) == read_tree(ref), (seed, k, cfg)
        shutil.rmtree(ref)
        prev = out


@pytest.mark.parametrize("name", ["hand_mixed", "odd_layout", "two_ranks"])
def test_provisioned_spares_first_checkpoint_direct(gpu, shm, oracle, name):
    """provision_spares: the very first checkpoint of a rotation recycles
    pre-created, page-locked spare files (direct D2H), byte-identical."""
    rec = load(name)
    spare = os.path.join(shm, "spare")
    states = [api.materialize_payloads(r, 0, rec.pit) for r in rec.ranks]
    engines = [api.CheckpointEngine(cfg_for("ring"), r.rank_id, 0) for r in rec.ranks]
    locked = 0
    for e, s in zip(engines, states):
        e.set_spare_dir(spare)
        locked += e.provision_spares(spare, s, copies=2)
    assert locked >= fixed_bytes(rec, oracle)
    out = os.path.join(shm, "c0")
    session = api.CheckpointSession(out, rec.ckpt_id, rec.iteration, rec.manifest_echo(), n_ranks=len(rec.ranks))
    tickets = [e.issue_checkpoint(session, s, rec.iteration) for e, s in zip(engines, states)]
    for t in tickets:
        t.wait_persisted()
    session.wait_complete(60)
    assert sum(t.stats()["file_dma_bytes"] for t in tickets) == fixed_bytes(rec, oracle)
    for e in engines:
        e.shutdown()
    assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))


def test_spares_accumulate_up_to_limit(gpu, shm):
    """retire_checkpoint keeps several spares per file name (suffixes), up to a cap."""
    rec = load("odd_layout")
    rotate(rec, shm, cfg_for("ring"), rounds=1)
    spare = os.path.join(shm, "spare")
    for k in range(6):  # retire 6 copies of the same checkpoint
        d = os.path.join(shm, f"x{k}")
        shutil.copytree(os.path.join(shm, "c0"), d)
        api.retire_checkpoint(d, spare)
    names = os.listdir(spare)
    per = {}
    for n in names:
        per.setdefault(n.split(".bin")[0], []).append(n)
    assert per and all(1 <= len(v) <= 4 for v in per.values())


@pytest.mark.parametrize("defer", ["0", "1"])
def test_auto_host_hashing_in_a_training_loop(gpu, defer, monkeypatch):
    """Auto checksum placement in a lazy loop with slack between checkpoints
    and rotation on tmpfs (every window lands in a page-locked file): the host
    workers take a share — as windows land, or after the D2H with
    TS_HOST_CK_DEFER=1. Every checkpoint's footers verify and the last one
    restores bit-exactly."""
    if not os.path.isdir("/dev/shm"):
        pytest.skip("needs tmpfs for page-locked files")
    monkeypatch.setenv("TS_HOST_CK_DEFER", defer)
    tmp = tempfile.mkdtemp(dir="/dev/shm")
    try:
        _auto_host_hashing_loop(tmp)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
        api.file_cache_release_all()


def _auto_host_hashing_loop(tmp):
    import time

    spec = S.RankSpec(0, seed=11, metadata_bytes=256)
    for i in range(24):
        spec.objects.append(S.ObjSpec(i + 1, 0, 0, 1, i % 3, (5 << 20) + 4096 * i + 13, S.pack_space(2, i, 0), 0))
    spec.objects.append(S.ObjSpec(100, 1, 1, 2, 0, meta=("meta",)))
    st = api.materialize_payloads(spec, 0, 1)
    spare = os.path.join(tmp, ".spare")
    eng = api.CheckpointEngine(api.EngineConfig(raw_chunk_bytes=4 << 20, staging_capacity_bytes=64 << 20,
                                                device_staging_bytes=32 << 20, flush_workers=4), 0, 0)
    eng.set_spare_dir(spare)
    prev, host_bytes = None, []
    for it in range(1, 9):
        api.mutate_update_step(st, it)
        d = os.path.join(tmp, f"c{it}")
        sess = api.CheckpointSession(d, it, it, None, 1)
        t = eng.issue_checkpoint(sess, st, it)
        eng.pre_update_barrier(t, host_block=1)
        t.wait_persisted()
        sess.wait_complete(60)
        host_bytes.append(t.stats()["host_checksum_bytes"])
        assert api.verify_checkpoint(os.path.join(d, "MANIFEST.tlv")).ok
        if prev:
            api.retire_checkpoint(prev, spare)
        prev = d
        time.sleep(0.4)  # slack: the training step between checkpoints
    eng.shutdown()
    assert max(host_bytes[3:]) > 0, host_bytes  # the auto policy handed the host a share
    rs = api.restore_checkpoint(os.path.join(prev, "MANIFEST.tlv"))[0]
    for o, so in zip(rs.objects, spec.objects):
        o.pattern_space, o.pattern_offset = so.space, so.offset
    rs.seed = spec.seed
    assert api.pattern_mismatches(api.RankState(0, seed=spec.seed, objects=[o for o in rs.objects if o.is_raw()]),
                                  8) == 0
