"""O_DIRECT flushes (EngineConfig.flush_mmap = 2, SURVEY §8 f2 "kernel-bypass
flush"): each staged window's 4 KiB-aligned body goes from the pinned pool to
the file with O_DIRECT (no page-cache copy), the ragged head/tail with
pwrite(2). The files must equal the oracle's canonical checkpoint byte for
byte and restore bit-exactly; on a filesystem that refuses O_DIRECT (tmpfs)
the writer stays buffered and the result is the same."""
import os
import random
import shutil

import pytest

from conftest import read_tree
from gpu_helpers import checkpoint_recipe
from paper_2601_16956_b200 import api
from test_gpu_fuzz import random_recipe

pytestmark = pytest.mark.gpu


def direct_dir(tmp_path):
    """A scratch directory on a filesystem that accepts O_DIRECT, or None."""
    root = os.environ.get("GRAFT_REPO_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for d in (str(tmp_path), "/var/tmp", os.path.join(root, "gpurun_out")):
        try:
            os.makedirs(d, exist_ok=True)
            probe = os.path.join(d, ".odirect_probe_%d" % os.getpid())
            fd = os.open(probe, os.O_WRONLY | os.O_CREAT | os.O_DIRECT, 0o644)
            os.close(fd)
            os.unlink(probe)
            return os.path.join(d, "odirect_%d" % os.getpid())
        except OSError:
            continue
    return None


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("mode", ["ring", "direct"])
@pytest.mark.parametrize("flush", [2, 3])  # O_DIRECT pwrite / O_DIRECT through io_uring
def test_direct_io_parity(gpu, oracle, tmp_path, seed, mode, flush):
    base = direct_dir(tmp_path) or str(tmp_path / "buffered")
    try:
        rng = random.Random(7000 + seed)
        rec = random_recipe(rng)
        w = rng.choice([4096, 65536, 1 << 20])
        cfg = api.EngineConfig(d2h_mode=mode, raw_chunk_bytes=w, staging_capacity_bytes=8 << 20,
                               device_staging_bytes=1 << 24, flush_workers=rng.choice([1, 3]), flush_mmap=flush)
        ours = os.path.join(base, "ours")
        checkpoint_recipe(rec, ours, cfg)
        ref = str(tmp_path / "oracle")
        orec = oracle.load_recipe_text(rec.to_text())
        oracle.write_checkpoint(orec, ref, ser_chunk=min(cfg.serialized_chunk_bytes, cfg.staging_capacity_bytes))
        assert read_tree(ours) == read_tree(ref), (seed, mode)
        for rs, spec in zip(api.restore_checkpoint(os.path.join(ours, "MANIFEST.tlv")), rec.ranks):
            for o, so in zip(rs.objects, spec.objects):
                if o.is_raw():
                    got = o.payload.cpu().numpy() if o.payload.is_cuda else o.payload.numpy()
                    exp = oracle.fill_pattern(so.size, spec.seed, so.space, rec.pit, so.offset)
                    assert (got == exp).all(), (seed, o.object_id)
    finally:
        shutil.rmtree(base, ignore_errors=True)


@pytest.mark.parametrize("flush", [2, 3])
def test_direct_io_engages(gpu, tmp_path, flush):
    """On an O_DIRECT-capable filesystem the aligned bodies of the windows take
    the O_DIRECT path (ticket stat direct_io_bytes) — through io_uring for
    flush_mmap=3 / direct_io="uring" (request counter); the files are checked
    by a restore."""
    import torch

    base = direct_dir(tmp_path)
    if base is None:
        pytest.skip("no O_DIRECT-capable filesystem on this box")
    uring = flush == 3 and api.N.lib.ts_io_uring_available() == 1
    try:
        n = 24 << 20
        x = torch.arange(n // 4, dtype=torch.int32, device="cuda")
        ops0 = api.N.lib.ts_io_uring_ops()
        eng = api.CheckpointEngine(api.EngineConfig(raw_chunk_bytes=4 << 20, staging_capacity_bytes=16 << 20,
                                                    device_staging_bytes=64 << 20, flush_mmap=flush), 0, 0)
        sess = api.CheckpointSession(os.path.join(base, "c"), 1, 1, None, n_ranks=1)
        st = api.RankState(objects=[api.StateObject(1, size_bytes=n, payload=x)])
        t = eng.issue_checkpoint(sess, st, 1)
        eng.pre_update_barrier(t)
        t.wait_persisted()
        sess.wait_complete(60)
        s = t.stats()
        assert s["direct_io_bytes"] >= n - (4 << 20), s
        ops1 = api.N.lib.ts_io_uring_ops()
        assert (ops1 > ops0) == uring, (ops0, ops1)
        rs = api.restore_checkpoint(os.path.join(base, "c", "MANIFEST.tlv"))
        assert torch.equal(rs[0].objects[0].payload.cuda().view(torch.int32).view(-1), x)
        # and read back O_DIRECT
        r = api.Restorer(os.path.join(base, "c", "MANIFEST.tlv"), direct_io="uring" if flush == 3 else True)
        rs = r.restore_rank(0)
        assert r.last_stats["direct_io_bytes"] >= n - (2 << 20), r.last_stats
        assert (api.N.lib.ts_io_uring_ops() > ops1) == uring
        assert torch.equal(rs.objects[0].payload.cuda().view(torch.int32).view(-1), x)
        eng.shutdown()
    finally:
        shutil.rmtree(base, ignore_errors=True)


@pytest.mark.parametrize("seed", range(4))
def test_direct_io_recycled_files(gpu, oracle, tmp_path, seed):
    """Rotation on a disk filesystem with O_DIRECT flushes: checkpoint A's files
    are retired into the spare directory and taken over (renamed, re-sized,
    every byte rewritten) by checkpoint B of the same layout and other bytes;
    B's tree must equal the oracle's."""
    base = direct_dir(tmp_path) or str(tmp_path / "buffered")
    try:
        # same layout (same file names: every file is recycled), other bytes
        ra, rb = random_recipe(random.Random(9100 + seed)), random_recipe(random.Random(9100 + seed))
        for r in rb.ranks:
            r.seed = (r.seed + 1) % 2**64
        spare = os.path.join(base, ".spare")
        cfg = api.EngineConfig(raw_chunk_bytes=65536, staging_capacity_bytes=8 << 20, device_staging_bytes=1 << 24,
                               flush_mmap=2)
        for rec, name in ((ra, "a"), (rb, "b")):
            if name == "b":
                api.retire_checkpoint(os.path.join(base, "a"), spare)
                n_spares = len(os.listdir(spare))
            session = api.CheckpointSession(os.path.join(base, name), rec.ckpt_id, rec.iteration,
                                            rec.manifest_echo(), n_ranks=len(rec.ranks))
            states = [api.materialize_payloads(r, 0, rec.pit) for r in rec.ranks]
            engines = [api.CheckpointEngine(cfg, r.rank_id, 0) for r in rec.ranks]
            for e in engines:
                e.set_spare_dir(spare)
            for t in [e.issue_checkpoint(session, s, rec.iteration) for e, s in zip(engines, states)]:
                t.wait_persisted()
            session.wait_complete(120)
            for e in engines:
                e.shutdown()
        ref = str(tmp_path / "oracle")
        oracle.write_checkpoint(oracle.load_recipe_text(rb.to_text()), ref,
                                ser_chunk=min(cfg.serialized_chunk_bytes, cfg.staging_capacity_bytes))
        assert read_tree(os.path.join(base, "b")) == read_tree(ref), seed
        assert n_spares > 0 and len(os.listdir(spare)) < n_spares  # B took A's files over
    finally:
        shutil.rmtree(base, ignore_errors=True)


@pytest.mark.parametrize("seed", range(6))
def test_direct_io_restore(gpu, oracle, tmp_path, seed):
    """Restore with O_DIRECT reads (Restorer(direct_io=True)) of a checkpoint on
    a disk filesystem: bit-exact shards, same result as the pread path."""
    base = direct_dir(tmp_path) or str(tmp_path / "buffered")
    try:
        rng = random.Random(9300 + seed)
        rec = random_recipe(rng)
        cfg = api.EngineConfig(raw_chunk_bytes=rng.choice([4096, 65536, 1 << 20]), staging_capacity_bytes=8 << 20,
                               device_staging_bytes=1 << 24, flush_mmap=rng.choice([1, 2, 3]))
        ours = os.path.join(base, "ours")
        checkpoint_recipe(rec, ours, cfg)
        os.sync()
        r = api.Restorer(os.path.join(ours, "MANIFEST.tlv"), direct_io=rng.choice([True, "uring"]))
        for i, spec in enumerate(rec.ranks):
            rs = r.restore_rank(i)
            assert rs.rank_id == spec.rank_id
            for o, so in zip(rs.objects, spec.objects):
                if o.is_raw():
                    got = o.payload.cpu().numpy() if o.payload.is_cuda else o.payload.numpy()
                    exp = oracle.fill_pattern(so.size, spec.seed, so.space, rec.pit, so.offset)
                    assert (got == exp).all(), (seed, o.object_id)
    finally:
        shutil.rmtree(base, ignore_errors=True)


def test_auto_direct_io_for_files_dropped_from_page_cache(gpu, tmp_path):
    """The default Restorer (direct_io=None) reads a file that is not in the
    page cache O_DIRECT (the auto mode had no test): the file is
    written, synced and dropped from the cache with posix_fadvise(DONTNEED),
    made read-only (the probe must not depend on write permission), then
    restored bit-exactly with direct_io_bytes > 0."""
    import stat

    import torch

    base = direct_dir(tmp_path)
    if base is None:
        pytest.skip("no O_DIRECT-capable filesystem on this box")
    try:
        n = 64 << 20
        x = torch.arange(n // 4, dtype=torch.int32, device="cuda") * 7
        eng = api.CheckpointEngine(api.EngineConfig(raw_chunk_bytes=8 << 20, staging_capacity_bytes=32 << 20,
                                                    device_staging_bytes=128 << 20, file_dma=False), 0, 0)
        sess = api.CheckpointSession(os.path.join(base, "c"), 1, 1, None, n_ranks=1)
        st = api.RankState(objects=[api.StateObject(1, size_bytes=n, payload=x)])
        t = eng.issue_checkpoint(sess, st, 1)
        t.wait_persisted()
        sess.wait_complete(60)
        eng.shutdown()
        api.file_cache_release_all()
        os.sync()
        for dp, _, fs in os.walk(os.path.join(base, "c")):
            for fn in fs:
                p = os.path.join(dp, fn)
                fd = os.open(p, os.O_RDONLY)
                os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
                os.close(fd)
                os.chmod(p, stat.S_IRUSR | stat.S_IRGRP)
        r = api.Restorer(os.path.join(base, "c", "MANIFEST.tlv"))
        rs = r.restore_rank(0)
        assert torch.equal(rs.objects[0].payload.cuda().view(torch.int32).view(-1), x)
        if r.last_stats["direct_io_bytes"] == 0:
            # a filesystem that keeps the pages resident despite DONTNEED
            # (e.g. tmpfs-backed overlays) cannot show the cold path
            pytest.skip("pages stayed cached after POSIX_FADV_DONTNEED")
        assert r.last_stats["direct_io_bytes"] >= n - (8 << 20), r.last_stats
    finally:
        shutil.rmtree(base, ignore_errors=True)
