"""Parity of the B200 snapshot path with the reference: checkpoint trees written
by the GPU engine are byte-identical to the trees the compiled reference wrote
for the same state (tests/golden/trees), in every D2H mode, with windows and
staging pools small enough to force multi-window pipelines and back-pressure."""
import json
import os
import shutil
import subprocess

import pytest
import torch

from conftest import GOLDEN, ROOT, golden_recipes, read_tree
from gpu_helpers import checkpoint_recipe
from paper_2601_16956_b200 import api
from paper_2601_16956_b200 import synthetic as S

pytestmark = pytest.mark.gpu
MODES = ["ring", "direct", "zerocopy", "ring-bulk", "hybrid"]


def cfg_for(mode, **kw):
    extra = {}
    if mode == "ring-bulk":  # TMA bulk copies for every fragment >= 32 KiB
        # (a full device shadow: the bulk path is used for one-pack images only)
        mode, extra = "ring", dict(pack_kernel="bulk", bulk_min_bytes=32768, device_staging_bytes=256 << 20)
    elif mode == "hybrid":  # the head path even for the goldens' KiB-sized fragments
        extra = dict(hybrid_direct_min_bytes=0)
    base = dict(d2h_mode=mode, raw_chunk_bytes=64 << 10, staging_capacity_bytes=1 << 20,
                device_staging_bytes=256 << 10, flush_workers=3)
    base.update(extra)
    base.update(kw)
    return api.EngineConfig(**base)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", golden_recipes())
def test_snapshot_bytes_equal_reference(gpu, tmp_path, name, mode):
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    out = str(tmp_path / "ckpt")
    _, states, stats, _ = checkpoint_recipe(rec, out, cfg_for(mode))
    assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))
    # the capture never modifies the state
    for st in states:
        assert api.pattern_mismatches(st, rec.pit) == 0
    for s in stats:
        assert s["snapshot_done"] and s["persisted_done"] and not s["failed"]


@pytest.mark.parametrize("name", ["hand_mixed", "zero3_tiny", "odd_layout"])
@pytest.mark.parametrize("mode", MODES)
def test_host_checksums_identical(gpu, tmp_path, name, mode):
    """checksum_on_gpu=0 (host FNV threads over the pinned pool) writes the same bytes."""
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    out = str(tmp_path / "ckpt")
    checkpoint_recipe(rec, out, cfg_for(mode, checksum_on_gpu=False))
    assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))


@pytest.mark.parametrize("strategy", ["sync", "two_phase", "lazy"])
def test_strategies_identical(gpu, tmp_path, strategy):
    name = "hand_mixed"
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    out = str(tmp_path / strategy)
    checkpoint_recipe(rec, out, cfg_for("ring", strategy=strategy))
    assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))


def test_shadow_ring_and_window_sizes(gpu, tmp_path):
    """Full device shadow, 2-slot ring, 1-window pool and huge windows agree."""
    name = "zero3_tiny"
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    ref = read_tree(os.path.join(GOLDEN, "trees", name))
    for i, kw in enumerate([dict(device_staging_bytes=1 << 30, raw_chunk_bytes=16 << 20, staging_capacity_bytes=64 << 20),
                            dict(device_staging_bytes=8 << 10, raw_chunk_bytes=4096, staging_capacity_bytes=4096),
                            dict(raw_chunk_bytes=10_000, staging_capacity_bytes=30_000, flush_workers=1)]):
        out = str(tmp_path / str(i))
        checkpoint_recipe(rec, out, cfg_for("ring", **kw))
        assert read_tree(out) == ref, kw


def test_consecutive_checkpoints_and_checksums(gpu, tmp_path, oracle):
    """Three lazy checkpoints of one rank through one engine with updates in
    between (run_training's loop): each checkpoint holds its own iteration."""
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", "odd_layout.recipe"))
    spec = rec.ranks[1]
    st = api.materialize_payloads(spec, 0, 0)
    eng = api.CheckpointEngine(cfg_for("ring"), spec.rank_id, 0)
    pending = None
    for it in range(1, 4):
        eng.pre_update_barrier(pending, host_block=1)
        api.mutate_update_step(st, it)
        sess = api.CheckpointSession(str(tmp_path / f"c{it}"), it, it, None, n_ranks=1)
        pending = eng.issue_checkpoint(sess, st, it)
        pending.wait_persisted()
        sess.wait_complete(30)
        for o in spec.objects:
            if o.kind == 0:
                exp = oracle.fnv1a64(oracle.fill_pattern(o.size, spec.seed, o.space, it, o.offset))
                assert pending.object_checksum(o.object_id) == exp
        restored = oracle.restore_checkpoint(str(tmp_path / f"c{it}" / "MANIFEST.tlv"))
        assert restored[0]["objects"][spec.objects[-1].object_id]["iteration"] == it
    eng.shutdown()


def test_lazy_barrier_is_load_bearing(gpu, tmp_path):
    """With the pre-update barrier (stream wait, no host block) an update issued
    right after the checkpoint cannot leak into it; skipping the barrier lets it
    leak (the reference's skip_update_barrier negative test, simulator.hpp:81-83)."""
    spec = S.RankSpec(0, seed=3, metadata_bytes=100)
    spec.objects = [S.ObjSpec(1, 0, 0, 1, 1, 64 << 20, S.pack_space(2, 0, 0), 0),
                    S.ObjSpec(2, 1, 1, 2, 0, meta=("meta",))]
    prod = torch.cuda.Stream()
    st = api.materialize_payloads(spec, 0, 1, stream=prod)
    eng = api.CheckpointEngine(cfg_for("ring", device_staging_bytes=8 << 20, raw_chunk_bytes=4 << 20,
                                       staging_capacity_bytes=16 << 20), 0, 0)
    for use_barrier in (True, False):
        with torch.cuda.stream(prod):
            torch.cuda._sleep(200_000_000)  # the producer is still busy at issue time
        sess = api.CheckpointSession(str(tmp_path / str(use_barrier)), 1, 1, None, 1)
        t = eng.issue_checkpoint(sess, st, 1, producer_stream=prod)
        upd = torch.cuda.Stream()
        if use_barrier:
            eng.pre_update_barrier(t, stream=upd, host_block=0)
        api.mutate_update_step(st, 2, stream=upd)
        t.wait_persisted()
        sess.wait_complete(30)
        r = api.restore_checkpoint(str(tmp_path / str(use_barrier) / "MANIFEST.tlv"))[0]
        raw = [o for o in r.objects if o.is_raw()][0]
        raw.pattern_space, raw.pattern_offset = spec.objects[0].space, 0
        r.seed = spec.seed
        bad = api.pattern_mismatches(r, 1)
        if use_barrier:
            assert bad == 0
        else:
            assert bad > 0
        torch.cuda.synchronize()
        api.mutate_update_step(st, 1)
        torch.cuda.synchronize()
    eng.shutdown()


def test_reference_restores_our_checkpoint(gpu, tmp_path):
    """The unmodified reference (oracle/_ref/ts_ref_driver) verifies and restores a
    checkpoint written by the B200 engine, with identical object checksums."""
    drv = os.path.join(ROOT, "oracle", "_ref", "ts_ref_driver")
    if not os.path.exists(drv):
        pytest.skip("oracle/_ref not built")
    rec = S.zero3_recipe("z", S.llama_tensors(96, 200, 3, vocab=300), 3, seed=5, metadata_bytes=5000,
                         iteration=4)
    out = str(tmp_path / "ours")
    _, _, stats, _ = checkpoint_recipe(rec, out, cfg_for("ring"))
    v = json.loads(subprocess.run([drv, "verify", out + "/MANIFEST.tlv"], capture_output=True, text=True,
                                  check=True).stdout)
    assert v["ok"] and v["objects"] == sum(len(r.objects) for r in rec.ranks)
    r = json.loads(subprocess.run([drv, "restore", out + "/MANIFEST.tlv"], capture_output=True, text=True,
                                  check=True).stdout)
    assert r["ok"]


def test_back_pressure_bounded_pool(gpu, tmp_path):
    """Staging capacity far below the checkpoint: lazy still completes (SPEC
    back-pressure property) and the bytes are unchanged."""
    name = "tiny_layout"
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    out = str(tmp_path / "bp")
    checkpoint_recipe(rec, out, cfg_for("direct", staging_capacity_bytes=8192, raw_chunk_bytes=8192))
    assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))


@pytest.mark.parametrize("name", ["hand_mixed", "odd_layout", "zero3_tiny"])
def test_rotation_reuses_files_byte_identical(gpu, tmp_path, name):
    """Checkpoint rotation: a checkpoint written over files recycled from a
    retired, different checkpoint (other iteration, other layout: larger and
    smaller files) is byte-identical to the reference's."""
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    other = S.load_recipe(os.path.join(GOLDEN, "recipes", "tiny_layout.recipe"))
    spare = str(tmp_path / "spare")
    # an unrelated checkpoint of the same rank ids to recycle
    for r, o in zip(rec.ranks, other.ranks):
        o.rank_id = r.rank_id
    other.ranks = other.ranks[:len(rec.ranks)]
    old = str(tmp_path / "old")
    checkpoint_recipe(other, old, cfg_for("ring"))
    api.retire_checkpoint(old, spare)
    assert not os.path.exists(old)
    assert len(os.listdir(spare)) > 0
    session = api.CheckpointSession(str(tmp_path / "new"), rec.ckpt_id, rec.iteration, rec.manifest_echo(),
                                    n_ranks=len(rec.ranks))
    states = [api.materialize_payloads(r, 0, rec.pit) for r in rec.ranks]
    engines = [api.CheckpointEngine(cfg_for("ring"), r.rank_id, 0) for r in rec.ranks]
    for e in engines:
        e.set_spare_dir(spare)
    tickets = [e.issue_checkpoint(session, s, rec.iteration) for e, s in zip(engines, states)]
    for t in tickets:
        t.wait_persisted()
    session.wait_complete(60)
    for e in engines:
        e.shutdown()
    assert read_tree(str(tmp_path / "new")) == read_tree(os.path.join(GOLDEN, "trees", name))


def test_retired_checkpoint_is_not_restorable(gpu, tmp_path):
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", "two_ranks.recipe"))
    d = str(tmp_path / "c")
    checkpoint_recipe(rec, d, cfg_for("ring"))
    assert api.verify_checkpoint(os.path.join(d, "MANIFEST.tlv")).ok
    api.retire_checkpoint(d, str(tmp_path / "spare"))
    with pytest.raises(api.FormatError) as ei:
        api.restore_checkpoint(os.path.join(d, "MANIFEST.tlv"))
    assert ei.value.kind == "missing_file"


@pytest.mark.parametrize("frac", [0.0, 0.3, 0.5, 1.0])
@pytest.mark.parametrize("mode", ["ring", "direct", "zerocopy", "hybrid"])
@pytest.mark.parametrize("name", ["hand_mixed", "zero3_tiny", "two_ranks"])
def test_checksum_split_identical(gpu, tmp_path, name, mode, frac):
    """Checksum placement split between the FNV kernels and host workers
    (checksum_host_frac) writes the same bytes; the host share is honoured."""
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    out = str(tmp_path / "ckpt")
    _, _, stats, _ = checkpoint_recipe(rec, out, cfg_for(mode, checksum_host_frac=frac))
    assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))
    dev = sum(o.size for r in rec.ranks for o in r.objects if o.kind == 0 and o.tier == 0)
    host = sum(s["host_checksum_bytes"] for s in stats)
    if frac == 0.0:
        assert host == 0
    elif frac == 1.0:
        assert host == dev
    else:
        assert 0 <= host <= dev


@pytest.mark.parametrize("share", [0.3, 1.0])
@pytest.mark.parametrize("staging", [256 << 10, 64 << 20])  # ring of slots / full device shadow
@pytest.mark.parametrize("name", ["hand_mixed", "odd_layout", "two_ranks", "zero3_tiny"])
def test_helper_gpu_d2h_identical(gpu, tmp_path, name, staging, share):
    """D2H load balancing (helper_devices): part of the windows copied by a
    helper GPU's copy engine (here the same device through a second stream; on a
    multi-GPU node a peer reading over NVLink) — the same bytes either way."""
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    out = str(tmp_path / "ckpt")
    _, _, stats, _ = checkpoint_recipe(rec, out, cfg_for("ring", device_staging_bytes=staging,
                                                         helper_devices=(0,), helper_share=share))
    assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))
    helper = sum(s["helper_bytes"] for s in stats)
    image = sum(s["image_bytes"] for s in stats)
    assert 0 < helper <= image
    if share == 1.0:
        assert helper == image or helper >= image - (64 << 10)  # every window (padding never moves)


@pytest.mark.parametrize("name", ["hand_mixed", "odd_layout", "tiny_layout", "nozero_dp2"])
def test_bulk_path_engaged_on_shadow(gpu, tmp_path, name):
    """With a full device shadow the TMA bulk kernel carries the large aligned
    fragments (one extra launch per rank) and the bytes stay identical; in a
    multi-slot ring only the warp kernel runs."""
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    launches = {}
    for label, kw in (("warp", dict(pack_kernel="warp", device_staging_bytes=256 << 20)),
                      ("bulk", dict(pack_kernel="bulk", bulk_min_bytes=32768, device_staging_bytes=256 << 20)),
                      ("ring", dict(pack_kernel="bulk", bulk_min_bytes=32768))):
        out = str(tmp_path / label)
        _, _, stats, _ = checkpoint_recipe(rec, out, cfg_for("ring", **kw))
        assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))
        launches[label] = sum(s["kernel_launches"] for s in stats)
    ranks_with_big = sum(1 for r in rec.ranks if any(o.kind == 0 and o.tier == 0 and o.size >= 32768 for o in r.objects))
    assert launches["bulk"] == launches["warp"] + ranks_with_big


@pytest.mark.parametrize("name", ["hand_mixed", "odd_layout", "tiny_layout", "nozero_dp2"])
def test_bulk_ring_two_stage_kernel(gpu, tmp_path, name):
    """pack_kernel="bulk-ring": the 2-stage (64 KiB shared memory) TMA bulk
    kernel also runs in a multi-slot HBM ring (one launch per ring chunk that
    holds bulk jobs); the bytes stay identical to the reference's."""
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    launches = {}
    for label, pk in (("warp", "warp"), ("bulk-ring", "bulk-ring")):
        out = str(tmp_path / label)
        # windows of 64 KiB (2 bulk jobs), a 4-window ring: many chunks per rank
        _, _, stats, _ = checkpoint_recipe(rec, out, cfg_for("ring", pack_kernel=pk, bulk_min_bytes=32768,
                                                             raw_chunk_bytes=64 << 10, device_staging_bytes=256 << 10))
        assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))
        launches[label] = sum(s["kernel_launches"] for s in stats)
    big = any(o.kind == 0 and o.tier == 0 and o.size >= 65536 for r in rec.ranks for o in r.objects)
    if big:
        assert launches["bulk-ring"] > launches["warp"]


@pytest.mark.parametrize("mode", ["ring", "direct", "zerocopy"])
def test_bounded_enqueue_many_windows(gpu, tmp_path, mode):
    """~1,300 windows of 64 KiB (the copier keeps at most 256 in flight and
    packs run a ring-full ahead of the copies): bytes and checksums intact."""
    n = (80 << 20) + 12345
    x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    eng = api.CheckpointEngine(api.EngineConfig(d2h_mode=mode, raw_chunk_bytes=64 << 10, staging_capacity_bytes=8 << 20,
                                                device_staging_bytes=2 << 20, flush_workers=3), 0, 0)
    sess = api.CheckpointSession(str(tmp_path / "c"), 1, 1, None, n_ranks=1)
    st = api.RankState(objects=[api.StateObject(1, size_bytes=n, payload=x),
                                api.StateObject(2, kind=api.KIND_STRUCTURED, residency=api.TIER_HOST, file_id=0,
                                                structured={"n": n})])
    t = eng.issue_checkpoint(sess, st, 1)
    eng.pre_update_barrier(t)
    t.wait_persisted()
    sess.wait_complete(60)
    assert t.object_checksum(1) == api.fnv1a64(x.cpu().numpy().tobytes())
    eng.shutdown()
    rs = api.restore_checkpoint(str(tmp_path / "c" / "MANIFEST.tlv"))
    assert torch.equal(rs[0].objects[0].payload.cuda(), x)


@pytest.mark.parametrize("mode", ["ring", "hybrid"])
@pytest.mark.parametrize("lane_max", [0, 4096, 1 << 40])
@pytest.mark.parametrize("staging", [256 << 10, 64 << 20])  # ring of slots / full device shadow
@pytest.mark.parametrize("name", ["hand_mixed", "odd_layout", "zero3_tiny", "two_ranks", "tiny_layout"])
def test_lane_checksums_identical(gpu, tmp_path, name, staging, lane_max, mode):
    """Device checksums by the lane-serial FNV kernel over the state (objects up
    to checksum_lane_max_bytes) next to the segment-parallel kernels over the
    ring slots: same bytes as the reference; the lane share is reported."""
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    out = str(tmp_path / "ckpt")
    _, states, stats, _ = checkpoint_recipe(
        rec, out, cfg_for(mode, checksum_lane_max_bytes=lane_max, checksum_host_frac=0.0,
                          device_staging_bytes=staging))
    assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))
    for st in states:
        assert api.pattern_mismatches(st, rec.pit) == 0
    dev = [o.size for r in rec.ranks for o in r.objects if o.kind == 0 and o.tier == 0]
    lane = sum(s["lane_checksum_bytes"] for s in stats)
    want = sum(x for x in dev if x <= lane_max)
    assert lane == want
    if lane:
        assert all(s["lane_ms"] > 0 for s in stats if s["lane_checksum_bytes"])
