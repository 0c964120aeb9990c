"""Error paths of the snapshot engine, against the reference's contract:

* a serializer failure (tlv encode error) fails the ticket and is reported on
  the next wait as ticket_error carrying the stream_error text
  (engine.cpp:341-357, provider.cpp:200-208, transfer.cpp:105-112), and the
  next lazy issue on that engine re-raises it (engine.cpp:523-525);
* a staging acquire past its deadline fails the ticket with "staging failed:
  staging cache: acquire deadline exceeded" (staging.cpp:67-75, engine.cpp:293-300);
* a write error while flushing (full filesystem, file size limit) fails the
  ticket with "flush failed: ..." (engine.cpp:417-423; format.cpp:20-32's
  pwrite_all error) instead of killing the process, and the checkpoint is
  never committed (no MANIFEST.tlv);
* lazy_serialize_overlap=false ("DataStates-Old", engine.cpp:575-576, 612-613)
  writes the same bytes as every other strategy.
"""
import os
import shutil
import subprocess
import sys
import tempfile

import pytest
import torch

from conftest import GOLDEN, ROOT, golden_recipes, read_tree
from gpu_helpers import checkpoint_recipe
from paper_2601_16956_b200 import _native as N
from paper_2601_16956_b200 import api
from paper_2601_16956_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def small_cfg(**kw):
    base = dict(d2h_mode="ring", raw_chunk_bytes=1 << 20, staging_capacity_bytes=4 << 20,
                device_staging_bytes=2 << 20, flush_workers=2)
    base.update(kw)
    return api.EngineConfig(**base)


def rank_with(raw_sizes, structured=None, seed=5):
    spec = S.RankSpec(0, seed=seed, metadata_bytes=64)
    oid = 1
    for sz in raw_sizes:
        spec.objects.append(S.ObjSpec(oid, 0, 0, 1, 1, sz, S.pack_space(2, oid, 0), 0))
        oid += 1
    spec.objects.append(S.ObjSpec(oid, 1, 1, 2, 1, meta=("meta",)))
    st = api.materialize_payloads(spec, 0, 1)
    if structured is not None:
        st.objects.append(api.StateObject(oid + 1, kind=api.KIND_STRUCTURED, residency=api.TIER_HOST,
                                          precision=2, file_id=1, structured=structured))
    return spec, st


def bad_utf8_value():
    return api.Value(N.lib.ts_value_string(b"ok\xff\xfe", 4))


@pytest.mark.parametrize("overlap", [True, False])
def test_serializer_failure_is_a_deferred_ticket_error(gpu, tmp_path, overlap):
    spec, st = rank_with([3 << 20], structured=bad_utf8_value())
    bad_oid = st.objects[-1].object_id
    eng = api.CheckpointEngine(small_cfg(lazy_serialize_overlap=overlap), 0, 0)
    sess = api.CheckpointSession(str(tmp_path / "a"), 1, 1, None, 1)
    t = eng.issue_checkpoint(sess, st, 1)  # lazy: issue itself does not raise
    with pytest.raises(api.TicketError) as ei:
        t.wait_persisted()
    assert str(ei.value) == f"object {bad_oid}: tlv: non-utf8 string at $"
    with pytest.raises(api.TicketError):
        t.wait_snapshot()
    assert t.stats()["failed"]
    # the next lazy issue waits for the previous snapshot and re-raises its failure
    sess2 = api.CheckpointSession(str(tmp_path / "b"), 2, 2, None, 1)
    with pytest.raises(api.TicketError):
        eng.issue_checkpoint(sess2, st, 2)
    assert not os.path.exists(tmp_path / "a" / "MANIFEST.tlv")
    eng.shutdown()


@pytest.mark.parametrize("strategy", ["sync", "two_phase"])
def test_serializer_failure_blocking_strategies_raise_at_issue(gpu, tmp_path, strategy):
    _, st = rank_with([1 << 20], structured=bad_utf8_value())
    eng = api.CheckpointEngine(small_cfg(strategy=strategy), 0, 0)
    sess = api.CheckpointSession(str(tmp_path / "a"), 1, 1, None, 1)
    with pytest.raises(api.TicketError, match="tlv: non-utf8 string"):
        eng.issue_checkpoint(sess, st, 1)
    eng.shutdown()


def test_cache_acquire_deadline(gpu, tmp_path):
    """A one-window pool with a zero acquire deadline: the copier's second
    window cannot get space in time (the first is still in flight)."""
    _, st = rank_with([64 << 20])
    eng = api.CheckpointEngine(small_cfg(staging_capacity_bytes=1 << 20, file_dma=False,
                                         cache_acquire_timeout_ns=0, d2h_mode="direct"), 0, 0)
    sess = api.CheckpointSession(str(tmp_path / "a"), 1, 1, None, 1)
    t = eng.issue_checkpoint(sess, st, 1)
    with pytest.raises(api.TicketError) as ei:
        t.wait_persisted()
    assert str(ei.value) == "staging failed: staging cache: acquire deadline exceeded"
    # a barrier on a failed ticket does not hang either
    with pytest.raises(api.TicketError):
        eng.pre_update_barrier(t, host_block=2)
    eng.shutdown()
    assert not os.path.exists(tmp_path / "a" / "MANIFEST.tlv")


def test_cache_deadline_met_when_generous(gpu, tmp_path):
    """The same pool with a generous deadline completes byte-identically."""
    name = "tiny_layout"
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    out = str(tmp_path / "ok")
    checkpoint_recipe(rec, out, small_cfg(staging_capacity_bytes=8192, raw_chunk_bytes=8192, file_dma=False,
                                          cache_acquire_timeout_ns=30 * 10**9, d2h_mode="direct"))
    assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))


_FSIZE_CHILD = r"""
import os, resource, signal, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, os.path.join(sys.argv[1], "tests"))
signal.signal(signal.SIGXFSZ, signal.SIG_IGN)
from test_gpu_errors import rank_with, small_cfg
from paper_2601_16956_b200 import api
out, flush_mmap = sys.argv[2], int(sys.argv[3])
_, st = rank_with([8 << 20, 3 << 20], structured={"blob": "x" * (1 << 20)})
eng = api.CheckpointEngine(small_cfg(flush_mmap=flush_mmap, file_dma=False), 0, 0)
# the fixed region fits (the file is pre-sized at issue), the append region does not
resource.setrlimit(resource.RLIMIT_FSIZE, (int(sys.argv[4]), resource.RLIM_INFINITY))
sess = api.CheckpointSession(out, 1, 1, None, 1)
t = eng.issue_checkpoint(sess, st, 1)
try:
    t.wait_persisted()
    print("NO ERROR")
except api.TicketError as e:
    print("TICKET_ERROR", e)
eng.shutdown()
print("MANIFEST", os.path.exists(os.path.join(out, "MANIFEST.tlv")))
"""


@pytest.mark.parametrize("flush_mmap", [0, 1, 2])
def test_flush_write_error_fails_ticket(gpu, tmp_path, flush_mmap):
    """A write failing during the flush (EFBIG past RLIMIT_FSIZE) surfaces as
    'flush failed: ...' on wait_persisted; no manifest is committed."""
    out = str(tmp_path / "ck")
    tre = 4096 + (8 << 20) + (3 << 20)  # header + both raw objects (2 MiB aligned, contiguous)
    r = subprocess.run([sys.executable, "-c", _FSIZE_CHILD, ROOT, out, str(flush_mmap), str(tre + 4096)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = dict(l.split(" ", 1) for l in r.stdout.splitlines() if " " in l)
    assert "TICKET_ERROR" in lines, r.stdout
    assert lines["TICKET_ERROR"].startswith(("flush failed: ", "finalize failed: ")), lines
    assert lines["MANIFEST"] == "False"


def _small_tmpfs():
    d = tempfile.mkdtemp()
    r = subprocess.run(["mount", "-t", "tmpfs", "-o", "size=16m", "tmpfs", d], capture_output=True)
    if r.returncode != 0:
        os.rmdir(d)
        return None
    return d


@pytest.mark.parametrize("flush_mmap", [0, 1])
def test_enospc_on_flush_fails_ticket_not_process(gpu, flush_mmap):
    """A 16 MiB tmpfs and a 48 MiB checkpoint: the writes (mapped copies reserve
    their range with fallocate first) fail with ENOSPC as a ticket error, never a
    SIGBUS (mapped writes on a full tmpfs)."""
    d = _small_tmpfs()
    if d is None:
        pytest.skip("cannot mount a small tmpfs here (needs CAP_SYS_ADMIN)")
    try:
        _, st = rank_with([32 << 20, 16 << 20])
        eng = api.CheckpointEngine(small_cfg(flush_mmap=flush_mmap, file_dma=False), 0, 0)
        sess = api.CheckpointSession(os.path.join(d, "ck"), 1, 1, None, 1)
        t = eng.issue_checkpoint(sess, st, 1)
        with pytest.raises(api.TicketError, match="^(flush|finalize) failed: "):
            t.wait_persisted()
        eng.shutdown()
        assert not os.path.exists(os.path.join(d, "ck", "MANIFEST.tlv"))
    finally:
        subprocess.run(["umount", d])
        shutil.rmtree(d, ignore_errors=True)


@pytest.mark.parametrize("name", golden_recipes())
def test_lazy_without_serialize_overlap_identical(gpu, tmp_path, name):
    """DataStates-Old: structured objects serialized inline on the training
    thread at issue (engine.cpp:575-576, 612-613); same bytes as the reference."""
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    out = str(tmp_path / "old")
    cfg = api.EngineConfig(raw_chunk_bytes=64 << 10, staging_capacity_bytes=1 << 20,
                           device_staging_bytes=256 << 10, flush_workers=3, lazy_serialize_overlap=False)
    _, _, stats, _ = checkpoint_recipe(rec, out, cfg)
    assert read_tree(out) == read_tree(os.path.join(GOLDEN, "trees", name))
    for s in stats:
        assert s["persisted_done"] and not s["failed"]
