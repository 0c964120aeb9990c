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


def verify_files_against_digest(tso, root, files, recipe=None, threads=None):
    """Every byte of each written file against a digest (tests/golden/digests),
    without a second copy of the checkpoint: size; 4 KiB header (the digest's, or
    the one the oracle derives from the recipe's plan); footer table equal to the
    digest's (and its own FNV / length trailer); the oracle's host-threaded FNV-1a
    of every footer range of OUR file equal to the digest's checksum; every byte
    of [4096, tensor_region_end) outside the raw entries zero; the append region's
    sha256 when the digest has it. Returns the number of bytes checked."""
    import hashlib
    import mmap
    import struct

    import numpy as np

    plan_hdr = {}
    if recipe is not None:
        for r in recipe.ranks:
            plan = tso.plan_layout(r.objects)
            ph = tso.plan_hash(plan)
            for fid in plan:
                plan_hdr[f"{tso.rank_dir_name(r.rank_id)}/file_{fid}.bin"] = (
                    tso.MAGIC + struct.pack("<I", 1) + ph.to_bytes(8, "little")).hex()
    checked = 0
    for rel, d in files.items():
        p = os.path.join(root, rel)
        assert os.path.getsize(p) == d["size"], (rel, os.path.getsize(p), d["size"])
        if "footer" not in d:  # MANIFEST.tlv and friends: small, hash them
            with open(p, "rb") as f:
                assert hashlib.sha256(f.read()).hexdigest() == d["sha256"], rel
            continue
        with open(p, "rb") as f:
            mm = mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ)
        try:
            buf = np.frombuffer(mm, dtype=np.uint8)
            hdr = d.get("header") or plan_hdr[rel]
            assert bytes(buf[:20]).hex() == hdr, rel
            assert not np.count_nonzero(buf[20:4096]), rel
            blob_len = struct.unpack("<Q", bytes(buf[-8:]))[0]
            blob = bytes(buf[len(buf) - 8 - blob_len:len(buf) - 8])
            tl = blob_len - 8
            assert struct.unpack("<Q", blob[tl:])[0] == tso.fnv1a64(blob[:tl]), rel
            n = struct.unpack("<Q", blob[:8])[0]
            ents = []
            for i in range(n):
                e = blob[8 + 41 * i: 8 + 41 * (i + 1)]
                oid = struct.unpack("<Q", e[:8])[0]
                foff, ln, base, ck = struct.unpack("<QQQQ", e[9:41])
                ents.append([oid, e[8], foff, ln, base, "%016x" % ck])
            assert ents == d["footer"], rel
            raw = [e for e in ents if e[1] == 0]
            base_addr = buf.ctypes.data
            got = tso.fnv_ranges_many([base_addr + e[2] for e in raw], [e[3] for e in raw], threads)
            bad = [e[0] for e, g in zip(raw, got) if "%016x" % g != e[5]]
            assert not bad, (rel, "objects whose bytes differ", bad[:10])
            tre = d.get("tensor_region_end") or max([e[2] + e[3] for e in raw], default=4096)
            cur = 4096
            for e in sorted(raw, key=lambda e: e[2]):
                if e[2] > cur:
                    assert not np.count_nonzero(buf[cur:e[2]]), (rel, "non-zero gap at", cur)
                cur = e[2] + e[3]
            if tre > cur:
                assert not np.count_nonzero(buf[cur:tre]), (rel, "non-zero tail at", cur)
            app = [e for e in ents if e[1] == 1]
            if app:
                lo = min(e[2] for e in app)
                hi = max(e[2] + e[3] for e in app)
                assert lo == tre and hi == len(buf) - 8 - blob_len, rel
                if "append_sha256" in d:
                    assert hashlib.sha256(buf[lo:hi]).hexdigest() == d["append_sha256"], rel
                else:  # per-object FNV of the concatenated pieces
                    by = {}
                    for e in sorted(app, key=lambda e: (e[0], e[4])):
                        by.setdefault(e[0], [e[5], b""])
                        by[e[0]][1] += bytes(buf[e[2]:e[2] + e[3]])
                    for oid, (ck, b) in by.items():
                        assert "%016x" % tso.fnv1a64(b) == ck, (rel, oid)
            checked += len(buf)
        finally:
            buf = None
            try:
                mm.close()
            except BufferError:  # views still held by a failing assertion's traceback
                pass
    return checked
