"""Randomized parity (SPEC.md:419-422 round-trip / determinism properties): random
rank states (sizes 1 B..1 MiB, random file ids, host/device tiers, source
alignments 1..256 B, structured objects) checkpointed by the GPU engine under
random engine configurations must equal, byte for byte, the oracle's canonical
checkpoint (the oracle is pinned to the compiled reference by test_oracle.py),
and restore bit-exactly."""
import os
import random

import pytest

from conftest import read_tree
from gpu_helpers import checkpoint_recipe
from paper_2601_16956_b200 import api
from paper_2601_16956_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def random_recipe(rng: random.Random) -> S.Recipe:
    nranks = rng.choice([1, 1, 2, 3])
    rec = S.Recipe("fuzz", rng.randrange(1, 100), rng.randrange(1, 1000), rng.choice([None, rng.randrange(0, 50)]))
    oid = rng.randrange(1, 1000)
    for r in range(nranks):
        rs = S.RankSpec(r, rng.randrange(4), rng.randrange(4), rng.randrange(4), rng.randrange(2**64),
                        rng.choice([0, 16, 300, 5000, 1 << 20, (1 << 20) + 77]))
        for _ in range(rng.randrange(1, 40)):
            if rng.random() < 0.15:
                meta = ("meta",) if rng.random() < 0.5 else ("tmeta", "t%d" % oid, rng.choice(["bf16", "fp32"]),
                                                           rng.randrange(1, 10**6), 0, rng.randrange(1, 10**5))
                rs.objects.append(S.ObjSpec(oid, 1, 1, 2, rng.choice([0, 1, 3]), meta=meta))
            else:
                size = rng.choice([1, 2, 15, 16, 17, 4095, 4096, 4097, rng.randrange(1, 1 << 20), rng.randrange(1, 5000)])
                o = S.ObjSpec(oid, 0, 0 if rng.random() < 0.85 else 1, rng.randrange(3), rng.choice([0, 1, 2, 7]),
                              size, rng.randrange(2**64), rng.randrange(2**40))
                o.align = rng.choice([1, 2, 4, 8, 16, 256])
                rs.objects.append(o)
            oid += rng.randrange(1, 5)
        rec.ranks.append(rs)
    return rec


def random_cfg(rng):
    mode = rng.choice(["ring", "direct", "zerocopy", "hybrid"])
    w = rng.choice([4096, 10_000, 65536, 1 << 20])
    return api.EngineConfig(
        d2h_mode=mode, raw_chunk_bytes=w, staging_capacity_bytes=rng.choice([w, 2 * w + 7, 8 << 20]),
        device_staging_bytes=rng.choice([8192, 1 << 16, 1 << 24]), flush_workers=rng.choice([1, 2, 5]),
        checksum_on_gpu=rng.random() < 0.7, flush_mmap=rng.choice([0, 1, 1, 2]),
        pack_kernel=rng.choice(["warp", "bulk"]), bulk_min_bytes=32768,
        serialized_chunk_bytes=rng.choice([1 << 20, 1 << 20, 4096]),
        hybrid_direct_min_bytes=0)  # (the HYBRID head path even for tiny fragments)


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_parity_with_oracle(gpu, oracle, tmp_path, seed):
    rng = random.Random(1000 + seed)
    rec = random_recipe(rng)
    cfg = random_cfg(rng)
    ours = str(tmp_path / "ours")
    checkpoint_recipe(rec, ours, cfg)
    ref = str(tmp_path / "oracle")
    orec = oracle.load_recipe_text(rec.to_text())
    oracle.write_checkpoint(orec, ref, ser_chunk=min(cfg.serialized_chunk_bytes, cfg.staging_capacity_bytes))
    assert read_tree(ours) == read_tree(ref), (seed, cfg)
    # bit-exact restore of every raw object
    for rs, spec in zip(api.restore_checkpoint(os.path.join(ours, "MANIFEST.tlv")), rec.ranks):
        for o, so in zip(rs.objects, spec.objects):
            if o.is_raw():
                got = o.payload.cpu().numpy() if o.payload.is_cuda else o.payload.numpy()
                exp = oracle.fill_pattern(so.size, spec.seed, so.space, rec.pit, so.offset)
                assert (got == exp).all(), (seed, o.object_id)
