"""bench.py's host-side helpers (no GPU): checkpoint cadence rule, the
reference arm's bounded samples, per-workload ncu traffic lookup."""
import os
import sys

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_auto_interval():
    assert bench.auto_interval(440, 1800) == 1      # cfg2: 23.6 GB snapshot fits a step
    assert bench.auto_interval(2140, 1800) == 2     # cfg4: 120.7 GB does not
    assert bench.auto_interval(1700, 1800) == 2     # < 10 % margin
    assert bench.auto_interval(1600, 1800) == 1
    assert bench.auto_interval(0, 0) >= 1


def test_reference_sample_is_bounded_and_labelled():
    rec, whole = bench.sample_recipe("cfg4", 0, 4_000_000_000)
    r = rec.ranks[0]
    raws = [o for o in r.objects if o.kind == 0]
    assert not whole and raws and r.raw_bytes <= 4_000_000_000
    assert [o for o in r.objects if o.kind == 1]  # the rank's metadata object stays
    rec, whole = bench.sample_recipe("cfg1", 0, 10**13)
    assert whole


def test_reference_sample_per_rank_differs():
    a, _ = bench.sample_recipe("cfg2", 0, 2_000_000_000)
    b, _ = bench.sample_recipe("cfg2", 1, 2_000_000_000)
    assert a.ranks[0].rank_id == 0 and b.ranks[0].rank_id == 1


def test_ncu_traffic_lookup():
    t4 = bench.ncu_traffic("cfg4", "ring", "warp")
    assert t4 is not None and 0.99 < t4 / 241_418_598_400 < 1.01
    t2 = bench.ncu_traffic("cfg2", "ring", "bulk")
    assert t2 is not None and 0.99 < t2 / 47_169_153_216 < 1.01
    assert bench.ncu_traffic("cfg3", "ring", "warp") is None
    assert bench.ncu_traffic("cfg4", "direct", "warp") is None
    # HYBRID: captured with another ring size, scaled per algorithmic byte
    th = bench.ncu_traffic("cfg4", "hybrid", "warp", 68_680_618_388)
    assert 0.99 * 68_680_618_388 < th < 68_680_618_388
