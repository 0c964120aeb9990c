"""The product's synthetic-state generator (paper_2601_16956_b200/synthetic.py)
equals the reference's generate_layout (restated in the oracle) object by object."""
import os

import pytest

from conftest import GOLDEN, golden_recipes
from paper_2601_16956_b200 import synthetic as S


@pytest.mark.parametrize("args", [
    (124_439_808, 12, 768, 1, 1, 1, False, 42, 2 << 20),
    (6_738_415_616, 32, 4096, 1, 1, 8, True, 42, 2 << 20),
    (65536, 4, 64, 2, 2, 2, True, 7, 4096),
    (100003, 3, 0, 1, 1, 3, True, 42, 1000),
    (50001, 2, 0, 1, 1, 2, False, 5, 300),
    (10**9 + 7, 7, 0, 3, 2, 5, True, 1, 17),
])
def test_generate_layout_matches_oracle(oracle, args):
    mine = S.generate_layout(*args)
    ref = oracle.generate_layout(*args)
    assert len(mine) == len(ref)
    for a, b in zip(mine, ref):
        assert (a.rank_id, a.tp_idx, a.pp_idx, a.dp_idx, a.seed, a.metadata_bytes) == \
               (b.rank_id, b.tp_idx, b.pp_idx, b.dp_idx, b.seed, b.metadata_bytes)
        assert [(o.object_id, o.kind, o.tier, o.precision, o.file_id, o.size, o.space, o.offset) for o in a.objects] == \
               [(o.object_id, o.kind, o.tier, o.precision, o.file_id, o.size, o.space, o.offset) for o in b.objects]


def test_config_sizes():
    r0 = S.config_recipe("cfg2", 0).ranks[0]
    assert r0.raw_bytes == 23_584_454_656
    assert S.config_recipe("cfg2", 1).ranks[0].raw_bytes == 10_107_623_424
    assert S.config_recipe("cfg1").ranks[0].raw_bytes + 2_097_120 == 1_744_254_432  # + metadata TLV
    g = S.config_recipe("cfg1b").ranks[0]
    assert sum(1 for o in g.objects if o.kind == 0) == 444 and g.raw_bytes == 1_493_277_696
    c3 = S.config_recipe("cfg3", 0).ranks[0]
    assert sum(1 for o in c3.objects if o.kind == 0) == 363 * 4
    assert abs(c3.raw_bytes - 22.78e9) < 0.05e9
    c4 = S.config_recipe("cfg4", 3).ranks[0]
    assert sum(1 for o in c4.objects if o.kind == 0) == 723 * 4
    assert c4.raw_bytes == 68_976_648_192 * 14 // 8


@pytest.mark.parametrize("name", golden_recipes())
def test_recipe_text_roundtrip(name):
    p = os.path.join(GOLDEN, "recipes", name + ".recipe")
    rec = S.load_recipe(p)
    with open(p) as f:
        assert rec.to_text() == f.read()
