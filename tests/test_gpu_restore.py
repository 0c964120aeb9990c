"""Restore on the B200 path (files -> pinned -> H2D -> scatter-unpack) of trees
written by the REFERENCE: restored shards are bit-exact (pattern verified on the
GPU), structured values equal, damage is reported with the reference's error
kinds (format.hpp:50-58) and object ids."""
import os
import shutil

import pytest
import torch

from conftest import GOLDEN, golden_recipes
from paper_2601_16956_b200 import api
from paper_2601_16956_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def expected_structured(oracle, spec, o, pit):
    r = oracle.Rank(spec.rank_id, spec.tp_idx, spec.pp_idx, spec.dp_idx, spec.seed, spec.metadata_bytes)
    oo = oracle.Obj(o.object_id, 1, 1, 2, o.file_id, meta=o.meta)
    v = oracle.structured_value(r, oo, pit)
    if "state_blob" in v:
        v["state_blob"] = v["state_blob"].tobytes()
    return v


@pytest.mark.parametrize("name", golden_recipes())
def test_restore_reference_tree_bit_exact(gpu, oracle, name):
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    ranks = api.restore_checkpoint(os.path.join(GOLDEN, "trees", name, "MANIFEST.tlv"))
    specs = {r.rank_id: r for r in rec.ranks}
    assert sorted(specs) == [r.rank_id for r in ranks]
    for rs in ranks:
        spec = specs[rs.rank_id]
        rs.seed = spec.seed
        by_id = {o.object_id: o for o in spec.objects}
        assert [o.object_id for o in rs.objects] == [o.object_id for o in spec.objects]
        for o in rs.objects:
            so = by_id[o.object_id]
            assert (o.kind, o.residency, o.precision, o.file_id) == (so.kind, so.tier, so.precision, so.file_id)
            if o.is_raw():
                assert o.size_bytes == so.size
                o.pattern_space, o.pattern_offset = so.space, so.offset
            else:
                assert o.structured == expected_structured(oracle, spec, so, rec.pit)
        dev_only = api.RankState(rs.rank_id, seed=spec.seed, arena=rs.arena,
                                 objects=[o for o in rs.objects if o.is_raw() and o.residency == 0])
        assert api.pattern_mismatches(dev_only, rec.pit) == 0
        for o in rs.objects:
            if o.is_raw() and o.residency != 0:
                exp = oracle.fill_pattern(o.size_bytes, spec.seed, o.pattern_space, rec.pit, o.pattern_offset)
                assert (o.payload.numpy() == exp).all()


def _damaged(tmp_path, name="zero3_tiny"):
    d = tmp_path / name
    shutil.copytree(os.path.join(GOLDEN, "trees", name), d)
    return d


def test_restore_detects_corruption(gpu, oracle, tmp_path):
    d = _damaged(tmp_path)
    f = d / "rank_0001" / "file_2.bin"
    entries = oracle.read_footer(str(f))
    oid, kind, foff, ln, base, ck = entries[len(entries) // 2]
    data = bytearray(f.read_bytes())
    data[foff + ln // 2] ^= 0x10
    f.write_bytes(bytes(data))
    with pytest.raises(api.FormatError) as ei:
        api.restore_checkpoint(str(d / "MANIFEST.tlv"))
    assert ei.value.kind == "corrupt_object" and ei.value.object_id == oid
    rep = api.verify_checkpoint(str(d / "MANIFEST.tlv"))
    assert not rep.ok and ("corrupt_object", oid) in rep.issues


def test_restore_detects_truncation_and_missing(gpu, tmp_path):
    d = _damaged(tmp_path)
    f = d / "rank_0002" / "file_1.bin"
    f.write_bytes(f.read_bytes()[:-5])
    with pytest.raises(api.FormatError) as ei:
        api.restore_checkpoint(str(d / "MANIFEST.tlv"))
    assert ei.value.kind == "incomplete_file"
    os.remove(f)
    with pytest.raises(api.FormatError) as ei:
        api.restore_checkpoint(str(d / "MANIFEST.tlv"))
    assert ei.value.kind == "missing_file"
    rep = api.verify_checkpoint(str(d / "MANIFEST.tlv"))
    assert not rep.ok and rep.issues[0][0] == "missing_file"


def test_verify_clean_trees(gpu):
    for name in golden_recipes():
        rep = api.verify_checkpoint(os.path.join(GOLDEN, "trees", name, "MANIFEST.tlv"))
        assert rep.ok, (name, rep.issues)
        assert rep.files_checked > 0


def test_restore_into_existing_shards(gpu, tmp_path):
    """Restore scatters into caller-owned shards (views of a flat buffer at
    2-/4-byte alignment) without touching bytes in between."""
    name = "zero3_tiny"
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    spec = rec.ranks[2]
    for o in spec.objects:
        o.align = 2 if o.precision == 0 else 4
    st = api.materialize_payloads(spec, 0, rec.pit + 7)  # wrong iteration on purpose
    guard = st.arena.clone()
    r = api.Restorer(os.path.join(GOLDEN, "trees", name, "MANIFEST.tlv"))
    r.restore_rank(2, 0, into=st)
    torch.cuda.synchronize()
    assert api.pattern_mismatches(st, rec.pit) == 0
    mask = torch.ones_like(guard, dtype=torch.bool)
    base = st.arena.data_ptr()
    for o in st.objects:
        if o.is_raw():
            a = o.payload.data_ptr() - base
            mask[a:a + o.size_bytes] = False
    assert torch.equal(st.arena[mask], guard[mask])
