"""The CPU oracle pinned against the reference: KATs and the
golden trees written by the compiled reference (tests/golden/make_golden.py)."""
import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, golden_recipes, read_tree

SURVEY_KATS = {
    "fnv_empty": "cbf29ce484222325",
    "fnv_a": "af63dc4c8601ec8c",
    "fnv_foobar": "85944171f73967e8",
    "pattern_42_L0_it0_off0": "380a127ea7eb6f998c5f5a543e8a98cb157179520c47be1c",
    "pattern_42_L0_it1_off5": "3a4be0a8bf26ad20a40a2c982e742067883644ad1206354f",
    "tlv_iter7_seed42": "060200000000000000030900000000000000697465726174696f6e010700000000000000"
                        "030800000000000000726e675f73656564012a00000000000000",
    "tlv_empty_map": "060000000000000000",
    "plan3_hash": "311b94ed6e450ef0",
    "plan1_hash": "86f05cc9e002c195",
}


def kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


def test_kat_file_matches_survey():
    k = kat()
    for key, v in SURVEY_KATS.items():
        assert k[key] == v, key
    assert k["plan3_offsets"] == [4096, 3500007424, 4500008960]
    assert k["plan3_end_f1"] == 4500013056 and k["plan3_end_f0"] == 4096
    assert k["metadata_2MiB_len"] == 2097120


def test_oracle_kats(oracle):
    k = kat()
    assert "%016x" % oracle.fnv1a64(b"") == k["fnv_empty"]
    assert "%016x" % oracle.fnv1a64(b"a") == k["fnv_a"]
    assert "%016x" % oracle.fnv1a64(b"foobar") == k["fnv_foobar"]
    sp = oracle.pack_space(1, 0, 0)
    assert oracle.fill_pattern(24, 42, sp, 0, 0).tobytes().hex() == k["pattern_42_L0_it0_off0"]
    assert oracle.fill_pattern(24, 42, sp, 1, 5).tobytes().hex() == k["pattern_42_L0_it1_off5"]
    assert oracle.tlv_encode({"iteration": 7, "rng_seed": 42}).hex() == k["tlv_iter7_seed42"]
    assert oracle.tlv_encode({}).hex() == k["tlv_empty_map"]
    assert oracle.tlv_encode([None, 1.5, "hé", b"\x01\x02", -3]).hex() == k["tlv_mixed_list"]
    objs = [oracle.Obj(1, 0, 0, 0, 1, 3_500_000_000), oracle.Obj(2, 0, 0, 0, 1, 1_000_000_000),
            oracle.Obj(3, 0, 0, 0, 1, 4096), oracle.Obj(4, 1, 1, 2, 0)]
    plan = oracle.plan_layout(objs)
    assert [off for _, off, _ in plan[1].fixed] == k["plan3_offsets"]
    assert plan[1].tensor_region_end == k["plan3_end_f1"] and plan[0].tensor_region_end == 4096
    assert "%016x" % oracle.plan_hash(plan) == k["plan3_hash"]
    assert "%016x" % oracle.plan_hash(oracle.plan_layout([oracle.Obj(1, 0, 0, 0, 1, 4096)])) == k["plan1_hash"]
    assert "%016x" % oracle.plan_hash(oracle.plan_layout([])) == k["plan_empty_hash"]
    r = oracle.Rank(0, seed=42, metadata_bytes=2 << 20)
    enc = oracle.tlv_encode(oracle.make_metadata_value(r, 0))
    assert len(enc) == k["metadata_2MiB_len"]
    assert "%016x" % oracle.fnv1a64(enc) == k["metadata_2MiB_fnv"]


def test_fnv_chained(oracle):
    data = np.arange(1000, dtype=np.uint8)
    h = oracle.fnv1a64(data[:300])
    assert oracle.fnv1a64(data[300:], h) == oracle.fnv1a64(data)


def test_pattern_windows_are_consistent(oracle):
    full = oracle.fill_pattern(4096, 9, 77, 3, 0)
    for off in (0, 1, 7, 8, 9, 1000, 4000):
        assert (oracle.fill_pattern(50, 9, 77, 3, off)[: max(0, min(50, 4096 - off))] ==
                full[off:off + 50]).all()
    assert oracle.match_pattern(full[5:100], 9, 77, 3, 5) == -1
    bad = full[5:100].copy()
    bad[17] ^= 1
    assert oracle.match_pattern(bad, 9, 77, 3, 5) == 17


@pytest.mark.parametrize("name", golden_recipes())
def test_oracle_writes_reference_bytes(oracle, tmp_path, name):
    rec = oracle.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    oracle.write_checkpoint(rec, str(tmp_path))
    assert read_tree(str(tmp_path)) == read_tree(os.path.join(GOLDEN, "trees", name))


@pytest.mark.parametrize("name", golden_recipes())
def test_oracle_restores_reference_tree(oracle, name):
    rec = oracle.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    ranks = oracle.restore_checkpoint(os.path.join(GOLDEN, "trees", name, "MANIFEST.tlv"))
    by_id = {r.rank_id: r for r in rec.ranks}
    for rr in ranks:
        spec = by_id[rr["rank_id"]]
        for o in spec.objects:
            got = rr["objects"][o.object_id]
            if o.kind == 0:
                assert got == oracle.payload_of(spec, o, rec.pit).tobytes()
            else:
                exp = oracle.structured_value(spec, o, rec.pit)
                if "state_blob" in exp:
                    exp["state_blob"] = exp["state_blob"].tobytes()
                assert got == exp


def _copy(name, tmp_path):
    dst = tmp_path / name
    shutil.copytree(os.path.join(GOLDEN, "trees", name), dst)
    return dst


def test_oracle_detects_tamper_truncation_and_bad_manifest(oracle, tmp_path):
    d = _copy("hand_mixed", tmp_path)
    f = d / "rank_0003" / "file_1.bin"
    data = bytearray(f.read_bytes())
    entries = oracle.read_footer(str(f))
    oid, kind, foff, ln, base, ck = next(e for e in entries if e[1] == 0)
    data[foff] ^= 0xFF
    f.write_bytes(bytes(data))
    with pytest.raises(oracle.FormatError) as ei:
        oracle.restore_checkpoint(str(d / "MANIFEST.tlv"))
    assert ei.value.kind == "corrupt_object" and ei.value.object_id == oid
    data[foff] ^= 0xFF
    f.write_bytes(bytes(data[:-3]))
    with pytest.raises(oracle.FormatError) as ei:
        oracle.restore_checkpoint(str(d / "MANIFEST.tlv"))
    assert ei.value.kind == "incomplete_file"
    m = (d / "MANIFEST.tlv").read_bytes()
    (d / "MANIFEST.tlv").write_bytes(m[:-1])
    with pytest.raises(oracle.FormatError) as ei:
        oracle.read_manifest(str(d / "MANIFEST.tlv"))
    assert ei.value.kind == "bad_manifest"


@pytest.mark.parametrize("name", golden_recipes())
def test_rank_digest_verifies_reference_tree(oracle, name):
    """The file-free digest (oracle/tso.py rank_digest, used for cfg4) describes
    every reference-written golden tree exactly, and the full-size structural
    verifier (tests/gpu_helpers.py) accepts those trees."""
    from gpu_helpers import verify_files_against_digest

    rec = oracle.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    files, infos = {}, []
    for r in rec.ranks:
        f, info = oracle.rank_digest(r, rec.pit, threads=2)
        files.update(f)
        infos.append(info)
    m = oracle.tlv_encode(oracle.manifest_value(rec.ckpt_id, rec.iteration, rec.manifest_echo(), infos))
    import hashlib

    files["MANIFEST.tlv"] = {"size": len(m), "sha256": hashlib.sha256(m).hexdigest()}
    root = os.path.join(GOLDEN, "trees", name)
    tree = read_tree(root)
    assert sorted(tree) == sorted(files)
    assert verify_files_against_digest(oracle, root, files, threads=2) == sum(
        len(v) for k, v in tree.items() if k != "MANIFEST.tlv")


def test_rank_digest_verifier_catches_one_flipped_byte(oracle, tmp_path):
    from gpu_helpers import verify_files_against_digest

    rec = oracle.load_recipe(os.path.join(GOLDEN, "recipes", "hand_mixed.recipe"))
    root = str(tmp_path / "t")
    shutil.copytree(os.path.join(GOLDEN, "trees", "hand_mixed"), root)
    files, _ = oracle.rank_digest(rec.ranks[0], rec.pit, threads=2)
    verify_files_against_digest(oracle, root, files, threads=2)
    for rel, d in files.items():  # one byte in an object, in a gap, in the header
        raws = [e for e in d["footer"] if e[1] == 0]
        gap = next((e[2] + e[3] for e in raws if (e[2] + e[3]) % 4096 and e[2] + e[3] < d["tensor_region_end"]),
                   None)
        for pos in [p for p in (raws[0][2] + raws[0][3] // 2 if raws else None, gap, 100) if p is not None]:
            p = os.path.join(root, rel)
            with open(p, "r+b") as f:
                f.seek(pos)
                b = f.read(1)
                f.seek(pos)
                f.write(bytes([b[0] ^ 1]))
            with pytest.raises(AssertionError):
                verify_files_against_digest(oracle, root, files, threads=2)
            with open(p, "r+b") as f:
                f.seek(pos)
                f.write(b)


def test_cfg1_rank_digest_matches_reference_digest(oracle):
    """rank_digest reproduces the reference-written full-size cfg1 digest (the
    same restatement made the cfg4 digest; make_oracle_digests.py re-pins it on
    every reference digest)."""
    with open(os.path.join(GOLDEN, "digests", "cfg1.json")) as f:
        ref = json.load(f)
    rec = oracle.load_recipe(os.path.join(GOLDEN, "recipes", "cfg1.recipe"))
    files, _ = oracle.rank_digest(rec.ranks[0], rec.pit)
    for rel, d in files.items():
        assert d["size"] == ref["files"][rel]["size"]
        assert d["footer"] == ref["files"][rel]["footer"]


def test_cfg4_digest_is_the_oracles(oracle):
    """The committed cfg4 digest's plan side (sizes, footer offsets, headers)
    equals what the oracle derives from the cfg4 recipe (checksums are covered by
    make_oracle_digests.py: 120 GB of hashing is too slow for the CPU suite)."""
    with open(os.path.join(GOLDEN, "digests", "cfg4_rank0.json")) as f:
        dig = json.load(f)
    rec = oracle.load_recipe(os.path.join(GOLDEN, "recipes", "cfg4_rank0.recipe"))
    r = rec.ranks[0]
    plan = oracle.plan_layout(r.objects)
    assert len([o for o in r.objects if o.kind == 0]) == 2892 and len(r.objects) == 3616
    for fid, fp in plan.items():
        d = dig["files"][f"rank_0000/file_{fid}.bin"]
        assert d["tensor_region_end"] == fp.tensor_region_end
        assert [(e[0], e[2], e[3]) for e in d["footer"] if e[1] == 0] == sorted(fp.fixed, key=lambda x: x[1])
        assert d["header"][24:40] == oracle.plan_hash(plan).to_bytes(8, "little").hex()
