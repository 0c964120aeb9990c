"""Value.from_py's Python-side TLV encoder (one native decode per value) must
produce exactly the bytes of the element-by-element native builder, and fall
back to it for anything outside the plain types (tlv.cpp:39-77)."""
import math
import random

import pytest

from paper_2601_16956_b200 import api


def slow(v):
    return api.Value(api._build(v)).encode()


def rand_value(rng, depth=0):
    k = rng.randrange(8 if depth < 4 else 5)
    if k == 0:
        return None
    if k == 1:
        return rng.choice([0, 1, -1, 2**63 - 1, -2**63, 2**64 - 1, 2**63, rng.randrange(-2**63, 2**63)])
    if k == 2:
        return rng.choice([0.0, -0.0, 1.5, math.inf, -math.inf, rng.random() * 1e300])
    if k == 3:
        return "".join(rng.choice(["a", "é", "中", "😀", "\x00", "key"]) for _ in range(rng.randrange(6)))
    if k == 4:
        return bytes(rng.randrange(256) for _ in range(rng.randrange(10)))
    if k == 5:
        return [rand_value(rng, depth + 1) for _ in range(rng.randrange(4))]
    if k == 6:
        return tuple(rand_value(rng, depth + 1) for _ in range(rng.randrange(3)))
    return {rng.choice(["b", "a", "é", "zz", "A", "", "中"]) + str(rng.randrange(3)): rand_value(rng, depth + 1)
            for _ in range(rng.randrange(5))}


@pytest.mark.parametrize("seed", range(200))
def test_fast_encoder_matches_native_builder(seed, native):
    v = rand_value(random.Random(seed))
    assert api.Value.from_py(v).encode() == slow(v)


def test_fallbacks(native):
    # surrogates, non-string keys colliding after str(), huge ints: native path semantics
    for v in [{"k": "\ud800"}, {1: 1, "1": 2}, {"a": [1, {"b": None}]}, [b"x", bytearray(b"y")]]:
        assert api.Value.from_py(v).encode() == slow(v)
    with pytest.raises(api.TlvError):
        api.Value.from_py(True)
    deep = []
    cur = deep
    for _ in range(300):
        nxt = []
        cur.append(nxt)
        cur = nxt
    try:
        fast = api.Value.from_py(deep).encode()
    except api.TsError:
        fast = None
    try:
        ref = slow(deep)
    except api.TsError:
        ref = None
    assert fast == ref


def test_kat_map(native):
    # {iteration: 7, rng_seed: 42} (62 B)
    exp = bytes.fromhex("060200000000000000" "030900000000000000" + b"iteration".hex() + "010700000000000000"
                        "030800000000000000" + b"rng_seed".hex() + "012a00000000000000")
    assert api.Value.from_py({"rng_seed": 42, "iteration": 7}).encode() == exp
