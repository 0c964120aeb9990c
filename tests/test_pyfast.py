"""The Python mirror's CPython fast path (csrc/pyfast, api._desc_array) fills the
same ts_object_desc entries and builds the same TLV values as the pure-Python
path, and defers to it (and its errors) for anything unusual. CPU only: CPU
tensors stand in for device payloads (only their addresses are read)."""
import ctypes as C
import random

import pytest
import torch

from paper_2601_16956_b200 import api


def rank_with(values, n_raw=50, seed=0):
    rng = random.Random(seed)
    buf = torch.empty(1 << 16, dtype=torch.uint8)
    rs = api.RankState(3, 1, 0, 2)
    oid = 1
    for _ in range(n_raw):
        sz = rng.randrange(1, 4096)
        off = rng.randrange(0, (1 << 16) - sz)
        rs.objects.append(api.StateObject(oid, api.KIND_RAW, rng.choice([0, 1]), rng.randrange(4), rng.randrange(3),
                                          sz, payload=buf[off:off + sz]))
        oid += 1
    for v in values:
        rs.objects.append(api.StateObject(oid, api.KIND_STRUCTURED, api.TIER_HOST, 2, rng.randrange(3),
                                          structured=v))
        oid += 1
    return rs


VALUES = [None, 0, -1, 2**63 - 1, -2**63, 2**64 - 1, 2**63, 1.5, float("inf"), "", "héllo", b"", b"\x00\xff",
          bytearray(b"ab"), [], [1, [2, [3]]], (4, 5), {}, {"b": 1, "a": [None, 2.5, "x"]}, {1: "int key"},
          {"name": "layers.0.w", "dtype": "bf16", "numel": 123, "shard_offset": 0, "shard_len": 9, "iteration": 7}]


def both(rs, need_payload=True):
    keep_f, keep_s = [], []
    fast = api._desc_array(rs, keep_f, need_payload)
    saved, api._pyfast = api._pyfast, None
    try:
        slow = api._desc_array(rs, keep_s, need_payload)
    finally:
        api._pyfast = saved
    return fast, slow, keep_f, keep_s


@pytest.mark.skipif(api._pyfast is None, reason="fast path not built")
def test_fast_descriptors_equal_python_path():
    rs = rank_with(VALUES + [api.Value.from_py({"pre": "built"})])
    fast, slow, keep, _keep_s = both(rs)
    for i, o in enumerate(rs.objects):
        for f, _ in api.N.ObjectDesc._fields_:
            if f == "value":
                continue
            assert getattr(fast[i], f) == getattr(slow[i], f), (i, f)
        if o.is_raw():
            assert fast[i].data == o.payload.data_ptr() and fast[i].value is None
        else:
            a, b = fast[i].value, slow[i].value
            n = api.N.lib.ts_value_encoded_size(a)
            assert n == api.N.lib.ts_value_encoded_size(b)
            ba, bb = (C.c_uint8 * max(1, n))(), (C.c_uint8 * max(1, n))()
            ln = C.c_size_t()
            api.N.lib.ts_value_encode(a, ba, n, C.byref(ln))
            api.N.lib.ts_value_encode(b, bb, n, C.byref(ln))
            assert bytes(ba) == bytes(bb), (i, o.structured)
    # the caller's pre-built Value is referenced, not copied, and kept alive
    assert fast[len(rs.objects) - 1].value == rs.objects[-1].structured.h
    assert any(k is rs.objects[-1].structured for k in keep)


@pytest.mark.skipif(api._pyfast is None, reason="fast path not built")
@pytest.mark.parametrize("bad", [True, object(), {"k": {1, 2}}, [1, False]])
def test_fast_path_defers_errors_to_python_path(bad):
    rs = rank_with([{"ok": 1}, bad], n_raw=3)
    with pytest.raises(Exception) as fast_err:
        api._desc_array(rs, [])
    saved, api._pyfast = api._pyfast, None
    try:
        with pytest.raises(Exception) as slow_err:
            api._desc_array(rs, [])
    finally:
        api._pyfast = saved
    assert type(fast_err.value) is type(slow_err.value)


@pytest.mark.skipif(api._pyfast is None, reason="fast path not built")
def test_fast_path_missing_payload_raises_like_python():
    rs = rank_with([], n_raw=2)
    rs.objects[1].payload = None
    with pytest.raises(api.TsError, match="payload not materialized"):
        api._desc_array(rs, [])
    fast, slow, _, _ = both(rs, need_payload=False)  # provision_spares: sizes only
    assert fast[1].data is None and fast[1].size_bytes == slow[1].size_bytes


def test_io_uring_probe_exported(native):
    assert native.lib.ts_io_uring_available() in (0, 1)
    assert native.lib.ts_io_uring_ops() >= 0
