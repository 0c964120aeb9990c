"""sm_100a kernels against the oracle: pattern fill/verify, gather-pack (device
and zero-copy host destinations), scatter-unpack. Integer/byte work: bit-exact."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _descs(native, items):
    arr = (native.PatternDesc * len(items))()
    for i, (ptr, size, space, off) in enumerate(items):
        arr[i].data, arr[i].size, arr[i].space, arr[i].offset = ptr, size, space, off
    return arr


def test_pattern_fill_matches_oracle(gpu, native, oracle):
    rng = np.random.default_rng(3)
    buf = torch.zeros(1 << 22, dtype=torch.uint8, device=gpu)
    items, pos = [], 1
    for k in range(60):
        size = int(rng.choice([1, 2, 7, 15, 16, 17, 4095, 65536 + 3, int(rng.integers(1, 50000))]))
        off = int(rng.integers(0, 1 << 40))
        space = int(rng.integers(0, 1 << 62))
        items.append((buf.data_ptr() + pos, size, space, off))
        pos += size + int(rng.integers(0, 40))
    arr = _descs(native, items)
    native.call(native.lib.ts_pattern_fill, arr, len(items), 42, 9, None)
    torch.cuda.synchronize()
    host = buf.cpu().numpy()
    base = buf.data_ptr()
    for ptr, size, space, off in items:
        got = host[ptr - base: ptr - base + size]
        assert (got == oracle.fill_pattern(size, 42, space, 9, off)).all()
    mism = C.c_uint64()
    native.call(native.lib.ts_pattern_verify, arr, len(items), 42, 9, None, C.byref(mism))
    assert mism.value == 0
    buf[items[5][0] - base] ^= 0xFF
    buf[items[30][0] - base + items[30][1] - 1] ^= 0x01
    native.call(native.lib.ts_pattern_verify, arr, len(items), 42, 9, None, C.byref(mism))
    assert mism.value == 2
    native.call(native.lib.ts_pattern_verify, arr, len(items), 42, 10, None, C.byref(mism))
    assert mism.value > 0.9 * sum(i[1] for i in items)


def _fragments(gpu, rng, n, max_size):
    src = torch.randint(0, 256, (n * max_size + 4096,), dtype=torch.uint8, device=gpu)
    frags, pos = [], 0
    for _ in range(n):
        size = int(rng.choice([1, 3, 16, 31, 4096, int(rng.integers(1, max_size))]))
        pos += int(rng.integers(0, 33))
        frags.append((pos, size))
        pos += size
    return src, frags


@pytest.mark.parametrize("dst_kind", ["device", "host"])
def test_pack_matches_numpy(gpu, native, dst_kind):
    rng = np.random.default_rng(11 if dst_kind == "device" else 12)
    src, frags = _fragments(gpu, rng, 300, 70_000)
    n = len(frags)
    offs, cur = [], 0
    for _, size in frags:
        cur = (cur + 4095) // 4096 * 4096 if rng.random() < 0.7 else cur + int(rng.integers(0, 5))
        offs.append(cur)
        cur += size
    dst_len = cur + 123
    if dst_kind == "device":
        dst = torch.full((dst_len,), 0xAB, dtype=torch.uint8, device=gpu)
    else:
        dst = torch.full((dst_len,), 0xAB, dtype=torch.uint8).pin_memory()
    srcs = (C.c_void_p * n)(*[src.data_ptr() + p for p, _ in frags])
    sizes = (C.c_uint64 * n)(*[s for _, s in frags])
    doffs = (C.c_uint64 * n)(*offs)
    native.call(native.lib.ts_pack, srcs, sizes, doffs, n, dst.data_ptr(), dst_len, 0, 0, None)
    torch.cuda.synchronize()
    s = src.cpu().numpy()
    exp = np.zeros(dst_len, dtype=np.uint8)
    for (p, size), o in zip(frags, offs):
        exp[o:o + size] = s[p:p + size]
    got = dst.cpu().numpy()
    assert (got == exp).all()


def test_unpack_roundtrip(gpu, native):
    rng = np.random.default_rng(5)
    img_len = 3 << 20
    img = torch.randint(0, 256, (img_len,), dtype=torch.uint8, device=gpu)
    out = torch.zeros(img_len + (1 << 14), dtype=torch.uint8, device=gpu)
    pieces, pos, dpos = [], 0, 1
    while pos < img_len - 100_000:
        size = int(rng.integers(1, 90_000))
        pos += int(rng.integers(0, 4000))
        dpos += int(rng.integers(0, 7))
        pieces.append((pos, size, dpos))
        pos += size
        dpos += size
    n = len(pieces)
    so = (C.c_uint64 * n)(*[p for p, _, _ in pieces])
    dsts = (C.c_void_p * n)(*[out.data_ptr() + d for _, _, d in pieces])
    sizes = (C.c_uint64 * n)(*[s for _, s, _ in pieces])
    native.call(native.lib.ts_unpack, img.data_ptr(), so, dsts, sizes, n, 0, 0, None)
    torch.cuda.synchronize()
    a, b = img.cpu().numpy(), out.cpu().numpy()
    for p, s, d in pieces:
        assert (b[d:d + s] == a[p:p + s]).all()


def test_kernel_launches_counted(gpu, native):
    before = native.lib.ts_kernel_launch_count()
    buf = torch.zeros(1000, dtype=torch.uint8, device=gpu)
    arr = _descs(native, [(buf.data_ptr(), 1000, 1, 0)])
    native.call(native.lib.ts_pattern_fill, arr, 1, 1, 1, None)
    assert native.lib.ts_kernel_launch_count() == before + 1


def test_fnv_device_matches_oracle(gpu, native, oracle):
    """Segment-parallel FNV-1a kernels == the serial byte chain (common.hpp:44-51)
    for every size class around the 16 KiB segment, misaligned starts, and chaining."""
    from paper_2601_16956_b200 import api

    rng = np.random.default_rng(8)
    buf = torch.randint(0, 256, (12 << 20,), dtype=torch.uint8, device=gpu)
    host = buf.cpu().numpy()
    sizes = [0, 1, 2, 15, 16, 17, 255, 16383, 16384, 16385, 32768, 32769, 100_000, 3 << 20, 5 << 20]
    sizes += [int(x) for x in rng.integers(1, 300_000, 40)]
    views, exp = [], []
    for s in sizes:
        off = int(rng.integers(0, (12 << 20) - s - 1))
        views.append(buf[off:off + s])
        exp.append(oracle.fnv1a64(host[off:off + s]))
    assert api.fnv1a64_device(views) == exp
    # chaining: continue from the state after the first part
    full = buf[7:7 + 1_000_003]
    a, b = full[:400_001], full[400_001:]
    ha = api.fnv1a64_device([a])[0]
    assert api.fnv1a64_device([b], init=[ha]) == [oracle.fnv1a64(host[7:7 + 1_000_003])]
    # all-zero and all-0xff inputs (degenerate low-byte trajectories)
    z = torch.zeros(70_000, dtype=torch.uint8, device=gpu)
    f = torch.full((70_000,), 255, dtype=torch.uint8, device=gpu)
    assert api.fnv1a64_device([z, f]) == [oracle.fnv1a64(np.zeros(70_000, np.uint8)),
                                           oracle.fnv1a64(np.full(70_000, 255, np.uint8))]


def test_fnv_lane_kernel_matches_oracle(gpu, native, oracle):
    """Lane-serial FNV-1a kernel (one lane per object chain, 4-stage register
    pipeline of 64-B blocks) == the serial byte chain: every block-pipeline
    remainder (0-3 blocks, 0-3 vectors, 0-15 bytes), misaligned heads,
    chaining, degenerate inputs, and many lanes of unequal lengths at once."""
    from paper_2601_16956_b200 import api

    rng = np.random.default_rng(11)
    buf = torch.randint(0, 256, (12 << 20,), dtype=torch.uint8, device=gpu)
    host = buf.cpu().numpy()
    sizes = [0, 1, 15, 16, 17, 63, 64, 65, 127, 128, 191, 192, 255, 256, 257, 319, 320, 511, 512, 1023]
    sizes += [64 * k + r for k in range(1, 9) for r in (0, 7, 16, 48, 63)]
    sizes += [100_000, 3 << 20, (5 << 20) + 3]
    sizes += [int(x) for x in rng.integers(1, 300_000, 70)]
    views, exp = [], []
    for s in sizes:
        off = int(rng.integers(0, (12 << 20) - s - 1))
        views.append(buf[off:off + s])
        exp.append(oracle.fnv1a64(host[off:off + s]))
    assert api.fnv1a64_device(views, lanes=True) == exp
    assert api.fnv1a64_device(views[:1], lanes=True) == exp[:1]
    full = buf[5:5 + 1_000_003]
    a, b = full[:400_001], full[400_001:]
    ha = api.fnv1a64_device([a], lanes=True)[0]
    assert api.fnv1a64_device([b], init=[ha], lanes=True) == [oracle.fnv1a64(host[5:5 + 1_000_003])]
    z = torch.zeros(70_000, dtype=torch.uint8, device=gpu)
    f = torch.full((70_000,), 255, dtype=torch.uint8, device=gpu)
    assert api.fnv1a64_device([z, f], lanes=True) == [oracle.fnv1a64(np.zeros(70_000, np.uint8)),
                                                      oracle.fnv1a64(np.full(70_000, 255, np.uint8))]
