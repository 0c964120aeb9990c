// Exact FNV-1a-64 (common.hpp:44-51) of many device byte ranges, segment-parallel.
//
// FNV-1a is a serial byte chain h <- (h ^ b) * P mod 2^64, P = 2^40 + 0x1b3.
// Split h = H * 256 + l (l = low byte). With x = l ^ b:
//     l' = (x * 0xb3) mod 256                      (an 8-bit automaton)
//     H' = H * P + (x << 32) + (x * 0x1b3 >> 8)    (mod 2^56, AFFINE in H)
// so once the low-byte trajectory is known, a segment of k bytes maps
// H -> P^k * H + C_seg, and segments combine with a cheap serial pass.
// The low byte is a T-function: its low nibble evolves on its own,
// lo' = ((lo ^ b) * 3) mod 16, and the high nibble depends only on itself and
// the known low-nibble trajectory. Hence three data passes per segment:
//   A: 16-way speculation of the start low nibble  -> nibble map piA (64 bits)
//      (serial scan over segments fixes each segment's start low nibble)
//   B: 16-way speculation of the start high nibble -> nibble map piB
//      (serial scan fixes the start byte of every segment)
//   C: Horner accumulation of C_seg with the known byte trajectory
// and a final per-object combine. ~40 integer ops/byte, all lanes busy: the
// checksum leaves the host cores free and costs a few ms of GPU per GB.
#include <cstdio>

#include "kernels.cuh"

namespace tsb::dev {

namespace {

constexpr uint64_t kP = 1099511628211ull;
constexpr uint64_t kM56 = (1ull << 56) - 1;

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t fnv_obj_of(const fnv_obj* __restrict__ o, uint32_t n, uint64_t g) {
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(&o[mid].seg0) <= g) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Visits the bytes of [p, p+n) in order with 16-B vector loads where aligned.
template <class F>
__device__ __forceinline__ void for_bytes(const uint8_t* p, uint64_t n, F&& f) {
  uint64_t i = 0;
  const uint64_t head = umin64(n, (16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15);
  for (; i < head; ++i) f(static_cast<uint32_t>(__ldg(p + i)));
  const uint4* v = reinterpret_cast<const uint4*>(p + i);
  const uint64_t nv = (n - i) >> 4;
  for (uint64_t k = 0; k < nv; ++k) {
    const uint4 w = __ldg(v + k);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t u = ws[q];
      f(u & 0xff);
      f((u >> 8) & 0xff);
      f((u >> 16) & 0xff);
      f(u >> 24);
    }
  }
  for (i += nv * 16; i < n; ++i) f(static_cast<uint32_t>(__ldg(p + i)));
}

struct seg_ref {
  const uint8_t* p;
  uint64_t len;
};

__device__ __forceinline__ seg_ref seg_of(const fnv_obj* o, uint32_t n, uint64_t g, uint32_t* obj) {
  const uint32_t i = fnv_obj_of(o, n, g);
  *obj = i;
  const uint64_t off = (g - o[i].seg0) * kFnvSeg;
  return {o[i].ptr + off, umin64(kFnvSeg, o[i].len - off)};
}

// Pass A: end low nibble for each of the 16 possible start low nibbles.
__global__ void __launch_bounds__(256) fnv_pass_a(const fnv_obj* __restrict__ o, uint32_t n, uint64_t nseg,
                                                  uint64_t* __restrict__ piA) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= nseg) return;
  uint32_t obj;
  const seg_ref s = seg_of(o, n, g, &obj);
  uint32_t v0 = 0x03020100u, v1 = 0x07060504u, v2 = 0x0b0a0908u, v3 = 0x0f0e0d0cu;
  for_bytes(s.p, s.len, [&](uint32_t b) {
    const uint32_t bb = (b & 15u) * 0x01010101u;
    v0 = ((v0 ^ bb) * 3u) & 0x0f0f0f0fu;
    v1 = ((v1 ^ bb) * 3u) & 0x0f0f0f0fu;
    v2 = ((v2 ^ bb) * 3u) & 0x0f0f0f0fu;
    v3 = ((v3 ^ bb) * 3u) & 0x0f0f0f0fu;
  });
  const uint32_t v[4] = {v0, v1, v2, v3};
  uint64_t m = 0;
#pragma unroll
  for (int s4 = 0; s4 < 16; ++s4) m |= static_cast<uint64_t>((v[s4 >> 2] >> (8 * (s4 & 3))) & 15u) << (4 * s4);
  piA[g] = m;
}

// Pass B: with the start low nibble fixed, end high nibble for the 16 start high nibbles.
__global__ void __launch_bounds__(256) fnv_pass_b(const fnv_obj* __restrict__ o, uint32_t n, uint64_t nseg,
                                                  const uint8_t* __restrict__ lo_start,
                                                  uint64_t* __restrict__ piB) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= nseg) return;
  uint32_t obj;
  const seg_ref s = seg_of(o, n, g, &obj);
  const uint32_t lo = lo_start[g];
  uint32_t w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) w[j] = (((2u * j) << 4) | lo) | ((((2u * j + 1) << 4) | lo) << 16);
  for_bytes(s.p, s.len, [&](uint32_t b) {
    const uint32_t bb = b * 0x00010001u;
#pragma unroll
    for (int j = 0; j < 8; ++j) w[j] = ((w[j] ^ bb) * 0xb3u) & 0x00ff00ffu;
  });
  uint64_t m = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    m |= static_cast<uint64_t>((w[j] >> 4) & 15u) << (4 * (2 * j));
    m |= static_cast<uint64_t>((w[j] >> 20) & 15u) << (4 * (2 * j + 1));
  }
  piB[g] = m;
}

// Pass C: Horner sum C_seg = sum_i P^(k-1-i) D(x_i) with the known byte trajectory.
__global__ void __launch_bounds__(256) fnv_pass_c(const fnv_obj* __restrict__ o, uint32_t n, uint64_t nseg,
                                                  const uint8_t* __restrict__ l_start,
                                                  uint64_t* __restrict__ cseg) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= nseg) return;
  uint32_t obj;
  const seg_ref s = seg_of(o, n, g, &obj);
  uint32_t l = l_start[g];
  uint64_t c = 0;
  for_bytes(s.p, s.len, [&](uint32_t b) {
    const uint32_t x = l ^ b;
    l = (x * 0xb3u) & 0xffu;
    c = c * kP + ((static_cast<uint64_t>(x) << 32) | ((x * 0x1b3u) >> 8));
  });
  cseg[g] = c & kM56;
}

// Serial scans over each object's segments (one thread per object).
__global__ void fnv_scan_a(const fnv_obj* __restrict__ o, uint32_t n, const uint64_t* __restrict__ states,
                           const uint64_t* __restrict__ piA, uint8_t* __restrict__ lo_start,
                           uint8_t* __restrict__ lo_end) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t g0 = o[i].seg0, g1 = g0 + (o[i].len + kFnvSeg - 1) / kFnvSeg;
  uint32_t lo = static_cast<uint32_t>(states[i] & 15);
  for (uint64_t g = g0; g < g1; ++g) {
    lo_start[g] = static_cast<uint8_t>(lo);
    lo = static_cast<uint32_t>(piA[g] >> (4 * lo)) & 15u;
  }
  lo_end[i] = static_cast<uint8_t>(lo);
}

__global__ void fnv_scan_b(const fnv_obj* __restrict__ o, uint32_t n, const uint64_t* __restrict__ states,
                           const uint64_t* __restrict__ piB, uint8_t* __restrict__ start,
                           uint8_t* __restrict__ lend) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t g0 = o[i].seg0, g1 = g0 + (o[i].len + kFnvSeg - 1) / kFnvSeg;
  uint32_t hi = static_cast<uint32_t>(states[i] >> 4) & 15u;
  for (uint64_t g = g0; g < g1; ++g) {
    const uint32_t lo = start[g];  // holds lo_start on entry
    start[g] = static_cast<uint8_t>((hi << 4) | lo);
    hi = static_cast<uint32_t>(piB[g] >> (4 * hi)) & 15u;
  }
  lend[i] = static_cast<uint8_t>((hi << 4) | lend[i]);
}

__device__ __forceinline__ uint64_t pow_p(uint64_t k) {
  uint64_t r = 1, b = kP;
  while (k) {
    if (k & 1) r *= b;
    b *= b;
    k >>= 1;
  }
  return r;
}

__global__ void fnv_combine(const fnv_obj* __restrict__ o, uint32_t n, uint64_t* __restrict__ states,
                            const uint64_t* __restrict__ cseg, const uint8_t* __restrict__ lend) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (o[i].len == 0) return;
  const uint64_t nseg = (o[i].len + kFnvSeg - 1) / kFnvSeg;
  const uint64_t pk = pow_p(kFnvSeg);
  uint64_t H = states[i] >> 8;
  for (uint64_t s = 0; s < nseg; ++s) {
    const uint64_t len = umin64(kFnvSeg, o[i].len - s * kFnvSeg);
    const uint64_t m = len == kFnvSeg ? pk : pow_p(len);
    H = (m * H + cseg[o[i].seg0 + s]) & kM56;
  }
  states[i] = (H << 8) | lend[i];
}

}  // namespace

uint64_t fnv_scratch_bytes(uint64_t nseg, uint32_t nobj) {
  return align_up_dev(nseg * 8, 256) * 2 + align_up_dev(nseg, 256) + align_up_dev(nobj, 256);
}

void launch_fnv(const fnv_obj* d_objs, uint32_t nobj, uint64_t nseg, uint64_t* d_states, void* d_scratch,
                cudaStream_t st) {
  if (nobj == 0) return;
  uint8_t* s = static_cast<uint8_t*>(d_scratch);
  uint64_t* a = reinterpret_cast<uint64_t*>(s);  // piA, reused for C
  uint64_t* b = reinterpret_cast<uint64_t*>(s + align_up_dev(nseg * 8, 256));
  uint8_t* lst = s + 2 * align_up_dev(nseg * 8, 256);
  uint8_t* lend = lst + align_up_dev(nseg, 256);
  const int T = 256;
  const unsigned gs = static_cast<unsigned>((nseg + T - 1) / T), go = (nobj + T - 1) / T;
  if (nseg) {
    fnv_pass_a<<<gs, T, 0, st>>>(d_objs, nobj, nseg, a);
    count_launch();
  }
  fnv_scan_a<<<go, T, 0, st>>>(d_objs, nobj, d_states, a, lst, lend);
  count_launch();
  if (nseg) {
    fnv_pass_b<<<gs, T, 0, st>>>(d_objs, nobj, nseg, lst, b);
    count_launch();
  }
  fnv_scan_b<<<go, T, 0, st>>>(d_objs, nobj, d_states, b, lst, lend);
  count_launch();
  if (nseg) {
    fnv_pass_c<<<gs, T, 0, st>>>(d_objs, nobj, nseg, lst, a);
    count_launch();
  }
  fnv_combine<<<go, T, 0, st>>>(d_objs, nobj, d_states, a, lend);
  count_launch();
}

}  // namespace tsb::dev
