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
//   A: speculation of the start low nibble  -> nibble map piA (64 bits)
//      (serial scan over segments fixes each segment's start low nibble)
//   B: speculation of the start high nibble -> nibble map piB
//      (serial scan fixes the start byte of every segment)
//   C: Horner accumulation of C_seg with the known byte trajectory
// and a final per-object combine. Both nibble maps satisfy f(s^8) = f(s)^8, so
// 8 candidates (two registers of 8-bit lanes) determine all 16. ~26 integer
// ops/byte, all lanes busy.
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
  const uint64_t sl = o[i].seglen;
  const uint64_t off = (g - o[i].seg0) * sl;
  return {o[i].ptr + off, umin64(sl, o[i].len - off)};
}

// Visits [p, p+n) in order: f1(byte) for an unaligned head / tail, f4(word)
// for each little-endian 32-bit word of the 16-B aligned body.
template <class F1, class F4>
__device__ __forceinline__ void for_words(const uint8_t* p, uint64_t n, F1&& f1, F4&& f4) {
  uint64_t i = 0;
  const uint64_t head = umin64(n, (16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15);
  for (; i < head; ++i) f1(static_cast<uint32_t>(__ldg(p + i)));
  const uint4* v = reinterpret_cast<const uint4*>(p + i);
  const uint64_t nv = (n - i) >> 4;
  for (uint64_t k = 0; k < nv; ++k) {
    const uint4 w = __ldg(v + k);
    f4(w.x);
    f4(w.y);
    f4(w.z);
    f4(w.w);
  }
  for (i += nv * 16; i < n; ++i) f1(static_cast<uint32_t>(__ldg(p + i)));
}

// Both nibble automata satisfy f(s ^ 8) = f(s) ^ 8 (x*3 +- 24 = x*3 + 8 mod
// 16, and the high nibble's carry-in does not depend on its own state), so a
// segment's 16-entry nibble map is fixed by the end states of the starts 0..7:
// map[s + 8] = map[s] ^ 8. Eight candidates = two registers of 8-bit lanes.
__device__ __forceinline__ uint64_t nibble_map8(uint32_t v0, uint32_t v1) {
  uint64_t m = 0;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const uint32_t e = ((s < 4 ? v0 : v1) >> (8 * (s & 3))) & 15u;
    m |= static_cast<uint64_t>(e) << (4 * s);
    m |= static_cast<uint64_t>(e ^ 8u) << (4 * (s + 8));
  }
  return m;
}

// Pass A: end low nibble for each start low nibble (lo' = ((lo ^ b) * 3) mod 16).
__global__ void __launch_bounds__(256) fnv_pass_a(const fnv_obj* __restrict__ o, uint32_t n, uint64_t nseg,
                                                  uint64_t* __restrict__ piA) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= nseg) return;
  uint32_t obj;
  const seg_ref s = seg_of(o, n, g, &obj);
  uint32_t v0 = 0x03020100u, v1 = 0x07060504u;
  auto step = [&](uint32_t bb) {  // bb: the byte's low nibble in every lane
    v0 = ((v0 ^ bb) * 3u) & 0x0f0f0f0fu;
    v1 = ((v1 ^ bb) * 3u) & 0x0f0f0f0fu;
  };
  for_words(
      s.p, s.len, [&](uint32_t b) { step((b & 15u) * 0x01010101u); },
      [&](uint32_t w) {
        const uint32_t lw = w & 0x0f0f0f0fu;
        step(__byte_perm(lw, 0, 0x0000));
        step(__byte_perm(lw, 0, 0x1111));
        step(__byte_perm(lw, 0, 0x2222));
        step(__byte_perm(lw, 0, 0x3333));
      });
  piA[g] = nibble_map8(v0, v1);
}

// Pass B: with the start low nibble fixed, end high nibble for each start high
// nibble. With x = l ^ b = 16*xh + xl and t = xl * 0xb3 (known once the
// low-nibble trajectory is), the byte update splits into
//     lo' = t mod 16,   hi' = (3*xh + (t >> 4)) mod 16.
// Lanes hold 3*(v ^ bh) + (t >> 4) <= 45 + 167 < 256 before the mask, so the
// carry-in needs no mask of its own.
__global__ void __launch_bounds__(256) fnv_pass_b(const fnv_obj* __restrict__ o, uint32_t n, uint64_t nseg,
                                                  const uint8_t* __restrict__ lo_start,
                                                  uint64_t* __restrict__ piB) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= nseg) return;
  uint32_t obj;
  const seg_ref s = seg_of(o, n, g, &obj);
  uint32_t lo = lo_start[g];
  uint32_t v0 = 0x03020100u, v1 = 0x07060504u;
  auto step = [&](uint32_t bl, uint32_t bh) {  // bl: low nibble in bits 0-3; bh: high nibble, every lane
    const uint32_t t = ((lo ^ bl) & 15u) * 0xb3u;
    lo = t & 15u;
    const uint32_t c = (t >> 4) * 0x01010101u;
    v0 = (((v0 ^ bh) * 3u) + c) & 0x0f0f0f0fu;
    v1 = (((v1 ^ bh) * 3u) + c) & 0x0f0f0f0fu;
  };
  for_words(
      s.p, s.len, [&](uint32_t b) { step(b, (b >> 4) * 0x01010101u); },
      [&](uint32_t w) {
        const uint32_t hw = (w >> 4) & 0x0f0f0f0fu;
        step(w, __byte_perm(hw, 0, 0x0000));
        step(w >> 8, __byte_perm(hw, 0, 0x1111));
        step(w >> 16, __byte_perm(hw, 0, 0x2222));
        step(w >> 24, __byte_perm(hw, 0, 0x3333));
      });
  piB[g] = nibble_map8(v0, v1);
}

// Pass C: Horner sum C_seg = sum_i P^(k-1-i) D(x_i) with the known byte
// trajectory, D(x) = (x << 32) + (x * 0x1b3 >> 8). Integer multiplies run on
// the half-rate fmaheavy pipe (ncu: 96 % busy with one 64-bit multiply per
// byte), so bytes go in pairs: C <- C * P^2 + (D0 * P + D1), and since
// D0 * P = (x0*q << 32) + (d0 << 40) + d0*q (mod 2^64, q = 0x1b3, d0 < 2^9)
// the pair term costs two 32-bit multiplies: 7 instead of ~11 per two bytes.
__global__ void __launch_bounds__(256) fnv_pass_c(const fnv_obj* __restrict__ o, uint32_t n, uint64_t nseg,
                                                  const uint8_t* __restrict__ l_start,
                                                  uint64_t* __restrict__ cseg) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= nseg) return;
  uint32_t obj;
  const seg_ref s = seg_of(o, n, g, &obj);
  constexpr uint32_t q = 0x1b3u;
  constexpr uint64_t kP2 = kP * kP;  // P^2 mod 2^64
  uint32_t l = l_start[g];
  uint64_t c = 0;
  auto step1 = [&](uint32_t b) {
    const uint32_t x = (l ^ b) & 0xffu;
    const uint32_t t = x * q;  // low byte: the next l ((x * 0xb3) mod 256); >> 8: D's low word
    l = t & 0xffu;
    c = c * kP + ((static_cast<uint64_t>(x) << 32) | (t >> 8));
  };
  auto step2 = [&](uint32_t b0, uint32_t b1) {
    const uint32_t x0 = (l ^ b0) & 0xffu;
    const uint32_t t0 = x0 * q;
    const uint32_t x1 = (t0 ^ b1) & 0xffu;
    const uint32_t t1 = x1 * q;
    l = t1 & 0xffu;
    const uint32_t d0 = t0 >> 8, d1 = t1 >> 8;
    const uint32_t e_lo = d0 * q + d1;             // < 2^18: no carry into the high word
    const uint32_t e_hi = x0 * q + ((d0 << 8) + x1);
    c = c * kP2 + ((static_cast<uint64_t>(e_hi) << 32) | e_lo);
  };
  for_words(
      s.p, s.len, step1,
      [&](uint32_t w) {
        step2(w, w >> 8);
        step2(w >> 16, w >> 24);
      });
  cseg[g] = c & kM56;
}

// ---------------------------------------------------------------------------
// Lane-serial FNV: one lane walks one object's whole chain, pass C's split
// arithmetic started from the object's known state (l = its low byte, c = the
// upper 56 bits; Horner needs no P^k fix-up then). ~7 integer ops per byte and
// a critical path of two dependent ops per byte (the low-byte automaton), so a
// lane runs ~0.2 GB/s and the whole kernel uses a few warps per SM: a tenth of
// the issue slots the speculating passes take for the same bytes.
//
// A lane's loads are its own contiguous stream, so latency is hidden by the
// lane itself: four 64-B stages in registers, the load of stage k+4 issued as
// soon as stage k is consumed (~1,500 cycles of work ahead of each load).
__device__ __forceinline__ uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

__global__ void __launch_bounds__(32) fnv_lane_kernel(const fnv_lane_obj* __restrict__ o, uint32_t n,
                                                      uint64_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t* p = o[i].ptr;
  const uint64_t len = o[i].len;
  const uint64_t h0 = o[i].init;
  constexpr uint32_t q = 0x1b3u;
  constexpr uint64_t kP2 = kP * kP;
  constexpr uint32_t kP2lo = static_cast<uint32_t>(kP2), kP2hi = static_cast<uint32_t>(kP2 >> 32);
  uint32_t l = static_cast<uint32_t>(h0) & 0xffu;
  // c in two 32-bit halves: c * P^2 + e is one wide multiply-add plus two
  // 32-bit ones (the compiler's 64-bit form spends six instructions)
  uint32_t clo = static_cast<uint32_t>(h0 >> 8), chi = static_cast<uint32_t>(h0 >> 40);
  auto step1 = [&](uint32_t b) {
    const uint32_t x = (l ^ b) & 0xffu;
    const uint32_t t = x * q;
    l = t & 0xffu;
    const uint64_t c = ((static_cast<uint64_t>(chi) << 32) | clo) * kP + ((static_cast<uint64_t>(x) << 32) | (t >> 8));
    clo = static_cast<uint32_t>(c);
    chi = static_cast<uint32_t>(c >> 32);
  };
  auto step2 = [&](uint32_t b0, uint32_t b1) {
    const uint32_t x0 = (l ^ b0) & 0xffu;
    const uint32_t t0 = x0 * q;
    const uint32_t x1 = (t0 ^ b1) & 0xffu;
    const uint32_t t1 = x1 * q;
    l = t1 & 0xffu;
    const uint32_t d0 = t0 >> 8, d1 = t1 >> 8;
    const uint32_t e_lo = d0 * q + d1;
    const uint32_t e_hi = t0 + ((d0 << 8) + x1);
    const uint64_t w = mad_wide(clo, kP2lo, (static_cast<uint64_t>(e_hi) << 32) | e_lo);
    const uint32_t hi = clo * kP2hi + (chi * kP2lo + static_cast<uint32_t>(w >> 32));
    clo = static_cast<uint32_t>(w);
    chi = hi;
  };
  auto word = [&](uint32_t w) {
    step2(w, w >> 8);
    step2(w >> 16, w >> 24);
  };
  auto vec = [&](const uint4& w) {
    word(w.x);
    word(w.y);
    word(w.z);
    word(w.w);
  };
  const uint64_t head = umin64(len, (16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15);
  for (uint64_t k = 0; k < head; ++k) step1(__ldg(p + k));
  const uint4* v = reinterpret_cast<const uint4*>(p + head);
  const uint64_t nv = (len - head) >> 4;
  const uint64_t nb = nv >> 2;  // 64-B blocks
  uint4 s0[4], s1[4], s2[4], s3[4];
  auto load = [&](uint4(&s)[4], uint64_t b) {
    if (b < nb) {
#pragma unroll
      for (int k = 0; k < 4; ++k) s[k] = __ldg(v + 4 * b + k);
    }
  };
  auto proc = [&](const uint4(&s)[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) vec(s[k]);
  };
  load(s0, 0);
  load(s1, 1);
  load(s2, 2);
  load(s3, 3);
  uint64_t b = 0;
  for (; b + 4 <= nb; b += 4) {
    proc(s0);
    load(s0, b + 4);
    proc(s1);
    load(s1, b + 5);
    proc(s2);
    load(s2, b + 6);
    proc(s3);
    load(s3, b + 7);
  }
  if (b < nb) proc(s0);
  if (b + 1 < nb) proc(s1);
  if (b + 2 < nb) proc(s2);
  for (uint64_t k = nb * 4; k < nv; ++k) vec(__ldg(v + k));
  for (uint64_t k = head + nv * 16; k < len; ++k) step1(__ldg(p + k));
  out[o[i].out] = ((((static_cast<uint64_t>(chi) << 32) | clo) & kM56) << 8) | l;
}

// ---------------------------------------------------------------------------
// Scans over each object's segments. The per-segment maps (nibble maps for
// passes A/B, affine maps H -> a*H + c for the combine) compose associatively,
// so each object's chain is cut into chunks of kChunk segments: compose each
// chunk in parallel, run the short serial chain over chunks, then expand the
// chunk starts back to segment starts in parallel.

constexpr uint32_t kChunk = 64;

__device__ __forceinline__ uint32_t nib(uint64_t m, uint32_t i) { return static_cast<uint32_t>(m >> (4 * i)) & 15u; }

// (m after p): x -> m[p[x]]
__device__ __forceinline__ uint64_t nib_compose(uint64_t m, uint64_t p) {
  uint64_t r = 0;
#pragma unroll
  for (uint32_t x = 0; x < 16; ++x) r |= static_cast<uint64_t>(nib(m, nib(p, x))) << (4 * x);
  return r;
}

__device__ __forceinline__ uint64_t obj_nseg(const fnv_obj& o) { return (o.len + o.seglen - 1) / o.seglen; }

// chunk c of the global chunk space -> (object, first segment, segment count)
struct chunk_ref {
  uint32_t obj;
  uint64_t g0, n;
};
__device__ __forceinline__ chunk_ref chunk_of(const fnv_obj* __restrict__ o, uint32_t n, uint64_t c) {
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(&o[mid].chunk0) <= c) lo = mid;
    else hi = mid;
  }
  const uint64_t k = c - o[lo].chunk0;
  const uint64_t ns = obj_nseg(o[lo]);
  const uint64_t g0 = o[lo].seg0 + k * kChunk;
  return {lo, g0, umin64(kChunk, ns - k * kChunk)};
}

__global__ void fnv_chunk_nib(const fnv_obj* __restrict__ o, uint32_t n,
                              uint64_t nchunk, const uint64_t* __restrict__ pi, uint64_t* __restrict__ cpi) {
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nchunk) return;
  const chunk_ref r = chunk_of(o, n, c);
  uint64_t m = 0xfedcba9876543210ull;
  for (uint64_t s = 0; s < r.n; ++s) m = nib_compose(pi[r.g0 + s], m);
  cpi[c] = m;
}

// Serial chain over an object's chunks: start nibble of every chunk.
// `shift` selects the nibble of the state the chain starts from (0: low, 4: high).
__global__ void fnv_chain_nib(const fnv_obj* __restrict__ o, uint32_t n,
                              const uint64_t* __restrict__ states, const uint64_t* __restrict__ cpi,
                              uint8_t* __restrict__ cstart, uint8_t* __restrict__ end_nib, uint32_t shift) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t c0 = o[i].chunk0, c1 = c0 + (obj_nseg(o[i]) + kChunk - 1) / kChunk;
  uint32_t x = static_cast<uint32_t>(states[o[i].sidx] >> shift) & 15u;
  for (uint64_t c = c0; c < c1; ++c) {
    cstart[c] = static_cast<uint8_t>(x);
    x = nib(cpi[c], x);
  }
  end_nib[i] = static_cast<uint8_t>(x);
}

// Expand chunk starts to segment starts. mode 0: out[g] = lo nibble;
// mode 1: out[g] = (hi << 4) | out[g] (out holds the low nibbles on entry).
__global__ void fnv_expand_nib(const fnv_obj* __restrict__ o, uint32_t n,
                               uint64_t nchunk, const uint64_t* __restrict__ pi,
                               const uint8_t* __restrict__ cstart, uint8_t* __restrict__ out, int mode) {
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nchunk) return;
  const chunk_ref r = chunk_of(o, n, c);
  uint32_t x = cstart[c];
  for (uint64_t s = 0; s < r.n; ++s) {
    const uint64_t g = r.g0 + s;
    out[g] = static_cast<uint8_t>(mode == 0 ? x : ((x << 4) | out[g]));
    x = nib(pi[g], x);
  }
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

// Affine composition over a chunk: H -> a*H + c (mod 2^56).
__global__ void fnv_chunk_affine(const fnv_obj* __restrict__ o, uint32_t n,
                                 uint64_t nchunk, const uint64_t* __restrict__ cseg, uint64_t* __restrict__ ca,
                                 uint64_t* __restrict__ cc) {
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nchunk) return;
  const chunk_ref r = chunk_of(o, n, c);
  const fnv_obj& ob0 = o[r.obj];
  const uint64_t pk = pow_p(ob0.seglen);
  uint64_t a = 1, cv = 0;
  const fnv_obj& ob = o[r.obj];
  for (uint64_t s = 0; s < r.n; ++s) {
    const uint64_t g = r.g0 + s;
    const uint64_t len = umin64(ob.seglen, ob.len - (g - ob.seg0) * ob.seglen);
    const uint64_t m = len == ob.seglen ? pk : pow_p(len);
    a = (m * a) & kM56;
    cv = (m * cv + cseg[g]) & kM56;
  }
  ca[c] = a;
  cc[c] = cv;
}

__global__ void fnv_combine(const fnv_obj* __restrict__ o, uint32_t n,
                            uint64_t* __restrict__ states, const uint64_t* __restrict__ ca,
                            const uint64_t* __restrict__ cc, const uint8_t* __restrict__ lo_end,
                            const uint8_t* __restrict__ hi_end, uint64_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (o[i].len == 0) {
    if (out) out[o[i].sidx] = states[o[i].sidx];
    return;
  }
  const uint64_t c0 = o[i].chunk0, c1 = c0 + (obj_nseg(o[i]) + kChunk - 1) / kChunk;
  uint64_t H = states[o[i].sidx] >> 8;
  for (uint64_t c = c0; c < c1; ++c) H = (ca[c] * H + cc[c]) & kM56;
  const uint64_t h = (H << 8) | (static_cast<uint64_t>(hi_end[i]) << 4) | lo_end[i];
  states[o[i].sidx] = h;
  if (out) out[o[i].sidx] = h;  // mapped pinned memory: no copy-engine round trip behind bulk D2H
}

}  // namespace

uint64_t fnv_scratch_bytes(uint64_t nseg, uint64_t nchunk, uint32_t nobj) {
  return align_up_dev(nseg * 8, 256) * 2 + align_up_dev(nseg, 256) + align_up_dev(nchunk * 8, 256) * 3 +
         align_up_dev(nchunk, 256) + align_up_dev(nobj, 256) * 2;
}

uint64_t fnv_prepare(fnv_obj* objs, uint32_t n, uint64_t* nchunk) {
  // Segment length: 16 KiB, shrunk (to >= 1 KiB) until the launch has about two
  // waves of threads, so many small fragments still fill the GPU.
  uint64_t total = 0;
  for (uint32_t i = 0; i < n; ++i) total += objs[i].len;
  uint64_t seglen = kFnvSeg;
  while (seglen > 1024 && total / seglen < 600000) seglen >>= 1;
  uint64_t g = 0, c = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint64_t ns = (objs[i].len + seglen - 1) / seglen;
    objs[i].seg0 = g;
    objs[i].chunk0 = c;
    objs[i].seglen = seglen;
    g += ns;
    c += (ns + kChunk - 1) / kChunk;
  }
  *nchunk = c;
  return g;
}

void launch_fnv(const fnv_obj* d_objs, uint32_t nobj, uint64_t nseg, uint64_t nchunk, uint64_t* d_states,
                void* d_scratch, cudaStream_t st, uint64_t* out_mapped) {
  if (nobj == 0) return;
  uint8_t* s = static_cast<uint8_t*>(d_scratch);
  auto take = [&](uint64_t bytes) {
    uint8_t* p = s;
    s += align_up_dev(bytes, 256);
    return p;
  };
  uint64_t* pa = reinterpret_cast<uint64_t*>(take(nseg * 8));  // piA, later C_seg
  uint64_t* pb = reinterpret_cast<uint64_t*>(take(nseg * 8));  // piB
  uint8_t* lst = take(nseg);                                   // segment start nibble, then byte
  uint64_t* cpi = reinterpret_cast<uint64_t*>(take(nchunk * 8));
  uint64_t* ca = reinterpret_cast<uint64_t*>(take(nchunk * 8));
  uint64_t* cc = reinterpret_cast<uint64_t*>(take(nchunk * 8));
  uint8_t* cst = take(nchunk);
  uint8_t* lo_end = take(nobj);
  uint8_t* hi_end = take(nobj);
  const int T = 256;
  const unsigned gs = static_cast<unsigned>((nseg + T - 1) / T), go = (nobj + T - 1) / T;
  const unsigned gc = static_cast<unsigned>((nchunk + T - 1) / T);
  auto L = [] { count_launch(); };
  if (nseg) {
    fnv_pass_a<<<gs, T, 0, st>>>(d_objs, nobj, nseg, pa); L();
    fnv_chunk_nib<<<gc, T, 0, st>>>(d_objs, nobj, nchunk, pa, cpi); L();
  }
  fnv_chain_nib<<<go, T, 0, st>>>(d_objs, nobj, d_states, cpi, cst, lo_end, 0); L();
  if (nseg) {
    fnv_expand_nib<<<gc, T, 0, st>>>(d_objs, nobj, nchunk, pa, cst, lst, 0); L();
    fnv_pass_b<<<gs, T, 0, st>>>(d_objs, nobj, nseg, lst, pb); L();
    fnv_chunk_nib<<<gc, T, 0, st>>>(d_objs, nobj, nchunk, pb, cpi); L();
  }
  fnv_chain_nib<<<go, T, 0, st>>>(d_objs, nobj, d_states, cpi, cst, hi_end, 4); L();
  if (nseg) {
    fnv_expand_nib<<<gc, T, 0, st>>>(d_objs, nobj, nchunk, pb, cst, lst, 1); L();
    fnv_pass_c<<<gs, T, 0, st>>>(d_objs, nobj, nseg, lst, pa); L();
    fnv_chunk_affine<<<gc, T, 0, st>>>(d_objs, nobj, nchunk, pa, ca, cc); L();
  }
  fnv_combine<<<go, T, 0, st>>>(d_objs, nobj, d_states, ca, cc, lo_end, hi_end, out_mapped); L();
}

void launch_fnv_lanes(const fnv_lane_obj* d_objs, uint32_t n, uint64_t* out, cudaStream_t st) {
  if (n == 0) return;
  // one warp per block: the block scheduler spreads the few warps over SMs
  fnv_lane_kernel<<<(n + 31) / 32, 32, 0, st>>>(d_objs, n, out);
  count_launch();
}

}  // namespace tsb::dev
