// sm_100a kernels of the B200 snapshot engine: gather-pack, scatter-unpack,
// synthetic-state pattern fill / verify. See kernels.cuh for the segment model.
//
// All of them are HBM-bound byte movers (no dense contraction on
// the path), so the design goal is full-width coalesced 128-bit accesses with
// enough bytes in flight per SM: persistent grid, one warp per 32 KiB tile of
// the virtual space, 4 x 16 B loads issued per lane before the stores.
#include <atomic>

#include "kernels.cuh"

namespace tsb::dev {

namespace {

std::atomic<unsigned long long> g_launches{0};

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Bytes [sh, sh+16) of the 32-byte concatenation A|B (little endian), sh in 1..15.
__device__ __forceinline__ uint4 funnel16(uint4 A, uint4 B, uint32_t sh) {
  const uint32_t q = sh >> 2, r = (sh & 3) * 8;
  uint32_t w0, w1, w2, w3, w4;
  switch (q) {
    case 0: w0 = A.x; w1 = A.y; w2 = A.z; w3 = A.w; w4 = B.x; break;
    case 1: w0 = A.y; w1 = A.z; w2 = A.w; w3 = B.x; w4 = B.y; break;
    case 2: w0 = A.z; w1 = A.w; w2 = B.x; w3 = B.y; w4 = B.z; break;
    default: w0 = A.w; w1 = B.x; w2 = B.y; w3 = B.z; w4 = B.w; break;
  }
  uint4 o;
  o.x = __funnelshift_r(w0, w1, r);
  o.y = __funnelshift_r(w1, w2, r);
  o.z = __funnelshift_r(w2, w3, r);
  o.w = __funnelshift_r(w3, w4, r);
  return o;
}

// One warp copies n bytes s -> d (s == nullptr: zero fill). Any alignment:
// stores are always 16-B aligned; a misaligned source is realigned with two
// aligned loads and a funnel shift (every access stays inside the source).
__device__ __forceinline__ void warp_copy(uint8_t* d, const uint8_t* s, uint64_t n, uint32_t lane) {
  uint32_t head = static_cast<uint32_t>((16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15);
  if (head > n) head = static_cast<uint32_t>(n);
  if (lane < head) d[lane] = s ? s[lane] : 0;
  d += head;
  if (s) s += head;
  n -= head;
  const uint64_t nv = n >> 4;
  uint4* dv = reinterpret_cast<uint4*>(d);
  uint64_t i = lane;
  if (s == nullptr) {
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (; i < nv; i += 32) st_stream(dv + i, z);
  } else if ((reinterpret_cast<uintptr_t>(s) & 15) == 0) {
    const uint4* sv = reinterpret_cast<const uint4*>(s);
    for (; i + 96 < nv; i += 128) {
      const uint4 a = ld_stream(sv + i), b = ld_stream(sv + i + 32);
      const uint4 c = ld_stream(sv + i + 64), e = ld_stream(sv + i + 96);
      st_stream(dv + i, a);
      st_stream(dv + i + 32, b);
      st_stream(dv + i + 64, c);
      st_stream(dv + i + 96, e);
    }
    for (; i < nv; i += 32) st_stream(dv + i, ld_stream(sv + i));
  } else {
    const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(s) & 15);
    const uint4* sa = reinterpret_cast<const uint4*>(s - sh);
    // The last output vector's second block sa[nv] holds needed bytes but may
    // extend past the end of the source object (never past its aligned 16-B
    // block, so never across a page): when it would, that vector is assembled
    // from byte loads, keeping every access inside the object.
    const uint64_t rem_src = n & 15;
    const uint64_t nfast = (16 - sh <= rem_src) ? nv : (nv ? nv - 1 : 0);
    for (; i + 32 < nfast; i += 64) {
      const uint4 a0 = ld_stream(sa + i), a1 = ld_stream(sa + i + 1);
      const uint4 b0 = ld_stream(sa + i + 32), b1 = ld_stream(sa + i + 33);
      st_stream(dv + i, funnel16(a0, a1, sh));
      st_stream(dv + i + 32, funnel16(b0, b1, sh));
    }
    for (; i < nfast; i += 32) st_stream(dv + i, funnel16(ld_stream(sa + i), ld_stream(sa + i + 1), sh));
    if (nfast < nv && i == nv - 1) {  // this lane owns the last vector
      const uint8_t* t = s + 16 * (nv - 1);
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        w[q] = static_cast<uint32_t>(t[4 * q]) | (static_cast<uint32_t>(t[4 * q + 1]) << 8) |
               (static_cast<uint32_t>(t[4 * q + 2]) << 16) | (static_cast<uint32_t>(t[4 * q + 3]) << 24);
      st_stream(dv + nv - 1, make_uint4(w[0], w[1], w[2], w[3]));
    }
  }
  const uint32_t rem = static_cast<uint32_t>(n & 15);
  if (lane < rem) d[nv * 16 + lane] = s ? s[nv * 16 + lane] : 0;
}

// Largest k with table[k].pos <= x (table sorted by pos, table[0].pos <= x).
template <class T>
__device__ __forceinline__ uint32_t find_seg(const T* t, uint32_t n, uint64_t x) {
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(&t[mid].pos) <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(512) pack_kernel(const seg* __restrict__ segs, uint32_t nsegs,
                                                   uint64_t lo, uint64_t hi, uint8_t* dst) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t ntiles = (hi - lo + kTileBytes - 1) / kTileBytes;
  for (uint64_t t = warp; t < ntiles; t += nwarps) {
    uint64_t a = lo + t * kTileBytes;
    const uint64_t b = min(a + kTileBytes, hi);
    uint32_t k = find_seg(segs, nsegs, a);
    while (a < b && k < nsegs) {
      const uint64_t pos = __ldg(&segs[k].pos), len = __ldg(&segs[k].len);
      const uint8_t* src = reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(&segs[k].src)));
      const uint64_t e = min(b, pos + len);
      if (e > a && src != TSB_BULK_SRC) warp_copy(dst + (a - lo), src ? src + (a - pos) : nullptr, e - a, lane);
      a = max(a, e);
      ++k;
    }
  }
}

__global__ void __launch_bounds__(512) unpack_kernel(const useg* __restrict__ segs, uint32_t nsegs,
                                                     uint64_t lo, uint64_t hi,
                                                     const uint8_t* __restrict__ src) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t ntiles = (hi - lo + kTileBytes - 1) / kTileBytes;
  for (uint64_t t = warp; t < ntiles; t += nwarps) {
    const uint64_t a = lo + t * kTileBytes;
    const uint64_t b = min(a + kTileBytes, hi);
    uint32_t k = __ldg(&segs[0].pos) <= a ? find_seg(segs, nsegs, a) : 0;
    for (; k < nsegs; ++k) {
      const uint64_t pos = __ldg(&segs[k].pos), len = __ldg(&segs[k].len);
      if (pos >= b) break;
      const uint64_t s0 = max(a, pos), s1 = min(b, pos + len);
      if (s1 > s0) {
        uint8_t* d = reinterpret_cast<uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(&segs[k].dst)));
        warp_copy(d + (s0 - pos), src + (s0 - lo), s1 - s0, lane);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Pattern (pattern.hpp:26-69) on device.

__device__ __forceinline__ uint64_t d_mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}
__device__ __forceinline__ uint64_t d_base(uint64_t seed, uint64_t space, uint64_t it) {
  uint64_t h = d_mix64(seed + 0x9e3779b97f4a7c15ull);
  h = d_mix64(h ^ space);
  h = d_mix64(h ^ it);
  return h | 1;
}
__device__ __forceinline__ uint64_t d_word(uint64_t base, uint64_t block) {
  uint64_t x = base + block * 0x9e3779b97f4a7c15ull;
  x ^= x >> 32;
  x *= 0xd6e8feb86659fd93ull;
  x ^= x >> 32;
  x *= 0xd6e8feb86659fd93ull;
  x ^= x >> 32;
  return x;
}
__device__ __forceinline__ uint8_t d_byte(uint64_t base, uint64_t pos) {
  return static_cast<uint8_t>(d_word(base, pos >> 3) >> (8 * (pos & 7)));
}
// The 16 pattern bytes starting at stream position p.
__device__ __forceinline__ uint4 d_pattern16(uint64_t base, uint64_t p) {
  const uint64_t blk = p >> 3;
  const uint32_t r = static_cast<uint32_t>(p & 7) * 8;
  const uint64_t w0 = d_word(base, blk), w1 = d_word(base, blk + 1);
  uint64_t lo64 = w0, hi64 = w1;
  if (r) {
    const uint64_t w2 = d_word(base, blk + 2);
    lo64 = (w0 >> r) | (w1 << (64 - r));
    hi64 = (w1 >> r) | (w2 << (64 - r));
  }
  return make_uint4(static_cast<uint32_t>(lo64), static_cast<uint32_t>(lo64 >> 32),
                    static_cast<uint32_t>(hi64), static_cast<uint32_t>(hi64 >> 32));
}

template <bool kVerify>
__device__ __forceinline__ uint64_t warp_pattern(uint8_t* d, uint64_t n, uint64_t base, uint64_t p,
                                                 uint32_t lane) {
  uint64_t bad = 0;
  uint32_t head = static_cast<uint32_t>((16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15);
  if (head > n) head = static_cast<uint32_t>(n);
  if (lane < head) {
    const uint8_t v = d_byte(base, p + lane);
    if (kVerify) bad += d[lane] != v;
    else d[lane] = v;
  }
  d += head;
  p += head;
  n -= head;
  const uint64_t nv = n >> 4;
  uint4* dv = reinterpret_cast<uint4*>(d);
  for (uint64_t i = lane; i < nv; i += 32) {
    const uint4 v = d_pattern16(base, p + 16 * i);
    if (kVerify) {
      const uint4 a = ld_stream(dv + i);
      bad += (__popc(__vcmpne4(a.x, v.x)) + __popc(__vcmpne4(a.y, v.y)) +
              __popc(__vcmpne4(a.z, v.z)) + __popc(__vcmpne4(a.w, v.w))) >> 3;
    } else {
      st_stream(dv + i, v);
    }
  }
  const uint32_t rem = static_cast<uint32_t>(n & 15);
  if (lane < rem) {
    const uint8_t v = d_byte(base, p + nv * 16 + lane);
    if (kVerify) bad += d[nv * 16 + lane] != v;
    else d[nv * 16 + lane] = v;
  }
  return bad;
}

template <bool kVerify>
__global__ void __launch_bounds__(512) pattern_kernel(const pseg* __restrict__ segs, uint32_t nsegs,
                                                      uint64_t total, uint64_t seed, uint64_t it,
                                                      unsigned long long* mismatch) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t ntiles = (total + kTileBytes - 1) / kTileBytes;
  uint64_t bad = 0;
  for (uint64_t t = warp; t < ntiles; t += nwarps) {
    uint64_t a = t * kTileBytes;
    const uint64_t b = min(a + kTileBytes, total);
    uint32_t k = find_seg(segs, nsegs, a);
    while (a < b && k < nsegs) {
      const pseg sg = segs[k];
      const uint64_t e = min(b, sg.pos + sg.len);
      if (e > a) {
        const uint64_t base = d_base(seed, sg.space, it);
        bad += warp_pattern<kVerify>(sg.data + (a - sg.pos), e - a, base, sg.offset + (a - sg.pos), lane);
      }
      a = max(a, e);
      ++k;
    }
  }
  if (kVerify) {
    for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if (lane == 0 && bad) atomicAdd(mismatch, static_cast<unsigned long long>(bad));
  }
}


// ---------------------------------------------------------------------------
// Bulk copy through shared memory with the TMA engine (cp.async.bulk).

// Stages of 32 KiB: 6 (192 KiB of shared memory per CTA) for a full-shadow
// pack that owns the GPU; 2 (64 KiB) for ring slots packed while training
// kernels hold most of every SM's shared memory.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int kBulkStages>
__global__ void __launch_bounds__(32) pack_bulk_kernel(const bulk_job* __restrict__ jobs, uint32_t njobs,
                                                       uint64_t lo, uint8_t* dst) {
  extern __shared__ __align__(128) uint8_t stage_buf[];
  __shared__ __align__(8) uint64_t bars[kBulkStages];
  __shared__ uint64_t st_dst[kBulkStages];  // store target / length of each stage, kept from its
  __shared__ uint32_t st_len[kBulkStages];  // issue: no dependent global load on the store path
  if (threadIdx.x != 0) return;
  const uint32_t first = blockIdx.x, step = gridDim.x;
  const uint32_t mine = first < njobs ? (njobs - first + step - 1) / step : 0;
  if (mine == 0) return;
  for (int s = 0; s < kBulkStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // job descriptors are read one issue ahead, so their load latency overlaps
  // the bulk copies instead of sitting on the single issuing thread's path
  bulk_job next = jobs[first];
  auto issue = [&](uint32_t i) {
    const bulk_job jb = next;
    if (i + 1 < mine) next = jobs[first + (i + 1) * step];
    const int s = static_cast<int>(i % kBulkStages);
    const uint32_t bar = smem_u32(&bars[s]);
    const uint32_t len = static_cast<uint32_t>(jb.len);
    st_dst[s] = jb.pos - lo;
    st_len[s] = len;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(len) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(stage_buf + s * kBulkJob)), "l"(jb.src), "r"(len), "r"(bar) : "memory");
  };
  for (uint32_t i = 0; i < mine && i < kBulkStages - 1; ++i) issue(i);
  for (uint32_t i = 0; i < mine; ++i) {
    const int s = static_cast<int>(i % kBulkStages);
    const uint32_t bar = smem_u32(&bars[s]);
    const uint32_t parity = (i / kBulkStages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst + st_dst[s]), "r"(smem_u32(stage_buf + s * kBulkJob)), "r"(st_len[s])
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (i + kBulkStages - 1 < mine) {
      // stage (i-1) % S is reused: the store issued from it one step ago must have read it
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue(i + kBulkStages - 1);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int grid_for(uint64_t bytes, int ctas, int threads) {
  const uint64_t tiles = (bytes + kTileBytes - 1) / kTileBytes;
  const uint64_t warps_per_cta = static_cast<uint64_t>(threads / 32);
  const uint64_t need = (tiles + warps_per_cta - 1) / warps_per_cta;
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(need, static_cast<uint64_t>(ctas))));
}

}  // namespace

int sm_count(int device) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n > 0 ? n : 148;
}

unsigned long long launches() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1); }

void launch_pack(const seg* d_segs, uint32_t nsegs, uint64_t lo, uint64_t hi, uint8_t* dst,
                 int ctas, int threads, cudaStream_t st) {
  if (hi <= lo || nsegs == 0) return;
  pack_kernel<<<grid_for(hi - lo, ctas, threads), threads, 0, st>>>(d_segs, nsegs, lo, hi, dst);
  count_launch();
}

void launch_pack_bulk(const bulk_job* d_jobs, uint32_t njobs, uint64_t lo, uint8_t* dst, int ctas,
                      cudaStream_t st, int stages) {
  if (njobs == 0) return;
  // The dynamic shared memory opt-in is per device (and per instantiation):
  // one process may drive engines (or helper streams) on several GPUs.
  static std::atomic<uint64_t> attr_set[2] = {{0}, {0}};
  const bool few = stages <= 2;
  const int smem = (few ? 2 : 6) * static_cast<int>(kBulkJob);
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set[few].load() & bit)) {
    if (few) cudaFuncSetAttribute(pack_bulk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    else cudaFuncSetAttribute(pack_bulk_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set[few].fetch_or(bit);
  }
  const int grid = static_cast<int>(std::min<uint64_t>(njobs, static_cast<uint64_t>(ctas)));
  if (few) pack_bulk_kernel<2><<<grid, 32, smem, st>>>(d_jobs, njobs, lo, dst);
  else pack_bulk_kernel<6><<<grid, 32, smem, st>>>(d_jobs, njobs, lo, dst);
  count_launch();
}

void launch_unpack(const useg* d_segs, uint32_t nsegs, uint64_t lo, uint64_t hi,
                   const uint8_t* src, int ctas, int threads, cudaStream_t st) {
  if (hi <= lo || nsegs == 0) return;
  unpack_kernel<<<grid_for(hi - lo, ctas, threads), threads, 0, st>>>(d_segs, nsegs, lo, hi, src);
  count_launch();
}

void launch_pattern_fill(const pseg* d_segs, uint32_t nsegs, uint64_t total, uint64_t seed,
                         uint64_t it, int ctas, int threads, cudaStream_t st) {
  if (total == 0 || nsegs == 0) return;
  pattern_kernel<false><<<grid_for(total, ctas, threads), threads, 0, st>>>(d_segs, nsegs, total,
                                                                            seed, it, nullptr);
  count_launch();
}

void launch_pattern_verify(const pseg* d_segs, uint32_t nsegs, uint64_t total, uint64_t seed,
                           uint64_t it, unsigned long long* d_mismatch, int ctas, int threads,
                           cudaStream_t st) {
  if (total == 0 || nsegs == 0) return;
  pattern_kernel<true><<<grid_for(total, ctas, threads), threads, 0, st>>>(d_segs, nsegs, total,
                                                                           seed, it, d_mismatch);
  count_launch();
}

}  // namespace tsb::dev
