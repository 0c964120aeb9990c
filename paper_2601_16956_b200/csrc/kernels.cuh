// Device side of the B200 snapshot engine (sm_100a).
//
// All kernels work on a "segment table": a list of byte ranges laid end to end
// in a virtual space (the per-rank checkpoint image for pack/unpack, the
// concatenated fragments for pattern fill/verify), sorted by virtual offset.
// Work is cut in fixed-size tiles of that virtual space and handed to warps by
// a persistent grid, so thousands of tiny fragments and a few huge ones cost the
// same per byte (no per-fragment launches, no idle lanes on small fragments).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tsb::dev {

// One piece of the image. src == nullptr => zero fill (alignment gaps);
// src == kBulkSrc => bytes written by the bulk-copy (TMA) kernel, skipped here.
#define TSB_BULK_SRC (reinterpret_cast<const uint8_t*>(uintptr_t{1}))
struct seg {
  uint64_t pos;  // virtual (image) offset
  uint64_t len;
  const uint8_t* src;
};

// One destination piece of an unpack (restore): image [pos, pos+len) -> dst.
struct useg {
  uint64_t pos;
  uint64_t len;
  uint8_t* dst;
};

// One fragment of the synthetic state: virtual [pos, pos+len) <-> data,
// whose byte 0 is byte `offset` of pattern space `space`.
struct pseg {
  uint64_t pos;
  uint64_t len;
  uint8_t* data;
  uint64_t space;
  uint64_t offset;
};

constexpr uint32_t kTileBytes = 32768;  // virtual bytes per warp task

// Gather-pack: writes image bytes [lo, hi) into dst (dst[0] = image byte lo).
// dst may be device memory (RING) or mapped pinned host memory (ZEROCOPY).
void launch_pack(const seg* d_segs, uint32_t nsegs, uint64_t lo, uint64_t hi, uint8_t* dst,
                 int ctas, int threads, cudaStream_t st);

// Bulk (TMA engine) copy jobs: dst image position, 16-B aligned source, length
// a multiple of 16 and <= kBulkJob. One elected thread per CTA drives a ring of
// shared-memory stages: cp.async.bulk global->shared completing on an
// mbarrier, then cp.async.bulk shared->global, so SM issue slots stay free.
constexpr uint32_t kBulkJob = 32768;
struct bulk_job {
  uint64_t pos;
  const uint8_t* src;
  uint64_t len;
};
// Copies jobs whose pos lies in [lo, hi) into dst (dst[0] = image byte lo).
void launch_pack_bulk(const bulk_job* d_jobs, uint32_t njobs, uint64_t lo, uint8_t* dst, int ctas,
                      cudaStream_t st, int stages = 6);

// Scatter-unpack: image bytes [lo, hi) held in src (src[0] = image byte lo)
// to the destination pieces that intersect the range.
void launch_unpack(const useg* d_segs, uint32_t nsegs, uint64_t lo, uint64_t hi,
                   const uint8_t* src, int ctas, int threads, cudaStream_t st);

void launch_pattern_fill(const pseg* d_segs, uint32_t nsegs, uint64_t total, uint64_t seed,
                         uint64_t iteration, int ctas, int threads, cudaStream_t st);
void launch_pattern_verify(const pseg* d_segs, uint32_t nsegs, uint64_t total, uint64_t seed,
                           uint64_t iteration, unsigned long long* d_mismatch, int ctas,
                           int threads, cudaStream_t st);

// ---------------------------------------------------------------------------
// Exact segment-parallel FNV-1a-64 (fnv.cu). Each object's state (in/out) is
// chained: pass the seed for a fresh checksum, a previous state to continue.
constexpr uint64_t kFnvSeg = 16384;
struct fnv_obj {
  const uint8_t* ptr;
  uint64_t len;
  uint64_t seg0;    // first global segment index (prefix sum of ceil(len / kFnvSeg))
  uint64_t chunk0;  // first global chunk index (chunks of 64 segments, per object)
  uint64_t sidx;    // index of this range's chain state in d_states / out (pieces of one
                    // object in later launches continue from the same state)
  uint64_t seglen;  // segment length of the launch (set by fnv_prepare, <= kFnvSeg)
};
inline uint64_t align_up_dev(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }
// Fills seg0/chunk0 of a host table; returns the segment count, *nchunk the chunk count.
uint64_t fnv_prepare(fnv_obj* objs, uint32_t n, uint64_t* nchunk);
uint64_t fnv_scratch_bytes(uint64_t nseg, uint64_t nchunk, uint32_t nobj);
// 11 launches on `st`; d_states (in: chain start, out: FNV state) per object;
// results also stored to `out_mapped` (device view of mapped pinned memory) if set.
void launch_fnv(const fnv_obj* d_objs, uint32_t nobj, uint64_t nseg, uint64_t nchunk, uint64_t* d_states,
                void* d_scratch, cudaStream_t st, uint64_t* out_mapped = nullptr);

// Lane-serial FNV-1a-64 (fnv.cu): one lane per object chain, ~7 integer ops per
// byte (the segment-parallel kernels above spend ~26: nibble speculation).
// For objects whose serial chain (~0.2 GB/s per lane) finishes within the time
// budget. Objects should be sorted by length, longest first (lanes of a warp
// then finish together). Writes out[o.out] = FNV state after o's bytes,
// starting from o.init.
struct fnv_lane_obj {
  const uint8_t* ptr;
  uint64_t len;
  uint64_t init;
  uint64_t out;
};
void launch_fnv_lanes(const fnv_lane_obj* d_objs, uint32_t n, uint64_t* out, cudaStream_t st);

int sm_count(int device);
unsigned long long launches();
void count_launch();

}  // namespace tsb::dev
