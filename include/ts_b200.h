/*
 * ts_b200.h — C-ABI of the B200-native snapshot engine (libts_b200.so).
 *
 * Drop-in boundary for the reference's State Provider / checkpoint-engine API
 * ("tierstream", /root/reference/proj; paths below are relative to it). Plain
 * pointers and sizes only; CUDA streams are passed as `void*` (cudaStream_t).
 * Every entry point names the reference interface it replaces.
 *
 * Error model: every call returns ts_status. Reference exception kinds map 1:1
 * (ts_error / stream_error / cache_timeout_error / ticket_error / format_error
 * kinds / tlv_error, common.hpp:21-24, provider.hpp:135-140, staging.hpp:18-21,
 * transfer.hpp:41-44, format.hpp:50-67, tlv.hpp:70-73). The message of the last
 * failure on the calling thread is ts_last_error(), its object id (when the
 * reference would carry one) ts_last_error_object() (-1 when none).
 * Failures inside engine threads are deferred to the next wait on the ticket,
 * as in the reference (transfer.cpp:105-128).
 */
#ifndef TS_B200_H
#define TS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 1

typedef enum ts_status {
  TS_OK = 0,
  TS_ERR_GENERIC = 1,        /* ts_error                         common.hpp:21 */
  TS_ERR_STREAM = 2,         /* stream_error{object_id}          provider.hpp:135 */
  TS_ERR_CACHE_TIMEOUT = 3,  /* cache_timeout_error              staging.hpp:18 */
  TS_ERR_TICKET = 4,         /* ticket_error                     transfer.hpp:41 */
  TS_ERR_TLV = 5,            /* tlv::tlv_error                   tlv.hpp:70 */
  /* format_error kinds, format.hpp:50-58, in declaration order */
  TS_ERR_MISSING_FILE = 10,
  TS_ERR_INCOMPLETE_FILE = 11,
  TS_ERR_CORRUPT_OBJECT = 12,
  TS_ERR_CORRUPT_FOOTER = 13,
  TS_ERR_BAD_MANIFEST = 14,
  TS_ERR_INVALID_ENTRIES = 15,
  TS_ERR_IO = 16,
  /* B200 side */
  TS_ERR_CUDA = 30,          /* CUDA runtime failure / no device: the product never falls back to CPU */
  TS_ERR_INVALID_ARG = 31
} ts_status;

const char* ts_last_error(void);
int64_t ts_last_error_object(void);
int ts_abi_version(void);

/* ------------------------------------------------------------------------ */
/* Enumerations (model.hpp:19-25, engine.hpp:30)                             */

enum { TS_TIER_DEVICE = 0, TS_TIER_HOST = 1, TS_TIER_PERSISTENT = 2 };
enum { TS_KIND_RAW = 0, TS_KIND_STRUCTURED = 1 };
enum { TS_PREC_FP16 = 0, TS_PREC_FP32 = 1, TS_PREC_OPAQUE = 2 };
enum { TS_STRATEGY_SYNC = 0, TS_STRATEGY_TWO_PHASE = 1, TS_STRATEGY_LAZY = 2 };

/* How device bytes reach the pinned host pool (B200 design choice):
 *  RING     gather-pack kernel into a bounded HBM staging ring, copy-engine D2H per window
 *  DIRECT   one copy-engine D2H per fragment straight from the state tensors
 *  ZEROCOPY gather-pack kernel storing straight into mapped pinned host memory
 *  HYBRID   RING whose image exceeds the ring: the last ring-full is packed into the ring at
 *           issue, the head leaves by copy-engine DMA per fragment piece straight from the
 *           state (same capture point, the SMs pack a ring-full instead of the image); a full
 *           device shadow is plain RING */
enum { TS_D2H_RING = 0, TS_D2H_DIRECT = 1, TS_D2H_ZEROCOPY = 2, TS_D2H_HYBRID = 3 };

/* ------------------------------------------------------------------------ */
/* TLV values (tlv.hpp:24-83). Handles own their children once attached.     */

typedef struct ts_value ts_value;
enum { TS_V_NULL = 0, TS_V_INT = 1, TS_V_FLOAT = 2, TS_V_STRING = 3, TS_V_BYTES = 4,
       TS_V_LIST = 5, TS_V_MAP = 6 };

ts_value* ts_value_null(void);
ts_value* ts_value_int(int64_t v);
ts_value* ts_value_float(double v);
ts_value* ts_value_string(const char* s, size_t n);
ts_value* ts_value_bytes(const void* p, size_t n);
ts_value* ts_value_list(void);
ts_value* ts_value_map(void);
ts_status ts_value_list_append(ts_value* list, ts_value* item);                 /* takes item */
ts_status ts_value_map_set(ts_value* map, const char* k, size_t kn, ts_value* v); /* takes v */
void ts_value_free(ts_value* v);
int ts_value_type(const ts_value* v);
int64_t ts_value_as_int(const ts_value* v);
double ts_value_as_float(const ts_value* v);
/* string/bytes payload view (valid while v lives) */
const uint8_t* ts_value_data(const ts_value* v, size_t* n);
size_t ts_value_len(const ts_value* v); /* list/map element count */
const ts_value* ts_value_list_get(const ts_value* v, size_t i);
const ts_value* ts_value_map_key(const ts_value* v, size_t i, size_t* kn, const char** k);
/* tlv::encode (tlv.cpp:191-196); *len receives the size even when cap is too small */
ts_status ts_value_encode(const ts_value* v, uint8_t* buf, size_t cap, size_t* len);
size_t ts_value_encoded_size(const ts_value* v);
/* tlv::decode (tlv.cpp:198-203): strict */
ts_status ts_value_decode(const uint8_t* buf, size_t n, ts_value** out);
/* make_metadata_value (model.cpp:206-231) */
ts_value* ts_make_metadata_value(int rank_id, int tp_idx, int pp_idx, int dp_idx, uint64_t seed,
                                 uint64_t metadata_bytes, uint64_t iteration);

/* ------------------------------------------------------------------------ */
/* State descriptors (state_object / rank_state, model.hpp:34-73)            */

typedef struct ts_object_desc {
  uint64_t object_id;
  uint8_t kind;      /* TS_KIND_* */
  uint8_t tier;      /* TS_TIER_*: device => `data` is a device pointer */
  uint8_t precision; /* TS_PREC_* (bookkeeping only) */
  uint8_t _pad;
  uint32_t file_id;
  uint64_t size_bytes;   /* raw: payload size; structured: ignored (learned at serialization) */
  const void* data;      /* raw payload (device or host pointer per tier) */
  const ts_value* value; /* structured payload; must outlive the snapshot */
} ts_object_desc;

typedef struct ts_rank_info {
  int32_t rank_id, tp_idx, pp_idx, dp_idx;
} ts_rank_info;

/* ------------------------------------------------------------------------ */
/* Layout planner (provider.cpp:17-72). Exposed for tests and restore tools.  */

typedef struct ts_fixed_assignment {
  uint64_t object_id, file_offset, length;
} ts_fixed_assignment;

/* plan_layout: per file id (ascending) writes tensor_region_end and the fixed
 * assignments in plan order. files_out/ends_out have room for n entries,
 * fixed_out for n entries. Returns counts in *n_files / *n_fixed and the
 * plan_hash (provider.cpp:17-35) in *hash. */
ts_status ts_plan_layout(const ts_object_desc* objs, size_t n, uint64_t alignment,
                         uint32_t* files_out, uint64_t* ends_out, size_t* n_files,
                         ts_fixed_assignment* fixed_out, uint32_t* fixed_file_out,
                         size_t* n_fixed, uint64_t* hash);

/* FNV-1a-64 (common.hpp:44-51) on host memory. */
uint64_t ts_fnv1a64(const void* p, size_t n, uint64_t state);

/* ------------------------------------------------------------------------ */
/* Engine (checkpoint_engine, engine.hpp:92-153)                             */

typedef struct ts_engine ts_engine;
typedef struct ts_session ts_session;
typedef struct ts_ticket ts_ticket;

typedef struct ts_engine_config {
  /* reference knobs, engine.hpp:34-52 */
  int32_t strategy;                 /* TS_STRATEGY_*, default lazy */
  int32_t lazy_serialize_overlap;   /* default 1 */
  uint64_t staging_capacity_bytes;  /* pinned host pool, allocated once (staging.hpp:23-31) */
  int32_t flush_workers;            /* host worker threads (flush + serialize + checksum) */
  int32_t _pad0;
  uint64_t raw_chunk_bytes;         /* D2H window, default 16 MiB (provider.hpp:24) */
  uint64_t serialized_chunk_bytes;  /* append chunk, default 1 MiB (provider.hpp:25) */
  uint64_t alignment;               /* default 4096 (provider.hpp:23) */
  int64_t cache_acquire_timeout_ns; /* < 0: wait forever; default 300 s (engine.hpp:50) */
  int32_t overwrite;                /* default 1 */
  /* B200 knobs */
  int32_t d2h_mode;                 /* TS_D2H_*, default HYBRID (= RING for a full device shadow) */
  uint64_t device_staging_bytes;    /* HBM staging ring; >= image bytes => full device shadow */
  uint64_t hybrid_direct_min_bytes; /* HYBRID: the head goes by DMA only when its mean fragment
                                       piece is at least this (default 1 MiB); else plain RING */
  int32_t pack_ctas;                /* 0 = auto (one per SM) */
  int32_t pack_threads;             /* threads per pack CTA, default 512 */
  int32_t pack_priority;            /* capture (pack + checksum) stream priority: 1 highest (default:
                                       the capture is latency-critical and must not starve behind
                                       back-to-back compute kernels), 0 default, -1 lowest; the D2H
                                       copy stream always runs at the lowest priority */
  int32_t write_files;              /* 0 = snapshot-only run (no file I/O, bench only) */
  int32_t checksum_on_gpu;          /* 1 (default): exact segment-parallel FNV-1a kernels on the
                                       device copy; 0: host threads over the pinned pool */
  int32_t flush_mmap;               /* 1 (default): fixed-region flushes copy into a shared mapping
                                       of the file (parallel per file); 0: pwrite(2); 2: O_DIRECT
                                       pwrite of each window's 4 KiB-aligned body straight from the
                                       pinned pool (page cache bypassed; disks), buffered where
                                       the filesystem refuses O_DIRECT (tmpfs); 3: as 2, each body
                                       submitted through the flush thread's io_uring as 4 MiB
                                       writes in flight together (pwrite where io_uring is
                                       unavailable) */
  int32_t pack_kernel;              /* RING pack: 1 (default) = TMA bulk copies (cp.async.bulk
                                       through shared memory) for 16-B aligned fragments >=
                                       bulk_min_bytes, warp kernel for the rest, when the whole
                                       image fits the device staging (one pack); 2 = also in a
                                       multi-slot ring, with a 2-stage (64 KiB) kernel; 0 = warp
                                       gather kernel for everything */
  uint64_t bulk_min_bytes;          /* default 1 MiB */
  int32_t file_dma;                 /* 1 (default): D2H windows land directly in page-locked
                                       file pages (cudaHostRegister of a shared mapping, tmpfs)
                                       when a registration of the file exists; with a spare
                                       directory set, finalized files are registered in the
                                       background for reuse by rotation. 0: always pool + flush */
  int32_t checksum_priority;        /* RING device checksums (they read the staged copy, off the
                                       capture path) on their own stream: 1 highest, 0 default,
                                       -1 lowest (default: yield the SMs to training kernels) */
  int32_t _pad2;
  double checksum_host_frac;        /* checksum_on_gpu=1: share of device-tier bytes hashed by host
                                       workers instead of the FNV kernels. 0: all on the GPU;
                                       < 0 (default): auto — sized from the measured host hashing
                                       rate and the checkpoint cadence, objects a host chain can
                                       finish within that time only */
  uint64_t ring_chunk_bytes;        /* RING without a full shadow: bytes per ring slot (0 = auto:
                                       ring/6, at most 8 GiB; rounded to whole windows) */
  int32_t numa_bind;                /* 1 (default): engine threads and the pinned pool on the GPU's
                                       NUMA node (multi-socket hosts; no-op on one node) */
  int32_t worker_nice;              /* nice increment of the worker threads (default 19: background
                                       to the training process's launching thread); 0 = none */
  uint32_t helper_mask;             /* RING: devices (bit i = device i) whose copy engines may carry
                                       part of this rank's D2H, reading the staged image over NVLink
                                       (peer access) into host memory through their own PCIe links:
                                       load balancing for ranks holding more than their share
                                       (cfg2's dp-0 rank). 0 (default): none */
  uint32_t _pad4;
  double helper_share;              /* fraction of the image the helpers carry, spread evenly */
  int64_t checksum_lane_max_bytes;  /* RING device checksums: objects up to this size are hashed by
                                       the lane-serial FNV kernel (one lane per object, ~7 integer
                                       ops per byte instead of ~26) straight from the state, before
                                       the capture completes. 0 (default): off (segment-parallel
                                       kernels only); -1: auto — in a multi-slot ring, objects a
                                       lane (~85 MB/s) finishes within 40 % of the capture time */
} ts_engine_config;

void ts_engine_config_default(ts_engine_config* cfg);

/* checkpoint_engine ctor (engine.cpp:164-204): spawns the copier + worker pool,
 * allocates the pinned pool and binds `device`. */
ts_status ts_engine_create(const ts_engine_config* cfg, int rank_id, int device, ts_engine** out);
/* checkpoint_engine::shutdown (engine.cpp:213-234) + dtor */
ts_status ts_engine_destroy(ts_engine* e);
/* NUMA node the engine placed its threads and pinned pool on (-1: none / single node). */
int ts_engine_numa_node(ts_engine* e);

/* Manifest echo of a layout-based session (engine.cpp:35-54); NULL => defaults of
 * the n_ranks ctor (engine.cpp:56-66). */
typedef struct ts_manifest_echo {
  int32_t tp, pp, dp, zero1;
  uint64_t seed, n_params;
  int32_t layers, _pad;
  uint64_t metadata_bytes;
} ts_manifest_echo;

/* Checkpoint rotation (B200 addition; the reference never deletes): retire a
 * checkpoint directory (MANIFEST.tlv removed first, so it is no longer
 * restorable) and move its rank files to `spare_dir`; an engine given the same
 * spare directory takes those files over for its next checkpoints instead of
 * allocating fresh page-cache pages. Same filesystem required. */
ts_status ts_retire_checkpoint(const char* ckpt_dir, const char* spare_dir);
ts_status ts_engine_set_spare_dir(ts_engine* e, const char* spare_dir);
/* Creates up to `copies` spare files per file of the rank's layout in
 * `spare_dir` (sized to tensor_region_end, page-locked when file_dma applies),
 * so the first checkpoints of a rotation already take the direct D2H path.
 * `locked_bytes` (may be NULL): bytes page-locked. */
ts_status ts_engine_provision_spares(ts_engine* e, const char* spare_dir, const ts_rank_info* rank,
                                     const ts_object_desc* objs, size_t n, int copies,
                                     uint64_t* locked_bytes);
/* Page-locked checkpoint files (ts_engine_config.file_dma): bytes currently
 * locked, and an explicit release of every idle registration (files of deleted
 * checkpoints are also released at the next issue). */
uint64_t ts_file_cache_bytes(void);
/* Page-lock activity since process start: [registrations, ns inside
 * cudaHostRegister, bytes registered, unregistrations, ns unregistering].
 * Page-locking holds the driver for seconds per 100 GB; a training loop
 * should see none of it after its rotation is warm. B200-side addition. */
void ts_file_cache_stats(uint64_t out[5]);
ts_status ts_file_cache_release_all(uint64_t* released_bytes);

/* checkpoint_session (engine.hpp:57-90). `writes_manifest` = 1 on the process that
 * commits MANIFEST.tlv once all n_ranks ranks persisted (local or remote). */
ts_status ts_session_create(const char* dir, uint64_t checkpoint_id, uint64_t iteration,
                            const ts_manifest_echo* echo, int n_ranks, int writes_manifest,
                            ts_session** out);
ts_status ts_session_destroy(ts_session* s);
/* Multi-process: per-rank manifest info blob (TLV of manifest_rank_info, format.cpp:310-335)
 * produced locally and fed to the committing process (the NCCL allgather payload). */
ts_status ts_session_rank_blob(ts_session* s, int rank_id, uint8_t* buf, size_t cap, size_t* len);
ts_status ts_session_add_remote_rank(ts_session* s, const uint8_t* blob, size_t len);
/* Register a rank's manifest info without issuing (engine.cpp:539-558 part of
 * issue_checkpoint) and mark a rank persisted: lets a host-side coordinator
 * assemble a manifest for ranks checkpointed elsewhere. */
ts_status ts_session_register_rank(ts_session* s, const ts_rank_info* rank,
                                   const ts_object_desc* objs, size_t n);
ts_status ts_session_rank_persisted(ts_session* s, int rank_id);
ts_status ts_session_wait_complete(ts_session* s, int64_t timeout_ns);
int ts_session_complete(ts_session* s);

/* issue_checkpoint (engine.cpp:518-619). `producer_stream` is the stream whose
 * prior work produced the state; capture is ordered after it without blocking
 * the host. */
ts_status ts_issue(ts_engine* e, ts_session* s, const ts_rank_info* rank,
                   const ts_object_desc* objs, size_t n, uint64_t iteration,
                   void* producer_stream, ts_ticket** out);

/* pre_update_barrier (engine.cpp:621-630). host_block=1: reference semantics
 * (host waits until the state may be mutated); host_block=0: the barrier is a
 * cudaStreamWaitEvent on `optimizer_stream` (no host block). */
ts_status ts_pre_update_barrier(ts_engine* e, ts_ticket* t, void* optimizer_stream,
                                int host_block, int64_t* blocked_ns);

/* transfer_ticket (transfer.hpp:52-88) */
ts_status ts_ticket_wait_captured(ts_ticket* t, int64_t* blocked_ns); /* state may be mutated */
ts_status ts_ticket_wait_snapshot(ts_ticket* t, int64_t* blocked_ns); /* all bytes in host memory */
ts_status ts_ticket_wait_persisted(ts_ticket* t, int64_t* blocked_ns);
typedef struct ts_ticket_stats {
  uint64_t checkpoint_id;
  uint64_t total_bytes, raw_bytes, serialized_bytes, image_bytes;
  int64_t issue_block_ns, barrier_block_ns;
  int64_t t_captured_ns, t_snapshot_ns, t_persisted_ns; /* relative to issue start; -1 pending */
  float pack_ms;   /* CUDA-event time of the pack kernels (RING/ZEROCOPY/HYBRID) */
  float d2h_ms;    /* CUDA-event time from first to last D2H window */
  uint32_t kernel_launches, copies;
  int32_t snapshot_done, persisted_done, failed;
  uint64_t file_dma_bytes; /* fixed-region bytes the copy engines wrote straight into file pages */
  uint64_t host_checksum_bytes; /* device-tier bytes hashed by host workers (rest: FNV kernels) */
  uint64_t helper_bytes;        /* image bytes D2H'd by helper GPUs (helper_mask) */
  uint64_t direct_io_bytes;     /* fixed-region bytes written with O_DIRECT (flush_mmap = 2) */
  uint64_t lane_checksum_bytes; /* device-tier bytes hashed by the lane-serial FNV kernel */
  float lane_ms;                /* CUDA-event time of the lane-serial FNV kernel */
  uint32_t _pad5;
  uint64_t packed_bytes;        /* image bytes written into the HBM ring by the pack kernels
                                   (RING: the image; HYBRID: the last ring-full; other modes 0) */
} ts_ticket_stats;
ts_status ts_ticket_stats_get(ts_ticket* t, ts_ticket_stats* out);
/* Per-object checksum accumulated at staging (transfer.cpp:163-166) */
ts_status ts_ticket_object_checksum(ts_ticket* t, uint64_t object_id, uint64_t* out);
void ts_ticket_release(ts_ticket* t);
/* Hands `n` structured values the caller passed to ts_issue over to the ticket:
 * they are freed once the ticket is released AND its job has finished with
 * them, so a non-blocking caller need not keep them alive until the snapshot
 * (the reference's rank_state owns its values for the job's duration,
 * engine.cpp:563-565). B200-side addition. */
ts_status ts_ticket_adopt_values(ts_ticket* t, ts_value* const* values, size_t n);

/* ------------------------------------------------------------------------ */
/* Restore (format.cpp:201-494)                                              */

typedef struct ts_restore ts_restore;
typedef struct ts_restore_object {
  uint64_t object_id;
  uint8_t kind, tier, precision, _pad;
  uint32_t file_id;
  uint64_t size_bytes;
} ts_restore_object;

/* read_manifest (format.cpp:407-428) */
ts_status ts_restore_open(const char* manifest_path, ts_restore** out);
/* Closing the last open handle frees the process-wide restore staging (pinned
 * window ring, per-device HBM window ring and scratch, up to ~4 GiB each). */
void ts_restore_close(ts_restore* r);
/* Frees that staging now (e.g. before training resumes while a handle stays
 * open); returns the bytes freed. B200-side addition (no reference counterpart). */
uint64_t ts_restore_release_staging(void);
int ts_restore_n_ranks(ts_restore* r);
ts_status ts_restore_rank_info(ts_restore* r, int index, ts_rank_info* out);
/* Reads the footers of the rank's files and lists its objects in manifest order,
 * with sizes (format.cpp:247-287 without the payload). */
ts_status ts_restore_rank_objects(ts_restore* r, int index, ts_restore_object* out, size_t cap,
                                  size_t* n);
/* restore_checkpoint for one rank (format.cpp:430-494), B200 path: files -> pinned
 * -> FNV verify -> H2D -> scatter-unpack into `dst[i].data` (device pointers of
 * raw objects, sizes must match). Structured objects become ts_value handles
 * fetched with ts_restore_structured. */
typedef struct ts_restore_stats {
  uint64_t bytes;
  double read_s, verify_s, h2d_unpack_s, total_s;
  float unpack_ms, h2d_ms;
  uint32_t kernel_launches;
  uint32_t _pad;
  uint64_t direct_bytes; /* fixed-region bytes copied H2D straight from page-locked files (no pread) */
  uint64_t direct_io_bytes; /* fixed-region bytes read O_DIRECT (ts_restore_set_direct_io) */
} ts_restore_stats;
/* 1 (default): files page-locked by this process (file_dma rotation) are read
 * by the copy engines from their page cache; 0: always pread into pinned memory. */
ts_status ts_restore_set_file_cache(ts_restore* r, int use);
/* 1: fixed-region reads of files that are not page-locked go O_DIRECT from the
 * disk into the pinned windows (4 KiB-aligned bodies; ragged ends and
 * filesystems that refuse O_DIRECT use pread; tmpfs never goes O_DIRECT, its
 * "direct" reads are page-cache reads). 0: pread. -1 (default): O_DIRECT for
 * files mostly absent from the page cache (cold; probed per file with
 * preadv2(RWF_NOWAIT) on 64 sampled pages). */
ts_status ts_restore_set_direct_io(ts_restore* r, int use); /* 2: O_DIRECT via io_uring */
/* io_uring diagnostics (B200-side): 1 when this process can create a ring;
 * requests submitted through io_uring so far (flush_mmap = 3, direct_io = 2). */
int ts_io_uring_available(void);
uint64_t ts_io_uring_ops(void);
ts_status ts_restore_rank(ts_restore* r, int index, const ts_object_desc* dst, size_t n,
                          int device, void* stream, ts_restore_stats* stats);
ts_status ts_restore_structured(ts_restore* r, int index, uint64_t object_id, ts_value** out);

/* verify_checkpoint (format.cpp:496-529): never fails on a damaged checkpoint;
 * issues are reported as (status kind, object id or -1). */
typedef struct ts_verify_issue { int32_t kind; int32_t _pad; int64_t object_id; } ts_verify_issue;
typedef struct ts_verify_report {
  int32_t ok;
  int32_t n_issues;
  uint64_t files_checked, objects_checked;
} ts_verify_report;
ts_status ts_verify(const char* manifest_path, ts_verify_report* rep, ts_verify_issue* issues,
                    size_t cap);

/* ------------------------------------------------------------------------ */
/* Device kernels of the synthetic state (pattern.hpp:57-81, model.cpp:233-244) */

typedef struct ts_pattern_desc {
  void* data;           /* device pointer */
  uint64_t size;
  uint64_t space;       /* pattern space (model.cpp:17-19) */
  uint64_t offset;      /* pattern offset of byte 0 */
} ts_pattern_desc;

/* mutate_update_step on device: every fragment <- pattern(seed, space, iteration) */
ts_status ts_pattern_fill(const ts_pattern_desc* d, size_t n, uint64_t seed, uint64_t iteration,
                          void* stream);
/* matches_pattern on device: *mismatched_bytes = total mismatching bytes (0 = bit-exact) */
ts_status ts_pattern_verify(const ts_pattern_desc* d, size_t n, uint64_t seed,
                            uint64_t iteration, void* stream, uint64_t* mismatched_bytes);

/* FNV-1a-64 of `n` device byte ranges, computed on the GPU (segment-parallel,
 * exact). `init` (host, may be NULL = fresh seed) chains from prior states;
 * results land in host `out`. Synchronous w.r.t. the host. */
ts_status ts_fnv1a64_device(const void* const* ptrs, const uint64_t* sizes, size_t n,
                            const uint64_t* init, uint64_t* out, void* stream);
/* Same result, lane-serial kernel (one lane per range, ~7 integer ops per byte;
 * a range's time is its length at ~0.2 GB/s). B200-side addition. */
ts_status ts_fnv1a64_device_lanes(const void* const* ptrs, const uint64_t* sizes, size_t n,
                                  const uint64_t* init, uint64_t* out, void* stream);

/* Raw kernel entry for microbenchmarks: gather `n` device fragments into `dst`
 * (device or mapped-host) at dst_offsets, zero-filling the gaps up to `dst_len`. */
ts_status ts_pack(const void* const* srcs, const uint64_t* sizes, const uint64_t* dst_offsets,
                  size_t n, void* dst, uint64_t dst_len, int ctas, int threads, void* stream);
ts_status ts_unpack(const void* src, const uint64_t* src_offsets, void* const* dsts,
                    const uint64_t* sizes, size_t n, int ctas, int threads, void* stream);

/* Number of this library's kernels launched so far (process-wide). */
uint64_t ts_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TS_B200_H */
