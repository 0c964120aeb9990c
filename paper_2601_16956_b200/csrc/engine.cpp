// B200 snapshot engine (see engine.hpp for the reference mapping).
#include "engine.hpp"

#include <fcntl.h>
#include <sys/resource.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <unordered_set>

namespace tsb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(TS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

float elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  // (the end event may trail the work that was observed complete by a few
  // commands on its stream)
  if (cudaEventSynchronize(b) != cudaSuccess || cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();  // clear: unrecorded events are not an error here
    return 0;
  }
  return ms;
}

void mkdirs(const std::string& path) {
  std::string cur;
  for (size_t i = 0; i <= path.size(); ++i) {
    if (i == path.size() || path[i] == '/') {
      if (!cur.empty() && ::mkdir(cur.c_str(), 0755) != 0 && errno != EEXIST)
        fail(TS_ERR_IO, "cannot create directory " + cur + ": " + std::strerror(errno));
    }
    if (i < path.size()) cur += path[i];
  }
}

namespace {
const bool g_trace = std::getenv("TS_TRACE") != nullptr;
// Per-lane rate of the lane-serial FNV kernel, measured on B200 (alone and
// beside the training load alike: 131 MB in 1.52-1.54 s,
// profiles/r2_lanes_kernel.jsonl): sizes the auto object cap
// (checksum_lane_max_bytes < 0).
constexpr double kLaneBytesPerS = 0.085e9;
const bool g_trace_copies = std::getenv("TS_TRACE_COPIES") != nullptr;  // per-job enqueue cost summary
#define TRACE(...)                                                                     \
  do {                                                                                 \
    if (g_trace) {                                                                     \
      std::fprintf(stderr, "[ts %lld] ", (long long)(now_ns() / 1000 % 100000000));    \
      std::fprintf(stderr, __VA_ARGS__);                                               \
      std::fprintf(stderr, "\n");                                                      \
    }                                                                                  \
  } while (0)

}  // namespace

// ---------------------------------------------------------------------------
// ticket

ticket_state::~ticket_state() {
  cudaSetDevice(device);
  for (cudaEvent_t e : {ev_start, ev_capture, ev_d2h_first, ev_d2h_last, ev_pack0})
    if (e) cudaEventDestroy(e);
}

void ticket_state::fail(ts_status s, const std::string& m, int64_t oid) {
  {
    std::lock_guard<std::mutex> g(mu);
    if (!failed) {
      failed = true;
      err_status = s;
      err = m;
      err_oid = oid;
    }
  }
  cv.notify_all();
}

void ticket_state::throw_if_failed_locked() {
  if (failed) throw error(TS_ERR_TICKET, err, err_oid);
}

int64_t ticket_state::wait_until(const std::function<bool()>& pred) {
  std::unique_lock<std::mutex> g(mu);
  const int64_t t0 = now_ns();
  cv.wait(g, [&] { return failed || pred(); });
  throw_if_failed_locked();
  return now_ns() - t0;
}

// ---------------------------------------------------------------------------
// job: everything one issued checkpoint of one rank needs.

struct job {
  struct rawo {
    uint64_t oid = 0;
    uint32_t f = 0;
    uint64_t file_off = 0, size = 0, img = 0;
    const uint8_t* src = nullptr;
    bool device = true;
    bool gpu_ck = false;  // hashed by the FNV kernels (else by host workers)
    // checksum actor state (pieces arrive in object order)
    uint64_t fnv = fnv_seed, hashed = 0;
    bool busy = false, queued = false;
    struct piece {
      const uint8_t* p;
      uint64_t len;
      uint32_t w;
    };
    std::deque<piece> q;
  };
  struct fstate {
    uint32_t fid = 0;
    uint64_t tre = header_reserved, img = 0;
    std::unique_ptr<file_writer> w;
    // fixed region page-locked in file_registry: D2H windows land in the file
    uint8_t* dma = nullptr;
    file_key key;
    bool claimed = false, released = false;
    int win_pending = 0, raw_pending = 0, struct_pending = 0;
    bool appended = true, finalizing = false, finalized = false;
    std::vector<size_t> structs;
    std::vector<footer_entry> appends;
    uint64_t append_end = 0;
  };
  struct win {
    uint64_t lo = 0, hi = 0;
    pinned_pool::region r;
    uint8_t* host = nullptr;  // landing address: the pool region, or the file pages (dma)
    bool dma = false;
    int helper = -1;  // index into engine::helpers_ when a helper GPU copies this window
    cudaEvent_t ev = nullptr;
    int refs = 0;
    uint32_t wp_begin = 0, wp_end = 0, fs_begin = 0, fs_end = 0, hp_begin = 0, hp_end = 0;
  };
  struct wpiece {
    uint32_t obj;
    uint64_t len, win_off;
  };
  struct fseg {
    uint32_t f;
    uint64_t file_off, len, win_off;
  };
  struct hpiece {
    const uint8_t* src;
    uint64_t len, win_off;
  };
  struct sobj {
    uint64_t oid = 0;
    uint32_t f = 0;
    const value* v = nullptr;
    std::vector<uint8_t> enc;
    uint64_t ck = 0;
  };

  std::shared_ptr<session> sess;  // outlives the handle the caller may drop (engine.cpp:124 is a raw pointer)
  // lazy: the caller's descriptors, prepared on the copier thread (engine::prepare)
  bool deferred = false;
  std::vector<ts_object_desc> descs;
  ts_rank_info rank{};
  std::shared_ptr<ticket_state> t;
  int rank_id = 0;
  uint64_t iteration = 0;
  layout_plan plan;
  std::vector<rawo> raws;
  std::vector<fstate> files;
  std::vector<win> wins;
  std::vector<wpiece> wp;
  std::vector<fseg> fs;
  std::vector<hpiece> hp;
  std::vector<sobj> sobjs;
  std::deque<uint32_t> ready;  // host-hashed objects with landed, unhashed pieces
  std::vector<dev::seg> segs;
  std::vector<cudaEvent_t> chunk_events;  // per-job, destroyed at the end
  std::vector<cudaEvent_t> ck_events;     // RING: checksums of chunk c done
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pack_events;  // kernel-only pack timing
  uint64_t img = 0;
  uint64_t win_bytes = 0;  // D2H window size W: windows are cut at multiples of W
  bool io = true;
  // device checksums (checksum_on_gpu): device-tier raw objects hashed by the
  // FNV kernels; results land in a pool region
  // D2H order of the windows when the whole image is addressable (shadow,
  // direct, zero-copy): files interleaved in proportion to their size, so the
  // flushers fill every file concurrently from the first window on.
  std::vector<uint32_t> worder;
  bool gpu_ck = false, host_ck = false;
  std::vector<uint32_t> fnv_objs;
  uint64_t* fnv_out = nullptr;  // engine's mapped results buffer
  cudaEvent_t fnv_ev = nullptr;
  // lane-serial checksums (RING): launched at the start of the capture over the
  // state; the capture and the results' publication wait for lane_ev1
  cudaEvent_t lane_ev0 = nullptr, lane_ev1 = nullptr;

  ~job() {
    for (auto& f : files)  // a claimed file that never finalized: its pages may be stale
      if (f.claimed && !f.released) file_registry::get().release(f.key, -1, false);
    for (auto e : chunk_events)
      if (e) cudaEventDestroy(e);
    for (auto e : ck_events)
      if (e) cudaEventDestroy(e);
    for (auto& pe : pack_events) {
      cudaEventDestroy(pe.first);
      cudaEventDestroy(pe.second);
    }
    if (lane_ev0) cudaEventDestroy(lane_ev0);
    if (lane_ev1) cudaEventDestroy(lane_ev1);
  }

  std::mutex mu;
  size_t wins_landed = 0, wins_enqueued = 0, structs_pending = 0, files_done = 0;
  std::condition_variable land_cv;  // wins_landed advanced (bounded enqueue in run_job)
  int64_t t_landed_all = -1;        // now_ns() when the last window landed (the D2H's end)
  // checksum placement inputs, taken at issue (engine::issue) for prepare
  double slack_s = 0, slack_d2h_s = 0, host_rate = 0;
  // host workers hash only once the whole image has landed (no competition
  // with the D2H for host memory bandwidth; every host object's chain ready)
  bool defer_hash = false;
  bool enqueue_done = false, snapshot_done = false, persisted = false;
};

// ---------------------------------------------------------------------------
// engine

namespace {
// Worker-task wrapper: a failure inside a task fails the ticket (and is
// reported on the next wait) instead of terminating the process.
template <class F>
std::function<void()> guarded(const std::shared_ptr<job>& j, F&& f) {
  return [j, f = std::forward<F>(f)]() mutable {
    try {
      f();
    } catch (const error& e) {
      j->t->fail(e.status, e.what(), e.object_id);
    } catch (const std::exception& e) {
      j->t->fail(TS_ERR_GENERIC, e.what());
    }
  };
}
}  // namespace

engine::engine(const ts_engine_config& cfg, int rank_id, int device)
    : cfg_(cfg), rank_id_(rank_id), device_(device) {
  if (cfg_.flush_workers < 1) fail(TS_ERR_GENERIC, "engine: need at least one flush worker");
  if (cfg_.raw_chunk_bytes == 0) fail(TS_ERR_GENERIC, "raw source: zero chunk size");
  if (cfg_.serialized_chunk_bytes == 0) fail(TS_ERR_GENERIC, "serialize_structured: zero chunk size");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(TS_ERR_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  sms_ = dev::sm_count(device_);
  if (cfg_.numa_bind) numa_ = numa_for_device(device_);
  {
    numa_prefer_scope near(numa_);  // pinned pool pages on the GPU's node
    pool_ = std::make_unique<pinned_pool>(cfg_.staging_capacity_bytes);
  }
  int lo_prio = 0, hi_prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  // Capture kernels preempt compute at CTA granularity (high priority): at low
  // priority they starve behind back-to-back training kernels and the capture,
  // hence the pre-update barrier, slips. Copies use the copy engines only.
  const int pack_prio = cfg_.pack_priority > 0 ? hi_prio : cfg_.pack_priority < 0 ? lo_prio : 0;
  cuda_check(cudaStreamCreateWithPriority(&pack_stream_, cudaStreamNonBlocking, pack_prio), "stream");
  cuda_check(cudaStreamCreateWithPriority(&copy_stream_, cudaStreamNonBlocking, lo_prio), "stream");
  // RING checksums read the staged copy, not the state: they are off the
  // capture path and may run at a lower priority than the pack.
  const int ck_prio = cfg_.checksum_priority > 0 ? hi_prio : cfg_.checksum_priority < 0 ? lo_prio : 0;
  cuda_check(cudaStreamCreateWithPriority(&ck_stream_, cudaStreamNonBlocking, ck_prio), "stream");
  // ...except where the capture depends on them: a ring slot is repacked only
  // after its checksums, so those run at the pack's priority (at low priority
  // they starve behind back-to-back training kernels and stall the capture)
  cuda_check(cudaStreamCreateWithPriority(&ck_hi_stream_, cudaStreamNonBlocking, pack_prio), "stream");
  // Lane-serial checksums read the state, so the capture waits for them: a
  // few warps for most of the D2H, at the pack's priority (TS_LANE_PRIO
  // overrides: 1 / 0 / -1, for A/B runs).
  {
    int lp = pack_prio;
    if (const char* e = std::getenv("TS_LANE_PRIO")) {
      const int v = std::atoi(e);
      lp = v > 0 ? hi_prio : v < 0 ? lo_prio : 0;
    }
    cuda_check(cudaStreamCreateWithPriority(&ck_lane_stream_, cudaStreamNonBlocking, lp), "stream");
  }
  // Workers (checksums, flushes, serialization, page locking) are background
  // work: a lower CPU priority keeps the training process's kernel-launching
  // thread responsive when every core is hashing.
  const int nice_inc = cfg_.worker_nice;
  // Helper GPUs for D2H load balancing (RING): a stream on each, with peer
  // access to this GPU's memory (the staged image is read over NVLink).
  for (int d = 0; d < 32; ++d) {
    if (!(cfg_.helper_mask & (1u << d)) || d >= ndev) continue;
    if (d != device_) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, d, device_);
      if (!can) continue;
    }
    auto h = std::make_unique<helper_dev>();
    h->dev = d;
    cuda_check(cudaSetDevice(d), "cudaSetDevice(helper)");
    if (d != device_) {
      const cudaError_t pe = cudaDeviceEnablePeerAccess(device_, 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) cuda_check(pe, "peer access (helper)");
      cudaGetLastError();
    }
    int hlo = 0, hhi = 0;
    cudaDeviceGetStreamPriorityRange(&hlo, &hhi);
    cuda_check(cudaStreamCreateWithPriority(&h->st, cudaStreamNonBlocking, hlo), "helper stream");
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    helpers_.push_back(std::move(h));
  }
  workers_ = std::make_unique<thread_pool>(cfg_.flush_workers, [this, nice_inc] {
    numa_bind_thread(numa_);
    if (nice_inc > 0) setpriority(PRIO_PROCESS, static_cast<id_t>(syscall(SYS_gettid)), nice_inc);
  });
  host_rate_ = 1.2e9 * cfg_.flush_workers;  // until measured: ~1.2 GB/s per worker (4 interleaved chains)
  copier_ = std::thread([this] { copier_loop(); });
  completer_ = std::thread([this] { completer_loop(); });
}

engine::~engine() {
  shutdown();
  cudaSetDevice(device_);
  if (ring_) cudaFree(ring_);
  if (segbuf_) cudaFree(segbuf_);
  if (fnvbuf_) cudaFree(fnvbuf_);
  if (ck_host_) cudaFreeHost(ck_host_);
  if (pack_stream_) cudaStreamDestroy(pack_stream_);
  if (ck_stream_) cudaStreamDestroy(ck_stream_);
  if (ck_hi_stream_) cudaStreamDestroy(ck_hi_stream_);
  if (ck_lane_stream_) cudaStreamDestroy(ck_lane_stream_);
  for (auto& h : helpers_) {
    cudaSetDevice(h->dev);
    for (auto e : h->free_ev) cudaEventDestroy(e);
    if (h->st) cudaStreamDestroy(h->st);
  }
  cudaSetDevice(device_);
  if (copy_stream_) cudaStreamDestroy(copy_stream_);
  for (auto e : ev_free_) cudaEventDestroy(e);
}

void engine::shutdown() {
  {
    std::lock_guard<std::mutex> g(mu_);
    if (stopping_ && !copier_.joinable()) return;
    stopping_ = true;
  }
  cv_.notify_all();
  if (copier_.joinable()) copier_.join();
  {
    std::lock_guard<std::mutex> g(mu_);
    copier_done_ = true;
  }
  cv_.notify_all();
  if (completer_.joinable()) completer_.join();
  // Let outstanding checksum / flush / finalize tasks run to completion.
  if (last_job_) {
    auto t = last_job_->t;
    std::unique_lock<std::mutex> g(t->mu);
    t->cv.wait(g, [&] { return t->failed || t->persisted; });
  }
  workers_.reset();
  last_job_.reset();
  retired_.clear();
}

cudaEvent_t engine::get_event() {
  {
    std::lock_guard<std::mutex> g(ev_mu_);
    if (!ev_free_.empty()) {
      auto e = ev_free_.back();
      ev_free_.pop_back();
      return e;
    }
  }
  cudaEvent_t e;
  cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync), "event");
  return e;
}

void engine::put_event(cudaEvent_t e) {
  std::lock_guard<std::mutex> g(ev_mu_);
  ev_free_.push_back(e);
}

cudaEvent_t engine::helper_event(size_t k) {
  auto& h = *helpers_[k];
  {
    std::lock_guard<std::mutex> g(h.mu);
    if (!h.free_ev.empty()) {
      auto e = h.free_ev.back();
      h.free_ev.pop_back();
      return e;
    }
  }
  cudaEvent_t e;  // events belong to the device of the stream they are recorded on
  cuda_check(cudaSetDevice(h.dev), "cudaSetDevice(helper)");
  const cudaError_t ce = cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync);
  cudaSetDevice(device_);
  cuda_check(ce, "helper event");
  return e;
}

void engine::put_helper_event(size_t k, cudaEvent_t e) {
  std::lock_guard<std::mutex> g(helpers_[k]->mu);
  helpers_[k]->free_ev.push_back(e);
}

uint8_t* engine::ensure_device_ring(uint64_t bytes) {
  if (ring_bytes_ < bytes) {
    if (ring_) cudaFree(ring_);
    ring_ = nullptr;
    ring_bytes_ = 0;
    cuda_check(cudaMalloc(&ring_, bytes), "cudaMalloc(device staging ring)");
    ring_bytes_ = bytes;
  }
  return ring_;
}

// The checksum scratch and the segment tables regrow when a job needs more
// (the auto checksum placement changes the GPU share, hence the segment
// length and count, from job to job). Stream-ordered on the pack stream,
// where every earlier user of the old buffer is already ordered (run_job
// orders each job after the previous one's checksums): a cudaFree there
// would synchronize the whole device — wait out the training kernels — and
// stall the training thread's own CUDA calls behind the driver for as long
// (measured: one 795 ms cudaEventRecord in a lazy training block).
// Headroom: 1.5x, so growth is rare.
uint8_t* engine::ensure_fnv_buffer(uint64_t bytes) {
  if (fnvbuf_bytes_ < bytes) {
    const uint64_t want = std::max<uint64_t>(bytes + bytes / 2, 1ull << 20);
    if (fnvbuf_) cuda_check(cudaFreeAsync(fnvbuf_, pack_stream_), "cudaFreeAsync(checksum scratch)");
    fnvbuf_ = nullptr;
    fnvbuf_bytes_ = 0;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&fnvbuf_), want, pack_stream_),
               "cudaMallocAsync(checksum scratch)");
    fnvbuf_bytes_ = want;
  }
  return fnvbuf_;
}

void* engine::ensure_seg_buffer(uint64_t bytes) {
  if (segbuf_bytes_ < bytes) {
    const uint64_t want = std::max<uint64_t>(bytes + bytes / 2, 1ull << 20);
    if (segbuf_) cuda_check(cudaFreeAsync(segbuf_, pack_stream_), "cudaFreeAsync(segment table)");
    segbuf_ = nullptr;
    segbuf_bytes_ = 0;
    cuda_check(cudaMallocAsync(&segbuf_, want, pack_stream_), "cudaMallocAsync(segment table)");
    segbuf_bytes_ = want;
  }
  return segbuf_;
}

uint64_t engine::provision_spares(const std::string& spare_dir, const ts_rank_info& rank,
                                  const ts_object_desc* objs, size_t n, int copies) {
  const layout_plan plan = plan_layout(objs, n, cfg_.alignment);
  mkdirs(spare_dir);
  struct item {
    int fd;
    uint64_t len;
  };
  std::vector<item> made;
  for (const auto& fp : plan.files) {
    if (fp.tensor_region_end <= header_reserved) continue;
    const std::string name = rank_dir_name(rank.rank_id) + "_file_" + std::to_string(fp.file_id) + ".bin";
    int have = 0;
    for (int k = 0; k < kMaxSpares; ++k)
      have += ::access((spare_dir + "/" + name + (k ? "." + std::to_string(k) : std::string())).c_str(), F_OK) == 0;
    for (int c = have; c < std::min(copies, kMaxSpares); ++c) {
      const std::string p = spare_put_name(spare_dir, name);
      const int fd = ::open(p.c_str(), O_RDWR | O_CREAT | O_EXCL, 0644);
      if (fd < 0) fail(TS_ERR_IO, "cannot create spare " + p + ": " + std::strerror(errno));
      if (::ftruncate(fd, static_cast<off_t>(fp.tensor_region_end)) != 0) {
        ::close(fd);
        fail(TS_ERR_IO, "cannot size spare " + p + ": " + std::strerror(errno));
      }
      made.push_back({fd, fp.tensor_region_end});
    }
  }
  // Lock the new files' pages, one thread per file (page allocation + pinning).
  std::atomic<uint64_t> locked{0};
  std::vector<std::thread> th;
  for (const auto& m : made)
    th.emplace_back([&, m] {
      file_key k;
      if (cfg_.file_dma && file_registry::get().want_register(m.fd, m.len, &k)) {
        file_registry::get().register_file(k, device_);
        locked += m.len;
      }
    });
  for (auto& t : th) t.join();
  for (const auto& m : made) ::close(m.fd);
  return locked.load();
}

namespace {
// The argument checks of plan_layout (duplicate ids, raw objects of unknown
// size; provider.cpp:37-50, same messages) plus missing payloads, in O(n log n)
// over the ids alone, so they raise at issue even when the plan is deferred.
void validate_objects(const ts_object_desc* objs, size_t n) {
  // first repeated id in object order (the position plan_layout reports it at)
  std::vector<std::pair<uint64_t, size_t>> ids(n);
  for (size_t i = 0; i < n; ++i) ids[i] = {objs[i].object_id, i};
  std::sort(ids.begin(), ids.end());
  size_t dup_at = n;
  for (size_t k = 1; k < n; ++k)
    if (ids[k].first == ids[k - 1].first) dup_at = std::min(dup_at, ids[k].second);
  for (size_t i = 0; i < n; ++i) {
    const ts_object_desc& d = objs[i];
    if (i == dup_at) fail(TS_ERR_GENERIC, "plan_layout: duplicate object id " + std::to_string(d.object_id));
    if (d.kind == TS_KIND_STRUCTURED) {
      if (!d.value) fail(TS_ERR_INVALID_ARG, "structured object without a value", static_cast<int64_t>(d.object_id));
    } else {
      if (d.size_bytes == 0) fail(TS_ERR_GENERIC, "plan_layout: raw buffer without a known size");
      if (!d.data) fail(TS_ERR_INVALID_ARG, "raw object without payload", static_cast<int64_t>(d.object_id));
    }
  }
}
}  // namespace

// issue_checkpoint (engine.cpp:518-619), lazy by default.
std::shared_ptr<ticket_state> engine::issue(const std::shared_ptr<session>& sp, const ts_rank_info& rank,
                                            const ts_object_desc* objs, size_t n,
                                            uint64_t iteration, cudaStream_t producer) {
  session& s = *sp;
  const int64_t t0 = now_ns();
  if (last_job_) {
    // Host slack of the checkpoint cadence: time from the previous checkpoint's
    // persist to this issue (EMA). ~0 when the caller waits for persist before
    // issuing again (closed loop), large when checkpoints are spaced by
    // training steps; forgotten after a long pause.
    int64_t prev_issue = 0, prev_persist = -1, prev_landed = -1;
    {
      std::lock_guard<std::mutex> g(last_job_->t->mu);
      prev_issue = last_job_->t->t_issue;
      prev_persist = last_job_->t->persisted ? last_job_->t->t_persisted : -1;
    }
    {
      std::lock_guard<std::mutex> g(last_job_->mu);
      prev_landed = last_job_->t_landed_all;
    }
    const double gap = prev_persist < 0 ? 0.0 : static_cast<double>(t0 - prev_issue - prev_persist) / 1e9;
    // (drops at once when the host fell behind, grows slowly)
    slack_s_ = gap > 120 ? 0 : gap < slack_s_ ? std::max(0.0, gap) : 0.75 * slack_s_ + 0.25 * gap;
    // time from the previous D2H's end to this issue: what deferred host
    // hashing can use
    const double gap2 = prev_landed < 0 ? 0.0 : static_cast<double>(t0 - prev_landed) / 1e9;
    slack_d2h_s_ = gap2 > 120 ? 0 : gap2 < slack_d2h_s_ ? std::max(0.0, gap2) : 0.75 * slack_d2h_s_ + 0.25 * gap2;
  }
  if (hash_bytes_.load() > (256ull << 20)) {  // host hashing rate of the previous jobs
    const double per_thread = static_cast<double>(hash_bytes_.load()) / std::max<double>(1, hash_busy_ns_.load()) * 1e9;
    host_rate_ = 0.9 * per_thread * cfg_.flush_workers;
    hash_bytes_ = 0;
    hash_busy_ns_ = 0;
  }
  // One consistent device view at a time (engine.cpp:523-525).
  if (cfg_.strategy == TS_STRATEGY_LAZY && last_job_) {
    auto prev = last_job_->t;
    std::unique_lock<std::mutex> g(prev->mu);
    prev->cv.wait(g, [&] { return prev->failed || prev->snapshot; });
    prev->throw_if_failed_locked();
  }
  const int64_t t_wait = now_ns();
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");

  auto j = std::make_shared<job>();
  j->slack_s = slack_s_;
  j->slack_d2h_s = slack_d2h_s_;
  j->host_rate = host_rate_;
  j->sess = sp;
  j->rank_id = rank.rank_id;
  j->iteration = iteration;
  j->io = cfg_.write_files != 0;
  // Argument errors stay issue-time errors, as in the reference (plan_layout's
  // checks, provider.cpp:37-50, and missing payloads); the plan itself is
  // built by prepare().
  validate_objects(objs, n);
  auto t = std::make_shared<ticket_state>();
  j->t = t;
  t->checkpoint_id = s.checkpoint_id();
  t->rank_id = rank.rank_id;
  t->device = device_;
  t->t_issue = t0;
  for (cudaEvent_t* e : {&t->ev_start, &t->ev_capture, &t->ev_d2h_first, &t->ev_d2h_last, &t->ev_pack0})
    cuda_check(cudaEventCreate(e), "cudaEventCreate");
  // The capture is ordered after everything already queued on the producer.
  cuda_check(cudaEventRecord(t->ev_start, producer), "cudaEventRecord(producer)");
  const int64_t t_rec = now_ns();

  // Lazy with overlapped serialization (the default): everything else — files
  // (open, pre-size, page-lock registry claim), the image layout, segment and
  // window tables, checksum placement, manifest registration, serializer tasks
  // — is prepared by the copier thread just before it enqueues the capture, so
  // the training thread pays for the plan, a descriptor copy and one event
  // record. Blocking strategies and inline serialization ("DataStates-Old")
  // prepare here, as the reference does (engine.cpp:531-573).
  const bool inline_ser = cfg_.strategy == TS_STRATEGY_LAZY && !cfg_.lazy_serialize_overlap;
  const bool deferred = cfg_.strategy == TS_STRATEGY_LAZY && !inline_ser;
  if (deferred) {
    j->descs.assign(objs, objs + n);
    j->rank = rank;
    j->deferred = true;
  } else {
    prepare(j, rank, objs, n);
  }
  if (inline_ser) {
    for (size_t k = 0; k < j->sobjs.size(); ++k) serialize_task(j, k);
  }
  {
    std::lock_guard<std::mutex> g(mu_);
    jobs_.push_back(j);
    // the previous job's tables, events and file states are torn down by the
    // copier, not on the training thread (~0.5 ms for 3,616 objects)
    if (last_job_) retired_.push_back(std::move(last_job_));
  }
  cv_.notify_all();
  last_job_ = j;
  TRACE("issue rank=%d n=%zu deferred=%d us: wait %.0f plan+ticket %.0f rest %.0f", rank.rank_id, n, (int)deferred,
        (t_wait - t0) / 1e3, (t_rec - t_wait) / 1e3, (now_ns() - t_rec) / 1e3);

  if (cfg_.strategy == TS_STRATEGY_SYNC) {
    t->wait_until([&] { return t->persisted; });
  } else if (cfg_.strategy == TS_STRATEGY_TWO_PHASE) {
    t->wait_until([&] { return t->snapshot; });
  }
  t->issue_block_ns = now_ns() - t0;
  return t;
}

// The host-side plan of one job (engine.cpp:531-573 of the reference's issue,
// plus the B200 image / window / checksum tables): training thread for the
// blocking strategies, copier thread for lazy.
void engine::prepare(const std::shared_ptr<job>& j, const ts_rank_info& rank, const ts_object_desc* objs, size_t n) {
  session& s = *j->sess;
  ticket_state* t = j->t.get();
  j->plan = plan_layout(objs, n, cfg_.alignment);

  std::unordered_map<uint64_t, size_t> by_id;
  by_id.reserve(n * 2);
  for (size_t i = 0; i < n; ++i) by_id.emplace(objs[i].object_id, i);

  // Files, image layout: each file's tensor region [4096, tre) maps to image
  // [img, img + tre - 4096), file images 4 KiB aligned so that every object
  // starts 16-B aligned in the image.
  const std::string rdir = s.rank_dir(rank.rank_id);
  if (j->io) {
    mkdirs(rdir);
    file_registry::get().sweep();  // registrations of deleted checkpoints
  }
  std::unordered_map<uint32_t, uint32_t> fidx;
  uint64_t cursor = 0;
  const std::string spare = spare_dir();
  for (const auto& fp : j->plan.files) {
    job::fstate fs;
    fs.fid = fp.file_id;
    fs.tre = fp.tensor_region_end;
    cursor = align_up(cursor, 4096);
    fs.img = cursor;
    cursor += fp.tensor_region_end - header_reserved;
    const std::string fname = "file_" + std::to_string(fp.file_id) + ".bin";
    const std::string recycled = spare.empty() ? std::string() : spare_take(spare, rank_dir_name(rank.rank_id) + "_" + fname);
    // Every opened file passes through the registry before it is truncated
    // (locked pages must never be dropped); a valid registration of exactly
    // [0, tre) makes the file's D2H windows land in its pages.
    auto on_open = [&](int fd) {
      uint8_t* m = file_registry::get().claim(fd, fp.tensor_region_end, &fs.key);
      if (!m) return false;
      fs.claimed = true;
      if (cfg_.file_dma && fp.tensor_region_end > header_reserved) {
        fs.dma = m;
      } else {  // not wanted here: drop it before the file changes
        file_registry::get().release(fs.key, -1, false);
        fs.released = true;
      }
      return fs.dma != nullptr;
    };
    try {
      fs.w = std::make_unique<file_writer>(rdir + "/" + fname, fp.tensor_region_end, j->plan.hash,
                                           cfg_.overwrite != 0, j->io, recycled, on_open);
    } catch (...) {  // (header write / pre-size failed after the claim: give the entry back)
      if (fs.claimed && !fs.released) file_registry::get().release(fs.key, -1, false);
      throw;
    }
    fs.append_end = fp.tensor_region_end;
    if (cfg_.flush_mmap >= 2 && !fs.dma) {
      if (fs.w->open_direct() && cfg_.flush_mmap == 3) fs.w->use_uring(true);
    }
    else if (cfg_.flush_mmap && !fs.dma) fs.w->map_fixed_region();
    fidx.emplace(fp.file_id, static_cast<uint32_t>(j->files.size()));
    j->files.push_back(std::move(fs));
  }
  j->img = cursor;

  // Raw objects in image order + the pack segment table covering [0, img)
  // (zero segments for alignment gaps and inter-file padding).
  uint64_t raw_bytes = 0, seg_end = 0;
  auto push_seg = [&](uint64_t pos, uint64_t len, const uint8_t* src) {
    if (len) j->segs.push_back({pos, len, src});
    seg_end = pos + len;
  };
  for (size_t fi = 0; fi < j->plan.files.size(); ++fi) {
    const auto& fp = j->plan.files[fi];
    auto& fs = j->files[fi];
    if (fs.img > seg_end) push_seg(seg_end, fs.img - seg_end, nullptr);
    uint64_t foff = header_reserved;
    for (const auto& a : fp.fixed) {
      const ts_object_desc& d = objs[by_id.at(a.object_id)];
      if (a.file_offset > foff)
        push_seg(fs.img + (foff - header_reserved), a.file_offset - foff, nullptr);
      job::rawo r;
      r.oid = a.object_id;
      r.f = static_cast<uint32_t>(fi);
      r.file_off = a.file_offset;
      r.size = a.length;
      r.img = fs.img + (a.file_offset - header_reserved);
      r.src = static_cast<const uint8_t*>(d.data);
      r.device = d.tier == TS_TIER_DEVICE;
      push_seg(r.img, r.size, r.device ? r.src : nullptr);
      j->raws.push_back(std::move(r));
      fs.raw_pending += 1;
      raw_bytes += a.length;
      foff = a.file_offset + a.length;
    }
  }

  j->gpu_ck = cfg_.checksum_on_gpu != 0;
  if (j->gpu_ck) {
    // Checksum placement: the host workers take a
    // share of the device-tier objects (spread evenly over the image, only
    // objects one host chain finishes within the budget), the FNV kernels the
    // rest. The share is fixed (checksum_host_frac >= 0) or sized so the host
    // keeps up with the checkpoint cadence at its measured rate (< 0, auto).
    uint64_t dev_bytes = 0;
    for (const auto& r : j->raws) dev_bytes += r.device ? r.size : 0;
    double frac = cfg_.checksum_host_frac;
    double obj_cap = 1e30;
    if (frac < 0) {
      // The FNV kernels overlap the D2H for free when nothing else runs on
      // the GPU; host workers are worth it only for the slack before the next
      // checkpoint (a training loop). A closed loop (caller waits for persist,
      // no slack) keeps everything on the GPU, so host-held pool windows can
      // never throttle the D2H.
      //
      // Host-hashed windows that land in the pinned pool hold it until hashed:
      // only when the pool takes all of them can hashing not throttle the D2H.
      uint64_t pool_bytes = 0;
      for (const auto& f : j->files)
        if (!(j->io && f.dma)) pool_bytes += f.tre - header_reserved;
      // Optional (TS_HOST_CK_DEFER=1): when every window lands in a
      // page-locked file (rotation), the host hashes after the D2H: its budget
      // is the time from the end of the D2H to the next issue and every host
      // object is complete from the start (4 chains per worker). Measured on
      // cfg4 it takes ~47 % of the bytes and cuts the GPU-side cost from
      // +4.0 % to +3.2 %, but the step slows more overall (5.3-5.6 % vs
      // 4.1-4.9 %: 16 workers hashing flat out right after the D2H also slow
      // the training process's host side), so hashing as windows land stays
      // the default (profiles/r2_defer_ab.jsonl).
      const char* dv = std::getenv("TS_HOST_CK_DEFER");
      const bool want_defer = dv && dv[0] == '1';
      const double d2h_s = static_cast<double>(j->img) / 50e9;
      const bool defer = want_defer && pool_bytes == 0 && j->io && j->slack_s > 0.05;
      const double budget = defer ? j->slack_d2h_s : j->slack_s;
      frac = dev_bytes ? std::min(1.0, 0.8 * j->host_rate * budget / static_cast<double>(dev_bytes)) : 0.0;
      // one host chain must finish within the budget
      obj_cap = 0.8 * chain_rate_ * (defer ? j->slack_d2h_s : d2h_s + j->slack_s);
      if (pool_bytes > pool_->capacity()) frac = 0.0;
      j->defer_hash = defer && frac > 0;
    }
    uint64_t seen = 0, host = 0;
    for (size_t k = 0; k < j->raws.size(); ++k) {
      auto& r = j->raws[k];
      if (!r.device) continue;
      seen += r.size;
      const bool to_host = frac > 0 && static_cast<double>(r.size) <= obj_cap &&
                           static_cast<double>(host + r.size) <= frac * static_cast<double>(seen) + 0.5;
      if (to_host) {
        host += r.size;
      } else {
        r.gpu_ck = true;
        j->fnv_objs.push_back(static_cast<uint32_t>(k));
      }
    }
    {
      std::lock_guard<std::mutex> g(t->mu);
      t->host_checksum_bytes = host;
    }
    j->host_ck = host > 0;
  }

  // D2H windows over [0, img) and their pieces (one sweep).
  const uint64_t W = std::min<uint64_t>(cfg_.raw_chunk_bytes, pool_->capacity());
  j->win_bytes = W;
  // Windows lie inside one file's fixed region (so a window has one contiguous
  // landing range: a pool region or the file's locked pages) and inside one
  // W-aligned slice of the image (so inside one ring chunk); the 4 KiB padding
  // between file images is never transferred.
  {
    size_t ri = 0;
    for (size_t fi = 0; fi < j->files.size(); ++fi) {
      auto& f = j->files[fi];
      const uint64_t fe = f.img + (f.tre - header_reserved);
      for (uint64_t lo = f.img; lo < fe;) {
        job::win w;
        w.lo = lo;
        w.hi = std::min(fe, (lo / W + 1) * W);
        lo = w.hi;
        w.dma = j->io && f.dma != nullptr;
        w.wp_begin = static_cast<uint32_t>(j->wp.size());
        w.fs_begin = static_cast<uint32_t>(j->fs.size());
        w.hp_begin = static_cast<uint32_t>(j->hp.size());
        while (ri < j->raws.size() && j->raws[ri].img + j->raws[ri].size <= w.lo) ++ri;
        for (size_t k = ri; k < j->raws.size() && j->raws[k].img < w.hi; ++k) {
          const auto& r = j->raws[k];
          const uint64_t a = std::max(w.lo, r.img), b = std::min(w.hi, r.img + r.size);
          if (b <= a) continue;
          j->wp.push_back({static_cast<uint32_t>(k), b - a, a - w.lo});
          if (!r.device) j->hp.push_back({r.src + (a - r.img), b - a, a - w.lo});
        }
        j->fs.push_back({static_cast<uint32_t>(fi), header_reserved + (w.lo - f.img), w.hi - w.lo, 0});
        if (j->io) f.win_pending += 1;
        if (w.dma) w.host = f.dma + header_reserved + (w.lo - f.img);
        w.wp_end = static_cast<uint32_t>(j->wp.size());
        w.fs_end = static_cast<uint32_t>(j->fs.size());
        w.hp_end = static_cast<uint32_t>(j->hp.size());
        j->wins.push_back(w);
      }
    }
    std::vector<std::pair<double, uint32_t>> key(j->wins.size());
    for (size_t k = 0; k < j->wins.size(); ++k) {
      const auto& w = j->wins[k];
      double frac = 0;
      if (w.fs_end > w.fs_begin) {
        const auto& f = j->files[j->fs[w.fs_begin].f];
        frac = double(w.lo > f.img ? w.lo - f.img : 0) / double(std::max<uint64_t>(1, f.tre - header_reserved));
      }
      key[k] = {frac, static_cast<uint32_t>(k)};
    }
    // Host-hashed pieces must reach their checksum actor in object order.
    const bool host_hashed = !cfg_.checksum_on_gpu || j->host_ck || !j->hp.empty();
    if (!host_hashed) std::stable_sort(key.begin(), key.end());
    for (const auto& kv : key) j->worder.push_back(kv.second);
  }

  // Structured objects, in rank.objects order (the canonical append order).
  for (size_t i = 0; i < n; ++i) {
    if (objs[i].kind != TS_KIND_STRUCTURED) continue;
    job::sobj so;
    so.oid = objs[i].object_id;
    so.f = fidx.at(objs[i].file_id);
    so.v = V(objs[i].value);
    auto& fs = j->files[so.f];
    fs.structs.push_back(j->sobjs.size());
    fs.struct_pending += 1;
    fs.appended = false;
    j->sobjs.push_back(std::move(so));
  }
  j->structs_pending = j->sobjs.size();

  s.register_rank(make_rank_info(rank, objs, n));

  {
    std::lock_guard<std::mutex> g(t->mu);
    t->raw_bytes = raw_bytes;
    t->image_bytes = j->img;
    t->total_bytes += raw_bytes;  // serialized bytes added as encoded
  }

  if (cfg_.strategy != TS_STRATEGY_LAZY || cfg_.lazy_serialize_overlap) {
    for (size_t k = 0; k < j->sobjs.size(); ++k) workers_->submit(guarded(j, [this, j, k] { serialize_task(j, k); }));
  }
}

int64_t engine::pre_update_barrier(const std::shared_ptr<ticket_state>& t, cudaStream_t opt_stream,
                                   int host_block) {
  if (!t || cfg_.strategy != TS_STRATEGY_LAZY) return 0;
  const int64_t t0 = now_ns();
  if (host_block == 2) {  // exact reference semantics: wait_snapshot (transfer.cpp:114-120)
    t->wait_until([&] { return t->snapshot; });
    const int64_t dt = now_ns() - t0;
    std::lock_guard<std::mutex> g(t->mu);
    t->barrier_block_ns += dt;
    return dt;
  }
  t->wait_until([&] { return t->capture_recorded; });
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  if (host_block) {
    cuda_check(cudaEventSynchronize(t->ev_capture), "barrier: cudaEventSynchronize");
  } else {
    cuda_check(cudaStreamWaitEvent(opt_stream, t->ev_capture, 0), "barrier: cudaStreamWaitEvent");
  }
  const int64_t dt = now_ns() - t0;
  std::lock_guard<std::mutex> g(t->mu);
  if (host_block && t->t_captured < 0) t->t_captured = now_ns() - t->t_issue;
  t->barrier_block_ns += dt;
  return dt;
}

// --- copier: enqueues the device side of each job -------------------------

void engine::copier_loop() {
  cudaSetDevice(device_);
  numa_bind_thread(numa_);
  std::vector<std::shared_ptr<job>> retired;
  for (;;) {
    std::shared_ptr<job> j;
    {
      std::unique_lock<std::mutex> g(mu_);
      cv_.wait(g, [&] { return stopping_ || !jobs_.empty(); });
      if (jobs_.empty()) return;
      j = jobs_.front();
      jobs_.pop_front();
      retired.swap(retired_);
    }
    retired.clear();  // (outside the lock)
    try {
      if (j->deferred) {
        try {
          prepare(j, j->rank, j->descs.data(), j->descs.size());
        } catch (const error& e) {  // (issue-time errors of the reference's issue: not "staging")
          j->t->fail(e.status, e.what(), e.object_id);
          throw;
        } catch (const std::exception& e) {
          j->t->fail(TS_ERR_GENERIC, e.what());
          throw;
        }
      }
      run_job(j);
    } catch (const error& e) {
      j->t->fail(e.status, std::string("staging failed: ") + e.what(), e.object_id);
    } catch (const std::exception& e) {
      j->t->fail(TS_ERR_GENERIC, std::string("staging failed: ") + e.what());
    }
    {
      std::lock_guard<std::mutex> g(j->mu);
      j->enqueue_done = true;
    }
    // The capture event must exist even on failure so barriers do not hang.
    {
      std::lock_guard<std::mutex> g(j->t->mu);
      if (!j->t->capture_recorded) {
        if (j->lane_ev1) cudaStreamWaitEvent(pack_stream_, j->lane_ev1, 0);
        cudaEventRecord(j->t->ev_capture, pack_stream_);
        j->t->capture_recorded = true;
      }
    }
    j->t->cv.notify_all();
    check_snapshot(j);
    for (size_t f = 0; f < j->files.size(); ++f) file_progress(j, f);
  }
}

void engine::run_job(const std::shared_ptr<job>& j) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  auto& t = *j->t;
  const int mode = cfg_.d2h_mode == TS_D2H_HYBRID ? TS_D2H_RING : cfg_.d2h_mode;
  TRACE("run_job rank=%d mode=%d img=%llu wins=%zu segs=%zu", j->rank_id, mode, (unsigned long long)j->img,
        j->wins.size(), j->segs.size());
  const int64_t timeout = cfg_.cache_acquire_timeout_ns;
  const int ctas = cfg_.pack_ctas > 0 ? cfg_.pack_ctas : sms_ * 2;
  const int threads = cfg_.pack_threads > 0 ? cfg_.pack_threads : 512;
  auto mark_capture = [&](cudaStream_t st) {
    cuda_check(cudaEventRecord(t.ev_capture, st), "cudaEventRecord(capture)");
    {
      std::lock_guard<std::mutex> g(t.mu);
      t.capture_recorded = true;
    }
    t.cv.notify_all();
  };
  auto push_window = [&](size_t w) {
    {
      std::lock_guard<std::mutex> g(mu_);
      inflight_.push_back({j, w});
    }
    cv_.notify_all();
    std::lock_guard<std::mutex> g(j->mu);
    j->wins_enqueued += 1;
  };
  auto acquire = [&](job::win& w) {
    if (w.dma) {  // lands in the file's locked pages: no pool region
      t.file_dma_bytes += w.hi - w.lo;
    } else {
      w.r = pool_->acquire(w.hi - w.lo, timeout >= 0 ? now_ns() + timeout : -1);
      w.host = pool_->data(w.r);
    }
    w.ev = get_event();
  };
  auto failed = [&] {
    std::lock_guard<std::mutex> g(t.mu);
    return t.failed;
  };
  // Bounded enqueue: at most `max_inflight` windows between enqueue and
  // landing (~8 GiB, 8-256 windows). An unbounded burst of copies fills the
  // copy stream's queue, after which every cudaMemcpyAsync blocks inside the
  // driver for a window's transfer time — and the training thread's own CUDA
  // calls (event records, graph launches) stall behind it (measured: 35 ms
  // mean, up to 494 ms per call on cfg4). Waiting here instead keeps the
  // driver free.
  const size_t max_inflight = std::clamp<size_t>(
      static_cast<size_t>((8ull << 30) / std::max<uint64_t>(j->win_bytes, 1)), 8, 256);
  auto throttle = [&] {
    std::unique_lock<std::mutex> g(j->mu);
    while (j->wins_enqueued >= j->wins_landed + max_inflight) {
      g.unlock();
      if (failed()) return;
      g.lock();
      j->land_cv.wait_for(g, std::chrono::milliseconds(20));
    }
  };

  // Device staging plan (RING): the whole image when it fits (device shadow);
  // else a ring of `nslots` chunks of whole windows (>= 1 GiB each when the
  // ring allows), packs running ahead of the copies, so the capture completes
  // once all but the last ring-full of the image has left the device.
  const uint64_t W = j->win_bytes;
  uint64_t chunk = 0;
  size_t nslots = 0, nchunks = 0;
  uint8_t* ring = nullptr;
  if (mode == TS_D2H_RING && j->img > 0) {
    // (a whole number of bulk jobs, so the TMA path can run on a full shadow too)
    const uint64_t want = align_up(j->img, cfg_.pack_kernel >= 1 ? static_cast<uint64_t>(dev::kBulkJob) : 256);
    const uint64_t cap = std::max<uint64_t>(cfg_.device_staging_bytes, 2 * W);
    if (cap >= want) {
      chunk = want;
      nslots = 1;
    } else {
      // Few large chunks: every pack launch after the first ring-full waits
      // for a free slot and then interrupts the training kernels once (at
      // high priority), so fewer, larger launches interfere less.
      const uint64_t want_chunk = cfg_.ring_chunk_bytes ? cfg_.ring_chunk_bytes
                                                        : std::min<uint64_t>(8ull << 30, cap / 6);
      chunk = std::max<uint64_t>(W, std::min<uint64_t>(want_chunk, cap / 2) / W * W);
      nslots = static_cast<size_t>(cap / chunk);
    }
    nchunks = (j->img + chunk - 1) / chunk;
    ring = ensure_device_ring(nslots == 1 ? want : nslots * chunk);
  }
  const bool use_ring = ring != nullptr;
  // HYBRID (multi-slot ring): only the last ring-full is packed — into its
  // own slots, at issue; the head chunks [0, H) leave the device straight
  // from the state by copy-engine DMA per fragment piece. The capture
  // completes at the same point as with the ring (all but the last ring-full
  // has left the device) but the SMs pack a ring-full instead of the image.
  // Only for large fragments: the head costs one DMA per fragment piece
  // (hybrid_direct_min_bytes: the least mean piece size, default 1 MiB).
  size_t H = (cfg_.d2h_mode == TS_D2H_HYBRID && use_ring && nslots > 1 && nchunks > nslots) ? nchunks - nslots : 0;
  if (H) {
    uint64_t hb = 0, np = 0;
    for (const auto& sg : j->segs) {
      if (sg.pos >= H * chunk) break;
      if (!sg.src) continue;
      hb += std::min<uint64_t>(sg.len, H * chunk - sg.pos);
      ++np;
    }
    if (np == 0 || hb / np < cfg_.hybrid_direct_min_bytes) H = 0;
  }
  auto slot_of = [&](size_t c) -> uint8_t* { return ring + (nslots == 1 ? 0 : ((c - H) % nslots) * chunk); };

  // TMA bulk jobs (pack_kernel = 1, RING only): large 16-B aligned device
  // fragments are cut at absolute kBulkJob boundaries of the image (so no job
  // straddles a ring chunk); the warp kernel skips those bytes.
  std::vector<dev::seg> wsegs;
  std::vector<dev::bulk_job> bjobs;
  const std::vector<dev::seg>* segs_for_warp = &j->segs;
  // (chunks must be kBulkJob multiples so that no job straddles two ring slots;
  // with odd window sizes the warp kernel does everything)
  // Only for a full device shadow (one pack of the whole image): in a ring of
  // slots every chunk's pack is issued while training kernels run, and the
  // bulk kernel's CTAs (192 KiB of shared memory each) then wait for whole SMs
  // — measured: cfg4 with a ring, 22 % step slowdown with bulk vs 4 % warp.
  // pack_kernel = 2 keeps the bulk path in a multi-slot ring with a 2-stage
  // (64 KiB) kernel, small enough to share an SM with training CTAs that leave
  // 64 KiB of shared memory free.
  const bool bulk_ring = cfg_.pack_kernel == 2 && nslots > 1;
  if (use_ring && ((nslots == 1 && cfg_.pack_kernel >= 1) || bulk_ring) && chunk % dev::kBulkJob == 0) {
    for (const auto& sg : j->segs) {
      const uint64_t body = sg.len & ~15ull;
      const bool bulk = sg.src && (reinterpret_cast<uintptr_t>(sg.src) & 15) == 0 && (sg.pos & 15) == 0 &&
                        body >= std::max<uint64_t>(cfg_.bulk_min_bytes, dev::kBulkJob);
      if (!bulk) {
        wsegs.push_back(sg);
        continue;
      }
      wsegs.push_back({sg.pos, body, TSB_BULK_SRC});
      if (sg.len > body) wsegs.push_back({sg.pos + body, sg.len - body, sg.src + body});
      for (uint64_t a = sg.pos; a < sg.pos + body;) {
        const uint64_t b = std::min(sg.pos + body, (a / dev::kBulkJob + 1) * dev::kBulkJob);
        bjobs.push_back({a, sg.src + (a - sg.pos), b - a});
        a = b;
      }
    }
    segs_for_warp = &wsegs;
  }
  dev::seg* d_segs = nullptr;
  dev::bulk_job* d_jobs = nullptr;
  if (j->img > 0 && mode != TS_D2H_DIRECT) {
    const uint64_t sb = align_up(segs_for_warp->size() * sizeof(dev::seg), 256);
    uint8_t* tb = static_cast<uint8_t*>(ensure_seg_buffer(sb + bjobs.size() * sizeof(dev::bulk_job)));
    d_segs = reinterpret_cast<dev::seg*>(tb);
    d_jobs = reinterpret_cast<dev::bulk_job*>(tb + sb);
    // Upload before waiting on the producer (a pageable H2D syncs its stream).
    cuda_check(cudaMemcpyAsync(d_segs, segs_for_warp->data(), segs_for_warp->size() * sizeof(dev::seg),
                               cudaMemcpyHostToDevice, pack_stream_), "upload segment table");
    if (!bjobs.empty())
      cuda_check(cudaMemcpyAsync(d_jobs, bjobs.data(), bjobs.size() * sizeof(dev::bulk_job), cudaMemcpyHostToDevice,
                                 pack_stream_), "upload bulk jobs");
  }
  // Device checksums. RING: per chunk over the ring slot right after its pack
  // (chained states, off the capture path). DIRECT / ZEROCOPY: over the state
  // itself before the capture completes. Table: one entry per (chunk, object
  // piece), grouped by chunk; launch k covers entries [cbeg[k], cbeg[k+1]).
  const uint32_t nf = static_cast<uint32_t>(j->fnv_objs.size());
  uint8_t* fbuf = nullptr;
  uint64_t ftb = 0, fsb = 0, lane_off = 0;
  std::vector<dev::fnv_obj> fo;
  std::vector<size_t> cbeg;
  std::vector<std::pair<uint64_t, uint64_t>> cdims;  // (nseg, nchunk) per launch
  // Lane-serial checksums (RING): objects one lane hashes well within the
  // capture time are hashed from the state itself at ~7 integer ops per byte
  // (a few warps, most of the D2H long) instead of by the speculating
  // segment-parallel kernels over the ring slots (~26 ops per byte).
  std::vector<char> lane_q;
  std::vector<dev::fnv_lane_obj> lanes;
  uint64_t lane_bytes = 0;
  if (nf && use_ring) {
    uint64_t lane_max = 0;
    if (cfg_.checksum_lane_max_bytes > 0) {
      lane_max = static_cast<uint64_t>(cfg_.checksum_lane_max_bytes);
    } else if (cfg_.checksum_lane_max_bytes < 0 && nslots > 1) {
      // the capture completes once all but the last ring-full has left the
      // device over PCIe (>= 50 GB/s): a lane gets 40 % of that time
      const double cap_s = static_cast<double>(j->img - std::min<uint64_t>(j->img, nslots * chunk)) / 50e9;
      lane_max = static_cast<uint64_t>(0.4 * kLaneBytesPerS * cap_s);
    }
    if (lane_max) {
      lane_q.assign(nf, 0);
      for (uint32_t q = 0; q < nf; ++q) {
        const auto& r = j->raws[j->fnv_objs[q]];
        if (r.size > lane_max) continue;
        lane_q[q] = 1;
        lanes.push_back({r.src, r.size, fnv_seed, q});
        lane_bytes += r.size;
      }
      // longest first: the lanes of a warp finish together
      std::stable_sort(lanes.begin(), lanes.end(),
                       [](const dev::fnv_lane_obj& a, const dev::fnv_lane_obj& b) { return a.len > b.len; });
    }
  }
  if (nf) {
    if (use_ring) {
      size_t k = 0;  // fnv_objs are in image order
      for (size_t c = 0; c < nchunks; ++c) {
        cbeg.push_back(fo.size());
        const uint64_t clo = c * chunk, chi = std::min(j->img, clo + chunk);
        while (k < nf && j->raws[j->fnv_objs[k]].img + j->raws[j->fnv_objs[k]].size <= clo) ++k;
        for (size_t q = k; q < nf && j->raws[j->fnv_objs[q]].img < chi; ++q) {
          if (!lane_q.empty() && lane_q[q]) continue;
          const auto& r = j->raws[j->fnv_objs[q]];
          const uint64_t a = std::max(clo, r.img), b = std::min(chi, r.img + r.size);
          // (head chunks of HYBRID: checksums over the state itself)
          fo.push_back({c < H ? r.src + (a - r.img) : slot_of(c) + (a - clo), b - a, 0, 0, q});
        }
      }
      cbeg.push_back(fo.size());
    } else {
      for (uint32_t q = 0; q < nf; ++q) {
        const auto& r = j->raws[j->fnv_objs[q]];
        fo.push_back({r.src, r.size, 0, 0, q});
      }
      cbeg = {0, fo.size()};
    }
    uint64_t max_scratch = 0;
    for (size_t k = 0; k + 1 < cbeg.size(); ++k) {
      uint64_t nch = 0;
      const uint32_t cnt = static_cast<uint32_t>(cbeg[k + 1] - cbeg[k]);
      const uint64_t nseg = dev::fnv_prepare(fo.data() + cbeg[k], cnt, &nch);
      cdims.push_back({nseg, nch});
      max_scratch = std::max(max_scratch, dev::fnv_scratch_bytes(nseg, nch, cnt));
    }
    ftb = align_up(fo.size() * sizeof(dev::fnv_obj), 256);
    fsb = align_up(nf * 8ull, 256);
    lane_off = ftb + fsb + align_up(max_scratch, 256);
    fbuf = ensure_fnv_buffer(lane_off + lanes.size() * sizeof(dev::fnv_lane_obj));
    std::vector<uint64_t> seeds(nf, fnv_seed);
    if (!fo.empty())  // (empty when the lane kernel takes every object)
      cuda_check(cudaMemcpyAsync(fbuf, fo.data(), fo.size() * sizeof(dev::fnv_obj), cudaMemcpyHostToDevice,
                                 pack_stream_), "upload checksum table");
    cuda_check(cudaMemcpyAsync(fbuf + ftb, seeds.data(), nf * 8ull, cudaMemcpyHostToDevice, pack_stream_),
               "upload checksum seeds");
    if (!lanes.empty())
      cuda_check(cudaMemcpyAsync(fbuf + lane_off, lanes.data(), lanes.size() * sizeof(dev::fnv_lane_obj),
                                 cudaMemcpyHostToDevice, pack_stream_),
                 "upload lane checksum table");
    if (ck_host_n_ < nf) {  // the previous job's results were consumed before its snapshot completed
      // (sized for every device-tier object, so a growing GPU share does not
      // reallocate: cudaFreeHost synchronizes the device)
      uint32_t ndev = 0;
      for (const auto& r : j->raws) ndev += r.device ? 1 : 0;
      if (ck_host_) cudaFreeHost(ck_host_);
      ck_host_ = nullptr;
      const uint32_t cap = std::max(nf, ndev);
      cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&ck_host_), cap * 8ull, cudaHostAllocMapped | cudaHostAllocPortable),
                 "cudaHostAlloc(checksums)");
      ck_host_n_ = cap;
    }
    j->fnv_out = ck_host_;
    j->fnv_ev = get_event();
  }
  bool fnv_publish = false;
  auto publish_fnv = [&] {
    {
      std::lock_guard<std::mutex> g(mu_);
      inflight_.push_back({j, 0, true});
    }
    cv_.notify_all();
  };
  // Launch k of the checksum kernels; the last one publishes the results
  // straight into the mapped pool region (a cudaMemcpy would queue behind the
  // bulk D2H windows on the copy engine).
  auto launch_checksums = [&](size_t k, cudaStream_t cs) {
    if (!nf || cbeg[k + 1] == cbeg[k]) {
      if (nf && k + 2 == cbeg.size()) goto publish;
      return;
    }
    {
      uint64_t* out = nullptr;
      cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&out), j->fnv_out, 0), "cudaHostGetDevicePointer");
      dev::launch_fnv(reinterpret_cast<dev::fnv_obj*>(fbuf) + cbeg[k], static_cast<uint32_t>(cbeg[k + 1] - cbeg[k]),
                      cdims[k].first, cdims[k].second, reinterpret_cast<uint64_t*>(fbuf + ftb), fbuf + ftb + fsb,
                      cs, out);
      t.kernel_launches += 11;
      cuda_check(cudaGetLastError(), "checksum kernels");
    }
    if (k + 2 != cbeg.size()) return;
  publish:
    if (j->lane_ev1) cuda_check(cudaStreamWaitEvent(cs, j->lane_ev1, 0), "wait lane checksums");
    cuda_check(cudaEventRecord(j->fnv_ev, cs), "event");
    // RING: the completer learns about the results only after the last
    // window, so it never blocks on the checksums ahead of windows whose
    // landing the bounded enqueue is waiting for
    // (DIRECT / ZEROCOPY publish once the copy stream waits on the event:
    // the completer recycles fnv_ev as soon as it has synchronized on it)
    fnv_publish = true;
  };
  cuda_check(cudaStreamWaitEvent(pack_stream_, t.ev_start, 0), "wait producer");
  cuda_check(cudaStreamWaitEvent(copy_stream_, t.ev_start, 0), "wait producer");
  cuda_check(cudaEventRecord(t.ev_pack0, mode == TS_D2H_DIRECT ? copy_stream_ : pack_stream_), "event");
  if (!lanes.empty()) {  // tables uploaded and the producer done: start hashing the state
    cudaEvent_t ready;
    cuda_check(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(ready, pack_stream_), "event");
    cuda_check(cudaStreamWaitEvent(ck_lane_stream_, ready, 0), "lane checksums wait");
    cudaEventDestroy(ready);
    cuda_check(cudaEventCreate(&j->lane_ev0), "event");
    cuda_check(cudaEventCreate(&j->lane_ev1), "event");
    uint64_t* out = nullptr;
    cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&out), j->fnv_out, 0), "cudaHostGetDevicePointer");
    cuda_check(cudaEventRecord(j->lane_ev0, ck_lane_stream_), "event");
    dev::launch_fnv_lanes(reinterpret_cast<dev::fnv_lane_obj*>(fbuf + lane_off), static_cast<uint32_t>(lanes.size()),
                          out, ck_lane_stream_);
    cuda_check(cudaGetLastError(), "lane checksum kernel");
    cuda_check(cudaEventRecord(j->lane_ev1, ck_lane_stream_), "event");
    t.kernel_launches += 1;
    t.lane_checksum_bytes = lane_bytes;
  }
  if (nf && !use_ring) {
    launch_checksums(0, pack_stream_);
    // DIRECT captures on the copy stream: it must also cover the checksum reads.
    cuda_check(cudaStreamWaitEvent(copy_stream_, j->fnv_ev, 0), "wait checksums");
    publish_fnv();
    fnv_publish = false;
  }
  if (j->img == 0) {
    mark_capture(pack_stream_);
    return;
  }
  const uint32_t nsegs = static_cast<uint32_t>(segs_for_warp->size());

  if (mode == TS_D2H_RING) {
    const bool shadow = nslots == 1;
    int64_t copy_call_ns = 0, copy_call_max_ns = 0;
    const int64_t t_enqueue0 = now_ns();
    j->chunk_events.assign(nchunks, nullptr);
    j->ck_events.assign(nchunks, nullptr);
    uint64_t seen_bytes = 0, helper_done = 0;
    size_t helper_next = 0;
    // Windows of each chunk, in D2H order: [cw0[c], cw0[c + 1]) (a shadow is one chunk).
    std::vector<size_t> cw0(nchunks + 1, j->wins.size());
    for (size_t c = 0, q = 0; c < nchunks; ++c) {
      cw0[c] = q;
      const uint64_t chi = std::min(j->img, (c + 1) * chunk);
      while (q < j->wins.size() && (shadow || j->wins[q].lo < chi)) ++q;
    }
    std::vector<cudaEvent_t> packed_ev(nchunks, nullptr);
    cuda_check(cudaEventRecord(t.ev_d2h_first, copy_stream_), "event");

    // Device checksums of chunk c over its ring slot, on the checksum stream,
    // overlapping the D2H.
    auto enqueue_checksums = [&](size_t c) {
      {
        // chunks whose slot is packed again in this job: capture path, pack
        // priority; the last ring-full: low priority (chained states keep the
        // launches in chunk order across the two streams)
        const bool reused = c + nslots < nchunks;
        cudaStream_t cs = reused ? ck_hi_stream_ : ck_stream_;
        if (!reused && c > 0 && c - 1 + nslots < nchunks) {  // first low-priority chunk after high ones
          cudaEvent_t hand;
          cuda_check(cudaEventCreateWithFlags(&hand, cudaEventDisableTiming), "event");
          cuda_check(cudaEventRecord(hand, ck_hi_stream_), "event");
          cuda_check(cudaStreamWaitEvent(ck_stream_, hand, 0), "checksum order");
          cudaEventDestroy(hand);
        }
        cuda_check(cudaStreamWaitEvent(cs, packed_ev[c], 0), "wait pack");
        launch_checksums(c, cs);
        cudaEvent_t ck;
        cuda_check(cudaEventCreateWithFlags(&ck, cudaEventDisableTiming), "event");
        cuda_check(cudaEventRecord(ck, cs), "event");
        j->ck_events[c] = ck;
      }
    };

    // Pack of chunk c (+ its host-tier bytes and device checksums). Enqueued as
    // soon as the slot's previous chunk has its D2H and checksums enqueued, so
    // packs run up to a ring-full ahead of the window copies; the GPU-side
    // waits order them after the slot is free.
    auto enqueue_pack = [&](size_t c) {
      const uint64_t clo = c * chunk, chi = std::min(j->img, clo + chunk);
      uint8_t* slot = slot_of(c);
      if (c >= nslots + H) {  // the slot's previous chunk must have left the device and been checksummed
        cuda_check(cudaStreamWaitEvent(pack_stream_, j->chunk_events[c - nslots], 0), "slot wait");
        if (nf) cuda_check(cudaStreamWaitEvent(pack_stream_, j->ck_events[c - nslots], 0), "slot wait");
      }
      // Packs and the previous chunk's pack-priority checksums take turns on
      // the SMs instead of splitting them (same total work; a pack that
      // shares the GPU with FNV kernels runs at 0.80 instead of 0.91 of the
      // HBM roofline). Low-priority checksums (the last ring-full) are never
      // waited for here: they must not delay the capture.
      if (nf && c > H && c - 1 + nslots < nchunks && j->ck_events[c - 1])
        cuda_check(cudaStreamWaitEvent(pack_stream_, j->ck_events[c - 1], 0), "pack after checksums");
      cudaEvent_t pa, pb;
      cuda_check(cudaEventCreate(&pa), "event");
      cuda_check(cudaEventCreate(&pb), "event");
      cuda_check(cudaEventRecord(pa, pack_stream_), "event");
      dev::launch_pack(d_segs, nsegs, clo, chi, slot, ctas, threads, pack_stream_);
      t.kernel_launches += 1;
      if (!bjobs.empty()) {
        auto lb = std::lower_bound(bjobs.begin(), bjobs.end(), clo,
                                   [](const dev::bulk_job& b, uint64_t x) { return b.pos < x; });
        auto ub = std::lower_bound(lb, bjobs.end(), chi, [](const dev::bulk_job& b, uint64_t x) { return b.pos < x; });
        if (ub > lb) {
          dev::launch_pack_bulk(d_jobs + (lb - bjobs.begin()), static_cast<uint32_t>(ub - lb), clo, slot,
                                bulk_ring ? 3 * sms_ : sms_, pack_stream_, bulk_ring ? 2 : 6);
          t.kernel_launches += 1;
        }
      }
      cuda_check(cudaEventRecord(pb, pack_stream_), "event");
      j->pack_events.push_back({pa, pb});
      // Host-tier bytes join the staged image in stream order, before the
      // capture event: the pre-update barrier then covers them too (copying
      // them at window landing, after the barrier, let an update leak in).
      for (size_t q = cw0[c]; q < cw0[c + 1]; ++q) {
        const auto& wq = j->wins[shadow ? j->worder[q] : q];
        for (uint32_t k = wq.hp_begin; k < wq.hp_end; ++k)
          cuda_check(cudaMemcpyAsync(slot + (wq.lo + j->hp[k].win_off - clo), j->hp[k].src, j->hp[k].len,
                                     cudaMemcpyHostToDevice, pack_stream_), "host-tier bytes to the staged image");
      }
      cuda_check(cudaGetLastError(), "pack kernel launch");
      cuda_check(cudaEventCreateWithFlags(&packed_ev[c], cudaEventDisableTiming), "event");
      cuda_check(cudaEventRecord(packed_ev[c], pack_stream_), "event");
      if (c + 1 == nchunks && H == 0) {  // (HYBRID: after the head's copies, below)
        // the lane checksums read the state: the capture covers them
        if (j->lane_ev1) cuda_check(cudaStreamWaitEvent(pack_stream_, j->lane_ev1, 0), "capture after lanes");
        mark_capture(pack_stream_);
      }
      if (nf && !(H && c >= H)) enqueue_checksums(c);
    };

    size_t next_pack = 0;
    t.packed_bytes = j->img - std::min<uint64_t>(j->img, H * chunk);
    if (H) {
      // HYBRID: the last ring-full is packed at once; then the head's
      // checksums over the state (the capture waits for them: pack priority;
      // after the packs, not beside them: a pack sharing the SMs with FNV
      // kernels runs at ~0.55 instead of ~0.9 of the HBM roofline), then the
      // tail's checksums over its slots (low priority, chained after the head).
      for (size_t c = H; c < nchunks; ++c) enqueue_pack(c);
      next_pack = nchunks;
      if (nf) {
        cudaEvent_t ready;
        cuda_check(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event");
        cuda_check(cudaEventRecord(ready, pack_stream_), "event");  // tables uploaded, producer done, tail packed
        cuda_check(cudaStreamWaitEvent(ck_hi_stream_, ready, 0), "head checksums wait");
        cudaEventDestroy(ready);
        for (size_t c = 0; c < H; ++c) {
          launch_checksums(c, ck_hi_stream_);
          cudaEvent_t ck;
          cuda_check(cudaEventCreateWithFlags(&ck, cudaEventDisableTiming), "event");
          cuda_check(cudaEventRecord(ck, ck_hi_stream_), "event");
          j->ck_events[c] = ck;
        }
        for (size_t c = H; c < nchunks; ++c) enqueue_checksums(c);
      }
    }
    for (size_t c = 0; c < nchunks && !failed(); ++c) {
      while (next_pack < nchunks && (next_pack < nslots || j->chunk_events[next_pack - nslots] != nullptr))
        enqueue_pack(next_pack++);
      if (c < H) {  // HYBRID head: copy-engine DMA per fragment piece, gaps zeroed on the host
        for (size_t q = cw0[c]; q < cw0[c + 1] && !failed(); ++q) {
          auto& win = j->wins[q];
          throttle();
          acquire(win);
          uint8_t* dst = win.host;
          size_t k = std::upper_bound(j->segs.begin(), j->segs.end(), win.lo,
                                      [](uint64_t x, const dev::seg& sg) { return x < sg.pos; }) - j->segs.begin();
          k = k ? k - 1 : 0;
          for (size_t qq = k; qq < j->segs.size() && j->segs[qq].pos < win.hi; ++qq) {
            const auto& sg = j->segs[qq];
            const uint64_t a = std::max(win.lo, sg.pos), b = std::min(win.hi, sg.pos + sg.len);
            if (b <= a) continue;
            if (sg.src) {
              cuda_check(cudaMemcpyAsync(dst + (a - win.lo), sg.src + (a - sg.pos), b - a, cudaMemcpyDeviceToHost,
                                         copy_stream_), "D2H fragment");
              t.copies += 1;
            } else {
              std::memset(dst + (a - win.lo), 0, b - a);
            }
          }
          for (uint32_t hk = win.hp_begin; hk < win.hp_end; ++hk)  // host-tier bytes, in stream order (capture)
            cuda_check(cudaMemcpyAsync(dst + j->hp[hk].win_off, j->hp[hk].src, j->hp[hk].len,
                                       cudaMemcpyHostToHost, copy_stream_), "host-tier bytes to the window");
          seen_bytes += win.hi - win.lo;
          cuda_check(cudaEventRecord(win.ev, copy_stream_), "event");
          push_window(q);
        }
        cudaEvent_t done;
        cuda_check(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event");
        cuda_check(cudaEventRecord(done, copy_stream_), "event");
        j->chunk_events[c] = done;
        if (c + 1 == H) {  // the state may change once the head has left and the tail is packed
          cuda_check(cudaStreamWaitEvent(pack_stream_, done, 0), "capture after the head");
          if (nf) cuda_check(cudaStreamWaitEvent(pack_stream_, j->ck_events[H - 1], 0), "capture after the head");
          if (j->lane_ev1) cuda_check(cudaStreamWaitEvent(pack_stream_, j->lane_ev1, 0), "capture after lanes");
          mark_capture(pack_stream_);
        }
        continue;
      }
      const uint64_t clo = c * chunk;
      uint8_t* slot = slot_of(c);
      cuda_check(cudaStreamWaitEvent(copy_stream_, packed_ev[c], 0), "wait pack");
      std::vector<char> helper_used(helpers_.size(), 0);
      for (size_t q = cw0[c]; q < cw0[c + 1]; ++q) {
        const size_t wi = shadow ? j->worder[q] : q;
        auto& win = j->wins[wi];
        throttle();
        acquire(win);
        const uint64_t len = win.hi - win.lo;
        cudaStream_t cs = copy_stream_;
        // helper share spread evenly over the image, round robin over helpers
        if (!helpers_.empty() && static_cast<double>(helper_done + len / 2) <
                                     cfg_.helper_share * static_cast<double>(seen_bytes + len)) {
          const size_t k = helper_next++ % helpers_.size();
          put_event(win.ev);
          win.ev = helper_event(k);
          win.helper = static_cast<int>(k);
          cs = helpers_[k]->st;
          if (!helper_used[k]) {  // once per chunk: the helper copies only after the pack
            cuda_check(cudaStreamWaitEvent(cs, packed_ev[c], 0), "helper waits for the pack");
            helper_used[k] = 1;
          }
          helper_done += len;
          t.helper_bytes += len;
        }
        seen_bytes += len;
        const int64_t tc0 = now_ns();
        const cudaError_t ce = cudaMemcpyAsync(win.host, slot + (win.lo - clo), len, cudaMemcpyDeviceToHost, cs);
        {
          const int64_t dt = now_ns() - tc0;
          copy_call_ns += dt;
          copy_call_max_ns = std::max<int64_t>(copy_call_max_ns, dt);
        }
        if (ce != cudaSuccess) {
          char m[256];
          std::snprintf(m, sizeof m, "D2H window [%llu, %llu) of chunk %zu at %llu (ring %llu B, host %p dma %d)",
                        (unsigned long long)win.lo, (unsigned long long)win.hi, c, (unsigned long long)clo,
                        (unsigned long long)ring_bytes_, (void*)win.host, (int)win.dma);
          cuda_check(ce, m);
        }
        t.copies += 1;
        cuda_check(cudaEventRecord(win.ev, cs), "event");
        push_window(wi);
        if (failed()) break;
      }
      for (size_t k = 0; k < helpers_.size(); ++k) {  // the slot is free once the helpers' copies are done
        if (!helper_used[k]) continue;
        cudaEvent_t he = helper_event(k);
        cuda_check(cudaEventRecord(he, helpers_[k]->st), "event");
        cuda_check(cudaStreamWaitEvent(copy_stream_, he, 0), "wait helper copies");
        put_helper_event(k, he);  // (re-recorded only after this wait was enqueued)
      }
      cudaEvent_t done;
      cuda_check(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event");
      cuda_check(cudaEventRecord(done, copy_stream_), "event");
      j->chunk_events[c] = done;
    }
    for (auto& e : packed_ev)  // (destruction is deferred until each event completes)
      if (e) cudaEventDestroy(e);
    if (fnv_publish) publish_fnv();
    cuda_check(cudaEventRecord(t.ev_d2h_last, copy_stream_), "event");
    if (g_trace_copies)
      std::fprintf(stderr, "[ts] run_job rank=%d windows=%zu: host time in cudaMemcpyAsync %.1f ms (max %.2f ms), "
                   "whole enqueue %.1f ms\n", j->rank_id, j->wins.size(), copy_call_ns / 1e6, copy_call_max_ns / 1e6,
                   (now_ns() - t_enqueue0) / 1e6);
    // later jobs reuse the ring and the checksum scratch: order them after these checksums
    if (nf) {
      cudaEvent_t tail;
      cuda_check(cudaEventCreateWithFlags(&tail, cudaEventDisableTiming), "event");
      cuda_check(cudaEventRecord(tail, ck_stream_), "event");
      cuda_check(cudaStreamWaitEvent(pack_stream_, tail, 0), "wait checksums");
      cudaEventDestroy(tail);
    }
  } else if (mode == TS_D2H_ZEROCOPY) {
    uint8_t* dbase = nullptr;
    cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dbase), pool_->base(), 0),
               "cudaHostGetDevicePointer");
    cuda_check(cudaEventRecord(t.ev_d2h_first, pack_stream_), "event");
    for (size_t q = 0; q < j->wins.size() && !failed(); ++q) {
      const size_t w = j->worder[q];
      auto& win = j->wins[w];
      throttle();
      acquire(win);
      uint8_t* dst = nullptr;  // device view of the mapped pool region / locked file pages
      if (win.dma) {
        const auto& f = j->files[j->fs[win.fs_begin].f];
        cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dst), f.dma, 0), "cudaHostGetDevicePointer");
        dst += win.host - f.dma;
      } else {
        dst = dbase + win.r.offset;
      }
      dev::launch_pack(d_segs, nsegs, win.lo, win.hi, dst, ctas, threads, pack_stream_);
      t.kernel_launches += 1;
      cuda_check(cudaGetLastError(), "pack kernel launch");
      for (uint32_t k = win.hp_begin; k < win.hp_end; ++k)  // host-tier bytes, in stream order (capture)
        cuda_check(cudaMemcpyAsync(win.host + j->hp[k].win_off, j->hp[k].src, j->hp[k].len, cudaMemcpyHostToHost,
                                   pack_stream_), "host-tier bytes to the window");
      cuda_check(cudaEventRecord(win.ev, pack_stream_), "event");
      push_window(w);
    }
    cuda_check(cudaEventRecord(t.ev_d2h_last, pack_stream_), "event");
    mark_capture(pack_stream_);
  } else {  // DIRECT: copy-engine DMA per fragment piece, gaps zeroed on the host
    cuda_check(cudaEventRecord(t.ev_d2h_first, copy_stream_), "event");
    for (size_t q = 0; q < j->wins.size() && !failed(); ++q) {
      const size_t w = j->worder[q];
      auto& win = j->wins[w];
      throttle();
      acquire(win);
      uint8_t* dst = win.host;
      size_t k = std::upper_bound(j->segs.begin(), j->segs.end(), win.lo,
                                  [](uint64_t x, const dev::seg& sg) { return x < sg.pos; }) - j->segs.begin();
      k = k ? k - 1 : 0;
      for (size_t qq = k; qq < j->segs.size() && j->segs[qq].pos < win.hi; ++qq) {
        const auto& sg = j->segs[qq];
        const uint64_t a = std::max(win.lo, sg.pos), b = std::min(win.hi, sg.pos + sg.len);
        if (b <= a) continue;
        if (sg.src) {
          cuda_check(cudaMemcpyAsync(dst + (a - win.lo), sg.src + (a - sg.pos), b - a,
                                     cudaMemcpyDeviceToHost, copy_stream_), "D2H fragment");
          t.copies += 1;
        } else {
          std::memset(dst + (a - win.lo), 0, b - a);
        }
      }
      for (uint32_t k = win.hp_begin; k < win.hp_end; ++k)  // host-tier bytes, in stream order (capture)
        cuda_check(cudaMemcpyAsync(dst + j->hp[k].win_off, j->hp[k].src, j->hp[k].len, cudaMemcpyHostToHost,
                                   copy_stream_), "host-tier bytes to the window");
      cuda_check(cudaEventRecord(win.ev, copy_stream_), "event");
      push_window(w);
    }
    cuda_check(cudaEventRecord(t.ev_d2h_last, copy_stream_), "event");
    mark_capture(copy_stream_);
  }
}

// --- completer: observes window completions in order ----------------------

void engine::completer_loop() {
  cudaSetDevice(device_);
  numa_bind_thread(numa_);
  for (;;) {
    pending_window pw;
    {
      std::unique_lock<std::mutex> g(mu_);
      cv_.wait(g, [&] { return !inflight_.empty() || copier_done_; });
      if (inflight_.empty()) return;
      pw = inflight_.front();
      inflight_.pop_front();
    }
    auto& j = pw.j;
    if (pw.fnv) {
      const cudaError_t e = cudaEventSynchronize(j->fnv_ev);
      put_event(j->fnv_ev);
      j->fnv_ev = nullptr;
      if (e != cudaSuccess) {
        j->t->fail(TS_ERR_CUDA, std::string("checksum kernels failed: ") + cudaGetErrorString(e));
        continue;
      }
      fnv_landed(j);
      continue;
    }
    auto& win = j->wins[pw.w];
    const cudaError_t e = cudaEventSynchronize(win.ev);
    if (win.helper >= 0) put_helper_event(static_cast<size_t>(win.helper), win.ev);
    else put_event(win.ev);
    win.ev = nullptr;
    if (e != cudaSuccess) {
      j->t->fail(TS_ERR_CUDA, std::string("staging failed: ") + cudaGetErrorString(e));
      {
        std::lock_guard<std::mutex> g(j->mu);
        j->wins_landed += 1;
      }
      j->land_cv.notify_all();
      if (!win.dma) pool_->release(win.r);
      continue;
    }
    {
      std::lock_guard<std::mutex> g(j->t->mu);
      if (j->t->t_captured < 0 && j->t->capture_recorded && cudaEventQuery(j->t->ev_capture) == cudaSuccess)
        j->t->t_captured = now_ns() - j->t->t_issue;
    }
    window_landed(j, pw.w);
  }
}

void engine::window_landed(const std::shared_ptr<job>& j, size_t wi) {
  auto& w = j->wins[wi];
  TRACE("landed rank=%d w=%zu pieces=%u fsegs=%u", j->rank_id, wi, w.wp_end - w.wp_begin, w.fs_end - w.fs_begin);
  // (host-tier bytes are already in the window: copied in stream order as part
  // of the capture, never here after the barrier)
  uint8_t* base = w.host;
  size_t newly_ready = 0;
  bool release_now = false;
  {
    std::lock_guard<std::mutex> g(j->mu);
    // a pool window holds one reference for its flush; a dma window is already in the file
    w.refs = (j->io && !w.dma && w.fs_end > w.fs_begin) ? 1 : 0;
    if (j->io && w.dma)
      for (uint32_t k = w.fs_begin; k < w.fs_end; ++k) j->files[j->fs[k].f].win_pending -= 1;
    for (uint32_t k = w.wp_begin; k < w.wp_end; ++k) {
      auto& r = j->raws[j->wp[k].obj];
      if (r.gpu_ck) continue;  // checksummed on the device
      w.refs += 1;
      r.q.push_back({base + j->wp[k].win_off, j->wp[k].len, static_cast<uint32_t>(wi)});
      if (!r.busy && !r.queued) {
        r.queued = true;
        j->ready.push_back(j->wp[k].obj);
        ++newly_ready;
      }
    }
    j->wins_landed += 1;
    release_now = w.refs == 0;
  }
  j->land_cv.notify_all();
  if (release_now && !w.dma) pool_->release(w.r);
  bool last;
  {
    std::lock_guard<std::mutex> g(j->mu);
    last = j->wins_landed == j->wins.size();
    if (last) j->t_landed_all = now_ns();
  }
  if (last)
    for (size_t f = 0; f < j->files.size(); ++f) file_progress(j, f);
  else if (j->io && w.dma)
    for (uint32_t k = w.fs_begin; k < w.fs_end; ++k) file_progress(j, j->fs[k].f);
  if (!j->defer_hash) {
    for (size_t k = 0; k < (newly_ready + 3) / 4; ++k)
      workers_->submit(guarded(j, [this, j] { hash_task(j, 0); }));
  } else if (last) {  // deferred: every worker drains the ready objects, 4 chains each
    for (int k = 0; k < workers_->size(); ++k) workers_->submit(guarded(j, [this, j] { hash_task(j, 0); }));
  }
  if (j->io && !w.dma && w.fs_end > w.fs_begin)
    workers_->submit(guarded(j, [this, j, wi] { flush_window(j, wi); }));
  check_snapshot(j);
}

// Device checksums of every device-tier raw object landed (transfer.cpp:71-83's
// per-object FNV, computed by the FNV kernels instead of the staging thread).
void engine::fnv_landed(const std::shared_ptr<job>& j) {
  const uint64_t* res = j->fnv_out;
  {
    std::lock_guard<std::mutex> g(j->t->mu);
    for (size_t i = 0; i < j->fnv_objs.size(); ++i) j->t->checksums[j->raws[j->fnv_objs[i]].oid] = res[i];
  }
  {
    std::lock_guard<std::mutex> g(j->mu);
    for (uint32_t k : j->fnv_objs) {
      j->raws[k].hashed = j->raws[k].size;
      j->files[j->raws[k].f].raw_pending -= 1;
    }
  }
  TRACE("checksums landed rank=%d objects=%zu", j->rank_id, j->fnv_objs.size());
  for (size_t f = 0; f < j->files.size(); ++f) file_progress(j, f);
}

void engine::window_release_ref(const std::shared_ptr<job>& j, size_t wi) {
  bool rel;
  {
    std::lock_guard<std::mutex> g(j->mu);
    rel = --j->wins[wi].refs == 0;
  }
  if (rel && !j->wins[wi].dma) pool_->release(j->wins[wi].r);
}

namespace {
// Advances k (1..4) independent FNV-1a chains by n bytes each, in lock-step:
// one chain is a 64-bit multiply latency chain (~4 cycles/byte); four give the
// core instruction-level parallelism.
void fnv_lockstep(const uint8_t* const* p, uint64_t* h, int k, uint64_t n) {
  switch (k) {
    case 4: {
      uint64_t a = h[0], b = h[1], c = h[2], d = h[3];
      const uint8_t *pa = p[0], *pb = p[1], *pc = p[2], *pd = p[3];
      for (uint64_t i = 0; i < n; ++i) {
        a = (a ^ pa[i]) * fnv_prime;
        b = (b ^ pb[i]) * fnv_prime;
        c = (c ^ pc[i]) * fnv_prime;
        d = (d ^ pd[i]) * fnv_prime;
      }
      h[0] = a, h[1] = b, h[2] = c, h[3] = d;
      return;
    }
    case 3: {
      uint64_t a = h[0], b = h[1], c = h[2];
      const uint8_t *pa = p[0], *pb = p[1], *pc = p[2];
      for (uint64_t i = 0; i < n; ++i) {
        a = (a ^ pa[i]) * fnv_prime;
        b = (b ^ pb[i]) * fnv_prime;
        c = (c ^ pc[i]) * fnv_prime;
      }
      h[0] = a, h[1] = b, h[2] = c;
      return;
    }
    case 2: {
      uint64_t a = h[0], b = h[1];
      const uint8_t *pa = p[0], *pb = p[1];
      for (uint64_t i = 0; i < n; ++i) {
        a = (a ^ pa[i]) * fnv_prime;
        b = (b ^ pb[i]) * fnv_prime;
      }
      h[0] = a, h[1] = b;
      return;
    }
    default:
      h[0] = fnv1a64(p[0], n, h[0]);
  }
}
}  // namespace

// Host checksum worker (checksum_on_gpu = 0, and host-tier objects): takes up
// to four objects with landed pieces and hashes them interleaved, each in
// object order (transfer.cpp:71-83 without the global monitor).
void engine::hash_task(const std::shared_ptr<job>& j, size_t) {
  for (;;) {
    uint32_t ids[4];
    std::vector<job::rawo::piece> pcs[4];
    int m = 0;
    {
      std::lock_guard<std::mutex> g(j->mu);
      while (m < 4 && !j->ready.empty()) {
        const uint32_t o = j->ready.front();
        j->ready.pop_front();
        auto& r = j->raws[o];
        r.queued = false;
        if (r.busy || r.q.empty()) continue;
        r.busy = true;
        pcs[m].assign(r.q.begin(), r.q.end());
        r.q.clear();
        ids[m++] = o;
      }
    }
    if (m == 0) return;
    const int64_t hs = now_ns();
    uint64_t hb = 0;
    uint64_t h[4];
    size_t pi[4] = {0, 0, 0, 0};
    uint64_t off[4] = {0, 0, 0, 0};
    for (int k = 0; k < m; ++k) h[k] = j->raws[ids[k]].fnv;
    for (;;) {
      int act[4], na = 0;
      for (int k = 0; k < m; ++k)
        if (pi[k] < pcs[k].size()) act[na++] = k;
      if (na == 0) break;
      uint64_t n = UINT64_MAX;
      const uint8_t* ptr[4];
      uint64_t hh[4];
      for (int q = 0; q < na; ++q) {
        const int k = act[q];
        n = std::min<uint64_t>(n, pcs[k][pi[k]].len - off[k]);
        ptr[q] = pcs[k][pi[k]].p + off[k];
        hh[q] = h[k];
      }
      fnv_lockstep(ptr, hh, na, n);
      hb += n * static_cast<uint64_t>(na);
      for (int q = 0; q < na; ++q) {
        const int k = act[q];
        h[k] = hh[q];
        off[k] += n;
        if (off[k] == pcs[k][pi[k]].len) {
          off[k] = 0;
          ++pi[k];
        }
      }
    }
    hash_bytes_ += hb;
    hash_busy_ns_ += static_cast<uint64_t>(now_ns() - hs);
    for (int k = 0; k < m; ++k) {
      auto& r = j->raws[ids[k]];
      uint64_t len = 0;
      for (const auto& pc : pcs[k]) len += pc.len;
      const bool done = r.hashed + len == r.size;
      r.fnv = h[k];
      if (done) {  // publish the checksum before the file can see raw_pending == 0
        std::lock_guard<std::mutex> g(j->t->mu);
        j->t->checksums[r.oid] = r.fnv;
      }
      {
        std::lock_guard<std::mutex> g(j->mu);
        r.hashed += len;
        r.busy = false;
        if (done) j->files[r.f].raw_pending -= 1;
        if (!r.q.empty() && !r.queued) {
          r.queued = true;
          j->ready.push_back(ids[k]);
        }
      }
      for (const auto& pc : pcs[k]) window_release_ref(j, pc.w);
      if (done) file_progress(j, r.f);
    }
  }
}

void engine::flush_window(const std::shared_ptr<job>& j, size_t wi) {
  auto& w = j->wins[wi];
  const uint8_t* base = w.host;
  bool ok = true;
  {
    std::lock_guard<std::mutex> g(j->t->mu);
    ok = !j->t->failed;
  }
  if (ok) {
    try {
      for (uint32_t k = w.fs_begin; k < w.fs_end; ++k) {
        const auto& s = j->fs[k];
        j->files[s.f].w->write_fixed(s.file_off, base + s.win_off, s.len);
      }
    } catch (const error& e) {
      j->t->fail(e.status, std::string("flush failed: ") + e.what(), e.object_id);
    }
  }
  {
    std::lock_guard<std::mutex> g(j->mu);
    for (uint32_t k = w.fs_begin; k < w.fs_end; ++k) j->files[j->fs[k].f].win_pending -= 1;
  }
  window_release_ref(j, wi);
  for (uint32_t k = w.fs_begin; k < w.fs_end; ++k) file_progress(j, j->fs[k].f);
}

// run_serializer (engine.cpp:341-386): encode on a worker; once every structured
// object of a file is encoded, lay the append region out in rank.objects order,
// split in serialized_chunk_bytes entries (the canonical single-flusher bytes).
void engine::serialize_task(const std::shared_ptr<job>& j, size_t si) {
  auto& so = j->sobjs[si];
  try {
    so.enc = encode(*so.v);
  } catch (const error& e) {
    j->t->fail(TS_ERR_STREAM, "object " + std::to_string(so.oid) + ": " + e.what(),
               static_cast<int64_t>(so.oid));
  }
  so.ck = fnv1a64(so.enc.data(), so.enc.size());
  TRACE("serialized rank=%d oid=%llu bytes=%zu", j->rank_id, (unsigned long long)so.oid, so.enc.size());
  bool file_ready;
  {
    std::lock_guard<std::mutex> g(j->mu);
    file_ready = --j->files[so.f].struct_pending == 0;
    j->structs_pending -= 1;
  }
  {
    std::lock_guard<std::mutex> g(j->t->mu);
    j->t->checksums[so.oid] = so.ck;
    j->t->serialized_bytes += so.enc.size();
    j->t->total_bytes += so.enc.size();
  }
  if (file_ready) {
    auto& f = j->files[so.f];
    const uint64_t chunk = std::min<uint64_t>(cfg_.serialized_chunk_bytes, pool_->capacity());
    uint64_t cur = f.tre;
    std::vector<footer_entry> entries;
    try {
      for (size_t k : f.structs) {
        const auto& s = j->sobjs[k];
        if (s.enc.empty()) continue;  // failed encode
        f.w->write_at(cur, s.enc.data(), s.enc.size());
        for (uint64_t b = 0; b < s.enc.size(); b += chunk) {
          const uint64_t len = std::min<uint64_t>(chunk, s.enc.size() - b);
          entries.push_back({s.oid, 1, cur + b, len, b, s.ck});
        }
        cur += s.enc.size();
      }
    } catch (const error& e) {
      j->t->fail(e.status, std::string("flush failed: ") + e.what(), e.object_id);
    }
    {
      std::lock_guard<std::mutex> g(j->mu);
      f.appends = std::move(entries);
      f.append_end = cur;
      f.appended = true;
    }
  }
  check_snapshot(j);
  if (file_ready) file_progress(j, so.f);
}

void engine::check_snapshot(const std::shared_ptr<job>& j) {
  bool now_done = false;
  {
    std::lock_guard<std::mutex> g(j->mu);
    if (!j->snapshot_done && j->enqueue_done && j->wins_landed == j->wins_enqueued &&
        j->structs_pending == 0) {
      j->snapshot_done = true;
      now_done = true;
    }
  }
  if (now_done) {
    {
      std::lock_guard<std::mutex> g(j->t->mu);
      if (!j->t->failed && j->wins_landed == j->wins.size()) {
        TRACE("snapshot rank=%d", j->rank_id);
        j->t->snapshot = true;
        j->t->t_snapshot = now_ns() - j->t->t_issue;
        // (events of an empty image were never recorded; a failed query must
        // not leave a stale per-thread error for a later cudaGetLastError)
        j->t->d2h_ms = j->img > 0 ? elapsed_ms(j->t->ev_d2h_first, j->t->ev_d2h_last) : 0.f;
        if (j->lane_ev1) j->t->lane_ms = elapsed_ms(j->lane_ev0, j->lane_ev1);
        if (!j->pack_events.empty()) {  // RING: sum of the pack kernels alone
          float sum = 0;
          for (auto& pe : j->pack_events) sum += elapsed_ms(pe.first, pe.second);
          j->t->pack_ms = sum;
        } else {
          j->t->pack_ms = elapsed_ms(j->t->ev_pack0, j->t->ev_capture);
        }
        if (j->t->t_captured < 0) j->t->t_captured = j->t->t_snapshot;
      }
    }
    j->t->cv.notify_all();
  }
}

void engine::file_progress(const std::shared_ptr<job>& j, size_t fi) {
  auto& f = j->files[fi];
  {
    std::lock_guard<std::mutex> g(j->mu);
    TRACE("file_progress rank=%d f=%zu fin=%d enq=%d winp=%d rawp=%d app=%d landed=%zu/%zu", j->rank_id, fi,
          (int)f.finalizing, (int)j->enqueue_done, f.win_pending, f.raw_pending, (int)f.appended, j->wins_landed,
          j->wins.size());
    if (f.finalizing || !j->enqueue_done || f.win_pending != 0 || f.raw_pending != 0 || !f.appended)
      return;
    if (j->wins_landed != j->wins.size()) return;  // persisted implies staged
    f.finalizing = true;
  }
  {
    std::lock_guard<std::mutex> g(j->t->mu);
    if (j->t->failed) return;
  }
  // finalize_file_locked (engine.cpp:470-514): raw entries from the plan, then
  // appends, sorted by file offset.
  std::vector<footer_entry> entries;
  const auto& fp = j->plan.files[fi];
  entries.reserve(fp.fixed.size() + f.appends.size());
  {
    std::lock_guard<std::mutex> g(j->t->mu);
    for (const auto& a : fp.fixed)
      entries.push_back({a.object_id, 0, a.file_offset, a.length, 0, j->t->checksums.at(a.object_id)});
  }
  entries.insert(entries.end(), f.appends.begin(), f.appends.end());
  std::sort(entries.begin(), entries.end(),
            [](const footer_entry& a, const footer_entry& b) { return a.file_offset < b.file_offset; });
  try {
    f.w->finalize_at(f.append_end, entries);
  } catch (const error& e) {
    j->t->fail(e.status, std::string("finalize failed: ") + e.what(), e.object_id);
    return;
  }
  if (const uint64_t d = f.w->direct_bytes()) {
    std::lock_guard<std::mutex> g(j->t->mu);
    j->t->direct_io_bytes += d;
  }
  if (j->io && f.w->fd() >= 0) {
    // Locked-page bookkeeping: stamp a used registration; with rotation on,
    // lock a new file's pages in the background for when it is recycled.
    auto& reg = file_registry::get();
    if (f.claimed && !f.released) {
      reg.release(f.key, f.w->fd(), true);
      f.released = true;
    } else if (cfg_.file_dma && !spare_dir().empty() && f.tre > header_reserved) {
      file_key k;
      if (reg.want_register(f.w->fd(), f.tre, &k)) {
        const int dev = device_;
        workers_->submit([k, dev] { file_registry::get().register_file(k, dev); });
      }
    }
  }
  bool all = false;
  {
    std::lock_guard<std::mutex> g(j->mu);
    f.finalized = true;
    all = ++j->files_done == j->files.size() && !j->persisted;
    if (all) j->persisted = true;
  }
  if (!all) {
    f.w.reset();  // unmap + close
    return;
  }
  {
    std::lock_guard<std::mutex> g(j->t->mu);
    j->t->persisted = true;
    j->t->t_persisted = now_ns() - j->t->t_issue;
  }
  try {
    j->sess->rank_persisted(j->rank_id);
  } catch (const error& e) {
    j->t->fail(e.status, std::string("manifest failed: ") + e.what());
  }
  j->t->cv.notify_all();
  f.w.reset();  // unmap + close after the waiters are released
}

}  // namespace tsb
