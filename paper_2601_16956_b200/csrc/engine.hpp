// B200 snapshot engine: the lazy capture path behind the State Provider API.
//
// Reference counterparts (paths relative to /root/reference/proj):
//   checkpoint_engine / issue / pre_update_barrier   engine.hpp:92-153, engine.cpp:164-630
//   checkpoint_session (manifest-last commit)        engine.hpp:57-90, engine.cpp:35-117
//   transfer_ticket (STAGED / PERSISTED, checksums)  transfer.hpp:52-114
//   staging_cache (bounded pool, back-pressure)      staging.hpp:23-78, staging.cpp:10-115
//
// What changes on B200: the per-rank state lives in HBM; capture is
// a gather-pack kernel (or direct copy-engine DMA) on low-priority streams
// ordered after the producer stream by a CUDA event, so issue never blocks the
// host and the pre-update barrier can be a stream wait. The staging pool is
// pinned host memory. Checksums, flushes and serialization run on a worker
// pool, object-parallel, with no global monitor.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "filereg.hpp"
#include "numa.hpp"
#include "format.hpp"
#include "kernels.cuh"

namespace tsb {

void cuda_check(cudaError_t e, const char* what);
// mkdir -p
void mkdirs(const std::string& path);
// Elapsed time between two timing events, 0 (and no lingering error) if either was not recorded.
float elapsed_ms(cudaEvent_t a, cudaEvent_t b);

class thread_pool {
 public:
  // `init` runs first on every worker thread (e.g. NUMA binding)
  explicit thread_pool(int n, std::function<void()> init = {});
  ~thread_pool();
  void submit(std::function<void()> f);
  int size() const { return static_cast<int>(threads_.size()); }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  bool stop_ = false;
  std::vector<std::thread> threads_;
};

// Bounded pinned host pool with the reference's allocation policy
// (staging.cpp:15-38: circular bump, wraparound, then first-fit) and FIFO-fair
// blocking acquire with an optional deadline (staging.cpp:44-80).
class pinned_pool {
 public:
  struct region {
    uint64_t id = 0, offset = 0, length = 0;
  };
  pinned_pool(uint64_t capacity);
  ~pinned_pool();
  region acquire(uint64_t size, int64_t deadline_ns);  // deadline < 0: none
  void release(const region& r);
  uint8_t* data(const region& r) const { return base_ + r.offset; }
  uint8_t* base() const { return base_; }
  uint64_t capacity() const { return capacity_; }
  uint64_t peak() const { return peak_; }

 private:
  bool find_locked(uint64_t size, uint64_t* off) const;
  uint8_t* base_ = nullptr;
  uint64_t capacity_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::map<uint64_t, uint64_t> live_;  // offset -> length
  std::deque<uint64_t> waiters_;
  uint64_t next_id_ = 1, next_token_ = 1, bump_ = 0, allocated_ = 0, peak_ = 0;
};

class session;

struct ticket_state {
  uint64_t checkpoint_id = 0;
  int rank_id = 0;
  std::mutex mu;
  std::condition_variable cv;
  bool capture_recorded = false;  // capture event enqueued (barrier may use it)
  bool snapshot = false, persisted = false, failed = false;
  ts_status err_status = TS_OK;
  std::string err;
  int64_t err_oid = -1;
  int64_t t_issue = 0, t_captured = -1, t_snapshot = -1, t_persisted = -1;
  int64_t issue_block_ns = 0, barrier_block_ns = 0;
  uint64_t total_bytes = 0, raw_bytes = 0, serialized_bytes = 0, image_bytes = 0;
  uint64_t file_dma_bytes = 0;  // fixed-region bytes DMA'd straight into file pages
  uint64_t host_checksum_bytes = 0;  // device-tier bytes hashed by host workers (rest: FNV kernels)
  uint64_t helper_bytes = 0;         // image bytes D2H'd by helper GPUs' copy engines (NVLink read)
  uint64_t direct_io_bytes = 0;      // fixed-region bytes written O_DIRECT (flush_mmap = 2)
  float pack_ms = 0, d2h_ms = 0, lane_ms = 0;
  uint64_t lane_checksum_bytes = 0;  // device-tier bytes hashed by the lane-serial FNV kernel
  uint64_t packed_bytes = 0;         // image bytes written by the pack kernels
  uint32_t kernel_launches = 0, copies = 0;
  cudaEvent_t ev_start = nullptr, ev_capture = nullptr, ev_d2h_first = nullptr,
              ev_d2h_last = nullptr, ev_pack0 = nullptr;
  int device = 0;
  std::unordered_map<uint64_t, uint64_t> checksums;
  // structured values handed over by the caller (ts_ticket_adopt_values): the
  // job holds the ticket, so they outlive every serializer that reads them
  std::vector<std::unique_ptr<value>> owned_values;

  ~ticket_state();
  void fail(ts_status s, const std::string& m, int64_t oid = -1);
  void throw_if_failed_locked();
  int64_t wait_until(const std::function<bool()>& pred);  // returns blocked ns
};

struct job;

class engine {
 public:
  engine(const ts_engine_config& cfg, int rank_id, int device);
  ~engine();
  std::shared_ptr<ticket_state> issue(const std::shared_ptr<session>& s, const ts_rank_info& rank,
                                      const ts_object_desc* objs, size_t n, uint64_t iteration,
                                      cudaStream_t producer);
  // host_block: 0 = stream wait on the capture event (no host block), 1 = host
  // waits for the capture, 2 = host waits for the full snapshot (reference).
  int64_t pre_update_barrier(const std::shared_ptr<ticket_state>& t, cudaStream_t opt_stream,
                             int host_block);
  void shutdown();
  void set_spare_dir(const std::string& d) {
    std::lock_guard<std::mutex> g(mu_);
    spare_dir_ = d;
  }
  std::string spare_dir() {
    std::lock_guard<std::mutex> g(mu_);
    return spare_dir_;
  }
  // Creates up to `copies` spare files per file of this rank's layout in
  // `spare_dir` (sized, page-locked when file_dma applies), so the first
  // checkpoints recycle them like later ones do. Returns the bytes locked.
  uint64_t provision_spares(const std::string& spare_dir, const ts_rank_info& rank,
                            const ts_object_desc* objs, size_t n, int copies);
  const ts_engine_config& config() const { return cfg_; }
  int device() const { return device_; }
  int numa_node() const { return numa_.node; }

 private:
  friend struct job;
  void prepare(const std::shared_ptr<job>& j, const ts_rank_info& rank, const ts_object_desc* objs, size_t n);
  void copier_loop();
  void completer_loop();
  void run_job(const std::shared_ptr<job>& j);
  void window_landed(const std::shared_ptr<job>& j, size_t w);
  void hash_task(const std::shared_ptr<job>& j, size_t obj);
  void flush_window(const std::shared_ptr<job>& j, size_t w);
  void window_release_ref(const std::shared_ptr<job>& j, size_t w);
  void serialize_task(const std::shared_ptr<job>& j, size_t s);
  void file_progress(const std::shared_ptr<job>& j, size_t f);
  void check_snapshot(const std::shared_ptr<job>& j);
  cudaEvent_t get_event();
  void put_event(cudaEvent_t e);
  // Helper GPUs (helper_mask): their copy engines read this GPU's staged image
  // over NVLink (peer access) and write it to host memory through their own
  // PCIe links — D2H load balancing for ranks holding more than their share.
  struct helper_dev {
    int dev = 0;
    cudaStream_t st = nullptr;
    std::mutex mu;
    std::vector<cudaEvent_t> free_ev;
  };
  cudaEvent_t helper_event(size_t k);
  void put_helper_event(size_t k, cudaEvent_t e);
  std::vector<std::unique_ptr<helper_dev>> helpers_;
  uint8_t* ensure_device_ring(uint64_t bytes);
  void* ensure_seg_buffer(uint64_t bytes);
  uint8_t* ensure_fnv_buffer(uint64_t bytes);
  void fnv_landed(const std::shared_ptr<job>& j);

  ts_engine_config cfg_;
  int rank_id_, device_, sms_;
  numa_place numa_;  // the GPU's NUMA node: engine threads + pinned pool live there
  std::unique_ptr<pinned_pool> pool_;
  std::unique_ptr<thread_pool> workers_;
  cudaStream_t pack_stream_ = nullptr, copy_stream_ = nullptr, ck_stream_ = nullptr;
  cudaStream_t ck_hi_stream_ = nullptr;
  cudaStream_t ck_lane_stream_ = nullptr;  // lane-serial checksums over the state (capture path)  // checksums a ring slot's reuse (hence the capture) waits for
  uint8_t* ring_ = nullptr;
  uint64_t ring_bytes_ = 0;
  void* segbuf_ = nullptr;
  uint64_t segbuf_bytes_ = 0;
  uint8_t* fnvbuf_ = nullptr;
  uint64_t fnvbuf_bytes_ = 0;
  uint64_t* ck_host_ = nullptr;  // mapped pinned checksum results (not from the staging pool:
  uint64_t ck_host_n_ = 0;       // holding pool space across the D2H could starve the windows)

  std::mutex ev_mu_;
  std::vector<cudaEvent_t> ev_free_;

  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::shared_ptr<job>> jobs_;
  struct pending_window {
    std::shared_ptr<job> j;
    size_t w;
    bool fnv = false;  // device checksums of the job instead of a D2H window
  };
  std::deque<pending_window> inflight_;
  bool stopping_ = false, copier_done_ = false;
  std::shared_ptr<job> last_job_;
  std::vector<std::shared_ptr<job>> retired_;  // dropped by the copier (under mu_)
  std::string spare_dir_;  // recycled files of retired checkpoints (retire_checkpoint)
  // checksum placement (auto): host hashing capacity, measured per job
  double host_rate_ = 0, chain_rate_ = 0.45e9, slack_s_ = 0, slack_d2h_s_ = 0;
  std::atomic<uint64_t> hash_bytes_{0}, hash_busy_ns_{0};
  std::thread copier_, completer_;
};

// Manifest info of one rank (engine.cpp:539-558): files in ascending id, object
// ids per file in rank.objects order, every object's bookkeeping fields.
manifest_rank make_rank_info(const ts_rank_info& rank, const ts_object_desc* objs, size_t n);

class session {
 public:
  session(const std::string& dir, uint64_t ckpt_id, uint64_t iteration, const ts_manifest_echo* echo,
          int n_ranks, bool writes_manifest);
  std::string rank_dir(int rank_id) const { return dir_ + "/" + rank_dir_name(rank_id); }
  const std::string& dir() const { return dir_; }
  uint64_t checkpoint_id() const { return m_.checkpoint_id; }
  uint64_t iteration() const { return m_.iteration; }
  void register_rank(manifest_rank info);
  std::vector<uint8_t> rank_blob(int rank_id);
  void add_remote_rank(const uint8_t* blob, size_t n);
  void rank_persisted(int rank_id);
  bool wait_complete(int64_t timeout_ns);
  bool complete();

 private:
  void maybe_commit_locked(std::unique_lock<std::mutex>& g);
  std::string dir_;
  manifest m_;
  int n_ranks_;
  bool writes_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::map<int, manifest_rank> ranks_;
  std::map<int, bool> persisted_;
  bool complete_ = false;
  bool committing_ = false;
  std::string commit_error_;
};

}  // namespace tsb
