// Restore and verify (format.cpp:201-529), B200 path:
//   files --pread--> pinned window ring --H2D--> HBM window ring --unpack--> shards
// with per-object FNV verification on host threads overlapping the transfers.
#include <fcntl.h>
#include <sys/uio.h>
#include <sys/vfs.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <sys/mman.h>
#include <cstdio>
#include <cstdlib>
#include <unordered_map>
#include <unordered_set>

#include "engine.hpp"
#include "restore.hpp"
#include "uring.hpp"

namespace tsb {

namespace {

const bool g_rtrace = std::getenv("TS_TRACE") != nullptr;
void rtrace(const char* what, int64_t t0) {
  if (g_rtrace) std::fprintf(stderr, "[ts restore] %-28s %9.3f ms\n", what, (now_ns() - t0) / 1e6);
}

struct fd_holder {
  int fd = -1;
  int dfd = -1;  // O_DIRECT descriptor (restore_handle::direct_io), else -1
  bool uring = false;  // direct reads through the thread's io_uring (direct_io = 2)
  ~fd_holder() {
    if (dfd >= 0) ::close(dfd);
    if (fd >= 0) ::close(fd);
  }
};

// True when fewer than half of 64 sampled pages of [0, len) are in the page
// cache: a cold file on a disk, where O_DIRECT reads beat pread (measured
// 3.8-4.0 vs 1.6-2.8 GB/s); warm files (just written) stay on pread from the
// page cache. Probed with preadv2(RWF_NOWAIT), which fails with EAGAIN for a
// page that is not cached whatever the caller's permissions on the file
// (mincore over a mapping reports page-cache state only to callers that could
// write the file, Linux >= 5.2, so read-only checkpoints would be misjudged).
bool mostly_uncached(int fd, uint64_t len) {
  if (len < (8ull << 20)) return false;
  const uint64_t pg = 4096, pages = len / pg;
  int resident = 0, answered = 0;
  for (int i = 0; i < 64; ++i) {
    unsigned char v = 0;
    struct iovec io = {&v, 1};
    const uint64_t at = (pages * static_cast<uint64_t>(2 * i + 1) / 128) * pg;
    const ssize_t k = ::preadv2(fd, &io, 1, static_cast<off_t>(at), RWF_NOWAIT);
    if (k == 1) ++resident, ++answered;
    else if (k < 0 && errno == EAGAIN) ++answered;
  }
  return answered == 64 && resident < 32;  // (no RWF_NOWAIT support: stay on pread)
}

// tmpfs serves O_DIRECT from its page cache (Linux >= 6.6 accepts the flag):
// there is nothing to bypass, so O_DIRECT is never used on it.
bool on_tmpfs(int fd) {
  struct statfs fs;
  return ::fstatfs(fd, &fs) == 0 && static_cast<unsigned long>(fs.f_type) == 0x01021994ul;
}

// Reads [off, off+n) of a file into p: the 4 KiB-aligned body O_DIRECT when
// the descriptor exists and p and off share their offset within a block, the
// rest (and any refused or short direct read) with pread.
void read_range(const fd_holder& f, uint8_t* p, uint64_t n, uint64_t off, const std::string& path,
                std::atomic<uint64_t>* direct) {
  constexpr uint64_t blk = 4096;
  if (f.dfd >= 0 && ((reinterpret_cast<uintptr_t>(p) - off) & (blk - 1)) == 0) {
    const uint64_t a = (off + blk - 1) & ~(blk - 1), e = (off + n) & ~(blk - 1);
    if (e > a) {
      const int64_t k = f.uring ? uring_pread(f.dfd, p + (a - off), e - a, a, 4ull << 20)
                                : static_cast<int64_t>(::pread(f.dfd, p + (a - off), e - a, static_cast<off_t>(a)));
      if (k == static_cast<int64_t>(e - a)) {
        *direct += e - a;
        if (a > off) pread_all(f.fd, p, a - off, off, path);
        if (off + n > e) pread_all(f.fd, p + (e - off), off + n - e, e, path);
        return;
      }
    }
  }
  pread_all(f.fd, p, n, off, path);
}

// Process-wide staging reused across restores while any restore handle is
// open (pinning and multi-GB allocations are slow); freed when the last one
// closes, so training after a restore gets its HBM and host memory back.
std::mutex g_stage_mu;
int g_stage_users = 0;
uint8_t* g_pinned = nullptr;
uint64_t g_pinned_bytes = 0;

// Device window ring, per device, grown on demand and kept (stream-ordered
// frees of a multi-GB buffer return it to the OS at the next sync: slow).
std::unordered_map<int, std::pair<uint8_t*, uint64_t>> g_dev_stage, g_dev_scratch, g_dev_fnv;
uint8_t* device_cached(std::unordered_map<int, std::pair<uint8_t*, uint64_t>>& m, int device, uint64_t bytes) {
  auto& e = m[device];
  if (e.second < bytes) {
    if (e.first) cudaFree(e.first);
    e.first = nullptr;
    e.second = 0;
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&e.first), bytes), "cudaMalloc(restore staging)");
    e.second = bytes;
  }
  return e.first;
}
uint8_t* device_stage(int device, uint64_t bytes) { return device_cached(g_dev_stage, device, bytes); }
uint8_t* device_scratch(int device, uint64_t bytes) { return device_cached(g_dev_scratch, device, bytes); }
uint8_t* device_fnv(int device, uint64_t bytes) { return device_cached(g_dev_fnv, device, bytes); }

uint8_t* pinned_stage(uint64_t bytes) {
  if (g_pinned_bytes < bytes) {
    if (g_pinned) cudaFreeHost(g_pinned);
    g_pinned = nullptr;
    g_pinned_bytes = 0;
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&g_pinned), bytes, cudaHostAllocPortable),
               "cudaHostAlloc(restore ring)");
    g_pinned_bytes = bytes;
  }
  return g_pinned;
}

void release_staging_locked() {
  if (g_pinned) cudaFreeHost(g_pinned);
  g_pinned = nullptr;
  g_pinned_bytes = 0;
  for (auto* m : {&g_dev_stage, &g_dev_scratch, &g_dev_fnv}) {
    for (auto& [dev, e] : *m) {
      if (!e.first) continue;
      cudaSetDevice(dev);
      cudaFree(e.first);
    }
    m->clear();
  }
}

}  // namespace

uint64_t restore_release_staging() {
  std::lock_guard<std::mutex> g(g_stage_mu);
  uint64_t b = g_pinned_bytes;
  for (auto* m : {&g_dev_stage, &g_dev_scratch, &g_dev_fnv})
    for (auto& kv : *m) b += kv.second.second;
  int cur = 0;
  cudaGetDevice(&cur);
  release_staging_locked();
  cudaSetDevice(cur);
  return b;
}

restore_handle::~restore_handle() {
  std::lock_guard<std::mutex> g(g_stage_mu);
  if (--g_stage_users == 0) {
    int cur = 0;
    cudaGetDevice(&cur);
    release_staging_locked();
    cudaSetDevice(cur);
  }
}

void restore_handle::load_rank(int index) {
  auto& rc = ranks.at(static_cast<size_t>(index));
  if (rc.loaded) return;
  const auto& r = m.ranks.at(static_cast<size_t>(index));
  for (const auto& mf : r.files) {
    file_info fi;
    fi.file_id = mf.file_id;
    fi.path = base + "/" + mf.path;
    fi.entries = read_footer(fi.path, &fi.size);
    fi.region_end = header_reserved;
    for (const auto& e : fi.entries) {
      if (e.file_offset + e.length > fi.size)
        fail(TS_ERR_CORRUPT_FOOTER, "entry range outside the file", static_cast<int64_t>(e.object_id));
      if (e.kind == 0) fi.region_end = std::max(fi.region_end, e.file_offset + e.length);
    }
    rc.files.push_back(std::move(fi));
  }
  // Object sizes + the manifest cross-checks of restore_checkpoint (format.cpp:446-470).
  std::unordered_set<uint64_t> listed;
  for (size_t k = 0; k < r.files.size(); ++k) {
    std::unordered_set<uint64_t> expected(r.files[k].object_ids.begin(), r.files[k].object_ids.end());
    std::unordered_set<uint64_t> found;
    for (const auto& e : rc.files[k].entries) {
      if (!expected.count(e.object_id))
        fail(TS_ERR_BAD_MANIFEST, "file contains an object the manifest does not list",
             static_cast<int64_t>(e.object_id));
      found.insert(e.object_id);
      rc.sizes[e.object_id] += e.length;
      rc.kinds[e.object_id] = e.kind;
    }
    for (uint64_t oid : r.files[k].object_ids)
      if (!found.count(oid))
        fail(TS_ERR_CORRUPT_FOOTER, "file is missing manifest-listed objects: " + rc.files[k].path,
             static_cast<int64_t>(oid));
  }
  for (const auto& o : r.objects)
    if (!rc.sizes.count(o.object_id))
      fail(TS_ERR_BAD_MANIFEST, "object missing from checkpoint", static_cast<int64_t>(o.object_id));
  rc.loaded = true;
}

restore_handle::restore_handle(const std::string& manifest_path) {
  m = read_manifest(manifest_path);
  const auto slash = manifest_path.find_last_of('/');
  base = slash == std::string::npos ? "." : manifest_path.substr(0, slash);
  ranks.resize(m.ranks.size());
  std::lock_guard<std::mutex> g(g_stage_mu);
  ++g_stage_users;
}

namespace {
// Pieces of one object sorted by object offset must tile [0, size) (format.cpp:269-278).
void check_tiling(std::vector<const footer_entry*>& pieces, uint64_t oid) {
  std::sort(pieces.begin(), pieces.end(),
            [](const footer_entry* a, const footer_entry* b) { return a->object_offset_base < b->object_offset_base; });
  uint64_t off = 0;
  for (const auto* e : pieces) {
    if (e->object_offset_base != off)
      fail(TS_ERR_CORRUPT_FOOTER, "gap in object byte ranges", static_cast<int64_t>(oid));
    off += e->length;
  }
}
}  // namespace

void restore_handle::restore_rank(int index, const ts_object_desc* dst, size_t n, int device,
                                  cudaStream_t st, ts_restore_stats* stats) {
  const int64_t t_begin = now_ns();
  load_rank(index);
  rtrace("load_rank", t_begin);
  auto& rc = ranks[static_cast<size_t>(index)];
  const auto& mr = m.ranks[static_cast<size_t>(index)];
  cuda_check(cudaSetDevice(device), "cudaSetDevice");

  std::unordered_map<uint64_t, const ts_object_desc*> dmap;
  for (size_t i = 0; i < n; ++i) dmap.emplace(dst[i].object_id, &dst[i]);

  // Image = each file's region [4096, region_end), 4 KiB aligned file images.
  struct rpiece {
    uint64_t pos, len;
    uint32_t obj;  // index into objs
    uint64_t obj_off;
  };
  struct robj {
    uint64_t oid, size, ck;
    const ts_object_desc* d;
    uint64_t fnv = fnv_seed, hashed = 0;
    bool busy = false;
    std::deque<std::pair<const uint8_t*, std::pair<uint64_t, int>>> q;  // ptr, (len, slot)
  };
  std::vector<robj> objs;
  std::vector<rpiece> pieces;
  std::vector<std::pair<uint64_t, uint64_t>> file_img;  // (img start, len)
  std::unordered_map<uint64_t, uint32_t> oidx;
  uint64_t img = 0, raw_bytes = 0;
  for (size_t k = 0; k < rc.files.size(); ++k) {
    const auto& fi = rc.files[k];
    img = align_up(img, 4096);
    const uint64_t fimg = img;
    file_img.push_back({fimg, fi.region_end - header_reserved});
    std::unordered_map<uint64_t, std::vector<const footer_entry*>> by_obj;
    for (const auto& e : fi.entries)
      if (e.kind == 0) by_obj[e.object_id].push_back(&e);
    for (auto& [oid, ps] : by_obj) {
      check_tiling(ps, oid);
      auto it = dmap.find(oid);
      if (it == dmap.end())
        fail(TS_ERR_INVALID_ARG, "restore: no destination for raw object", static_cast<int64_t>(oid));
      if (it->second->size_bytes != rc.sizes[oid])
        fail(TS_ERR_INVALID_ARG, "restore: destination size mismatch", static_cast<int64_t>(oid));
      robj o;
      o.oid = oid;
      o.size = rc.sizes[oid];
      o.ck = ps.front()->checksum;
      o.d = it->second;
      oidx[oid] = static_cast<uint32_t>(objs.size());
      for (const auto* e : ps)
        pieces.push_back({fimg + (e->file_offset - header_reserved), e->length,
                          static_cast<uint32_t>(objs.size()), e->object_offset_base});
      objs.push_back(std::move(o));
      raw_bytes += rc.sizes[oid];
    }
    img = fimg + (fi.region_end - header_reserved);
  }
  std::sort(pieces.begin(), pieces.end(), [](const rpiece& a, const rpiece& b) { return a.pos < b.pos; });

  // Device scatter table (device-tier destinations only).
  std::vector<dev::useg> usegs;
  std::vector<uint32_t> useg_dev;  // per scatter segment: index of its object among device-tier objects
  std::vector<uint32_t> dev_objs;
  std::vector<int64_t> dev_index(objs.size(), -1);
  for (uint32_t i = 0; i < objs.size(); ++i)
    if (objs[i].d->tier == TS_TIER_DEVICE) {
      dev_index[i] = static_cast<int64_t>(dev_objs.size());
      dev_objs.push_back(i);
    }
  for (const auto& p : pieces) {
    const auto& o = objs[p.obj];
    if (o.d->tier == TS_TIER_DEVICE) {
      usegs.push_back({p.pos, p.len, static_cast<uint8_t*>(const_cast<void*>(o.d->data)) + p.obj_off});
      useg_dev.push_back(static_cast<uint32_t>(dev_index[p.obj]));
    }
  }

  // Pipeline: K device windows of W bytes (one H2D target + scatter-unpack
  // launch each; windows are independent, any order; a stream callback frees
  // the slot) fed through a small pool of P pinned pieces of R bytes: each
  // pool task preads one piece and enqueues its H2D at once, so the copy
  // engine reads the piece while it is still in the host's last-level cache
  // (PCIe reads are coherent) — two passes over host DRAM per byte instead of
  // three when whole windows were staged first (tools/restore_stage_probe.cu:
  // 51 GB/s with 32 x 4 MiB pieces vs 37-41 GB/s for 1 GiB windows,
  // profiles/r2_restore_stage_probe.jsonl), and 128 MiB of pinned staging
  // instead of K x W. (Large device windows: fewer, longer unpack launches —
  // 1 GiB: 90 % of the HBM roofline vs 82-85 % at 256 MiB.)
  // Knobs for experiments: TS_RESTORE_WINDOWS (device ring depth),
  // TS_RESTORE_READ_MB (piece size R), TS_RESTORE_PIECES (P).
  const char* kw = std::getenv("TS_RESTORE_WINDOWS");
  const int K = std::max(2, std::min(8, kw ? std::atoi(kw) : 4));  // (slot_busy holds 8)
  const uint64_t W = std::min<uint64_t>(1ull << 30, std::max<uint64_t>(64ull << 20, align_up(img / K + 1, 2ull << 20)));
  const char* rp = std::getenv("TS_RESTORE_READ_MB");
  const uint64_t R = static_cast<uint64_t>(std::max(1, std::min(64, rp ? std::atoi(rp) : 4))) << 20;
  const char* pp = std::getenv("TS_RESTORE_PIECES");
  const int P = std::max(2, std::min(256, pp ? std::atoi(pp) : 32));
  // One restore at a time uses the rings: take the lock first and size them
  // under it, so a concurrent restore cannot reallocate them in between.
  std::lock_guard<std::mutex> stage_guard(g_stage_mu);
  uint8_t* hring = pinned_stage(R * P);
  rtrace("pinned stage", t_begin);
  uint8_t* dring = nullptr;
  dev::useg* d_usegs = nullptr;
  dring = device_stage(device, W * K);
  if (!usegs.empty()) {
    d_usegs = reinterpret_cast<dev::useg*>(device_scratch(device, usegs.size() * sizeof(dev::useg)));
    cuda_check(cudaMemcpyAsync(d_usegs, usegs.data(), usegs.size() * sizeof(dev::useg),
                               cudaMemcpyHostToDevice, st), "upload unpack table");
  }
  cudaEvent_t ev_a, ev_b;
  cudaEventCreate(&ev_a);
  cudaEventCreate(&ev_b);

  // Device checksums over the restored shards (the whole chain file -> pinned
  // -> H2D -> unpack), window by window in image order on their own stream:
  // chained per-object states, so they overlap the remaining transfers instead
  // of following them. Tables are built up front; the sequencer below launches
  // window w once it is unpacked and every earlier window has been launched.
  const uint32_t nf = static_cast<uint32_t>(dev_objs.size());
  const uint64_t nwin = img ? (img + W - 1) / W : 0;
  struct fnv_window {
    std::vector<dev::fnv_obj> fo;
    uint64_t nseg = 0, nchunk = 0;
  };
  std::vector<fnv_window> fwin(nwin);
  uint64_t max_tab = 0, max_scr = 0;
  for (uint64_t w = 0; w < nwin; ++w) {
    const uint64_t lo = w * W, hi = std::min(img, lo + W);
    auto uit = std::lower_bound(usegs.begin(), usegs.end(), lo,
                                [](const dev::useg& u, uint64_t x) { return u.pos + u.len <= x; });
    for (; uit != usegs.end() && uit->pos < hi; ++uit) {
      const uint64_t a = std::max(lo, uit->pos), b = std::min(hi, uit->pos + uit->len);
      if (b > a) fwin[w].fo.push_back({uit->dst + (a - uit->pos), b - a, 0, 0, useg_dev[uit - usegs.begin()]});
    }
    auto& fw = fwin[w];
    if (fw.fo.empty()) continue;
    fw.nseg = dev::fnv_prepare(fw.fo.data(), static_cast<uint32_t>(fw.fo.size()), &fw.nchunk);
    max_tab = std::max<uint64_t>(max_tab, fw.fo.size() * sizeof(dev::fnv_obj));
    max_scr = std::max<uint64_t>(max_scr, dev::fnv_scratch_bytes(fw.nseg, fw.nchunk, static_cast<uint32_t>(fw.fo.size())));
  }
  const uint64_t st_b = align_up(std::max<uint64_t>(nf, 1) * 8ull, 256), tab_b = align_up(std::max<uint64_t>(max_tab, 1), 256);
  uint8_t* fbuf = device_fnv(device, st_b + tab_b + max_scr);
  uint64_t* d_states = reinterpret_cast<uint64_t*>(fbuf);
  dev::fnv_obj* d_tab = reinterpret_cast<dev::fnv_obj*>(fbuf + st_b);
  uint8_t* d_scr = fbuf + st_b + tab_b;
  struct stream_guard {
    cudaStream_t s = nullptr;
    ~stream_guard() {
      if (s) cudaStreamDestroy(s);
    }
  } fst;
  cuda_check(cudaStreamCreateWithFlags(&fst.s, cudaStreamNonBlocking), "checksum stream");
  const std::vector<uint64_t> seeds(std::max<uint32_t>(nf, 1), fnv_seed);
  if (nf) cuda_check(cudaMemcpyAsync(d_states, seeds.data(), nf * 8ull, cudaMemcpyHostToDevice, fst.s), "upload");
  std::vector<cudaEvent_t> win_unpacked(nwin, nullptr);
  std::vector<char> win_ready(nwin, 0);
  uint64_t next_fnv = 0;
  std::atomic<uint32_t> launches_f{0};
  auto fnv_advance = [&]() {  // under cuda_mu
    for (; next_fnv < nwin && win_ready[next_fnv]; ++next_fnv) {
      auto& fw = fwin[next_fnv];
      if (fw.fo.empty()) continue;
      cuda_check(cudaStreamWaitEvent(fst.s, win_unpacked[next_fnv], 0), "checksums wait for the unpack");
      cuda_check(cudaMemcpyAsync(d_tab, fw.fo.data(), fw.fo.size() * sizeof(dev::fnv_obj), cudaMemcpyHostToDevice,
                                 fst.s), "upload checksum table");
      dev::launch_fnv(d_tab, static_cast<uint32_t>(fw.fo.size()), fw.nseg, fw.nchunk, d_states, d_scr, fst.s);
      launches_f += 11;
      cuda_check(cudaGetLastError(), "checksum kernels");
    }
  };

  std::vector<fd_holder> fds(rc.files.size());
  for (size_t k = 0; k < rc.files.size(); ++k) {
    fds[k].fd = ::open(rc.files[k].path.c_str(), O_RDONLY);
    if (fds[k].fd < 0) fail(TS_ERR_MISSING_FILE, "cannot open " + rc.files[k].path);
    if (!on_tmpfs(fds[k].fd) &&
        (direct_io > 0 || (direct_io < 0 && mostly_uncached(fds[k].fd, rc.files[k].region_end))))
      fds[k].dfd = ::open(rc.files[k].path.c_str(), O_RDONLY | O_DIRECT);  // -1 (refused): pread
    fds[k].uring = fds[k].dfd >= 0 && direct_io == 2;
  }
  // Page-locked files (registered by this process's engines): H2D straight
  // from the page cache, no pread. Pinned against claims/drops until the end.
  struct reg_reads {
    std::vector<const uint8_t*> map;
    std::vector<file_key> key;
    ~reg_reads() {
      for (size_t k = 0; k < map.size(); ++k)
        if (map[k]) file_registry::get().release_read(key[k]);
    }
  } regs;
  regs.map.assign(rc.files.size(), nullptr);
  regs.key.resize(rc.files.size());
  uint64_t direct_bytes = 0;
  std::atomic<uint64_t> odirect_bytes{0};
  if (use_file_cache)
    for (size_t k = 0; k < rc.files.size(); ++k)
      if (file_img[k].second > 0) {
        regs.map[k] = file_registry::get().acquire_read(fds[k].fd, rc.files[k].region_end, &regs.key[k]);
        if (regs.map[k]) direct_bytes += file_img[k].second;
      }
  // host address of image byte `pos` of a window staged at `hs` ([lo, hi))
  auto host_src = [&](uint64_t pos, uint64_t lo, const uint8_t* hs) -> const uint8_t* {
    size_t k = std::upper_bound(file_img.begin(), file_img.end(), pos,
                                [](uint64_t x, const std::pair<uint64_t, uint64_t>& f) { return x < f.first; }) -
               file_img.begin();
    k = k ? k - 1 : 0;
    if (regs.map[k] && pos >= file_img[k].first && pos < file_img[k].first + file_img[k].second)
      return regs.map[k] + header_reserved + (pos - file_img[k].first);
    return hs + (pos - lo);
  };

  struct shared_state {
    std::mutex mu;
    std::condition_variable cv;
    int slot_busy[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    std::string err;
    ts_status err_status = TS_OK;
    int64_t err_oid = -1;
  } S;
  const int nthreads = static_cast<int>(std::min<unsigned>(16, std::max(2u, std::thread::hardware_concurrency())));
  struct host_cb_arg {
    shared_state* s;
    int slot;
  };
  std::vector<host_cb_arg> cb_args(K);
  for (int k = 0; k < K; ++k) cb_args[k] = {&S, k};
  std::mutex cuda_mu;  // keeps each window's H2D + unpack + callback contiguous on the stream
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> unpack_ev;  // kernel-only unpack timing (roofline)
  struct ev_list_guard {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v;
    ~ev_list_guard() {
      for (auto& e : v) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
      }
    }
  } unpack_ev_guard{unpack_ev};
  std::atomic<uint32_t> launches_a{0};
  const int ctas = dev::sm_count(device) * 2;
  auto set_err = [&](const error& e) {
    std::lock_guard<std::mutex> g(S.mu);
    if (S.err_status == TS_OK) {
      S.err_status = e.status;
      S.err = e.what();
      S.err_oid = e.object_id;
    }
  };
  // Host-tier objects' bytes of image range [a, b), found at `src` (image
  // byte a), to their host buffers.
  auto copy_host_tier = [&](uint64_t a0, uint64_t b0, const uint8_t* src) {
    auto pit = std::lower_bound(pieces.begin(), pieces.end(), a0,
                                [](const rpiece& p, uint64_t x) { return p.pos + p.len <= x; });
    for (; pit != pieces.end() && pit->pos < b0; ++pit) {
      const auto& o = objs[pit->obj];
      if (o.d->tier == TS_TIER_DEVICE) continue;
      const uint64_t a = std::max(a0, pit->pos), b = std::min(b0, pit->pos + pit->len);
      if (b > a)
        std::memcpy(static_cast<uint8_t*>(const_cast<void*>(o.d->data)) + pit->obj_off + (a - pit->pos),
                    src + (a - a0), b - a);
    }
  };
  // Every byte of window [lo, hi) is on the device (its H2Ds enqueued): the
  // scatter-unpack, the device checksums' turn, and the callback freeing the
  // slot. Under cuda_mu. After a failure only the slot is freed.
  auto window_done = [&](uint64_t lo, uint64_t hi, int slot) {
    bool ok;
    {
      std::lock_guard<std::mutex> g(S.mu);
      ok = S.err_status == TS_OK;
    }
    if (ok) {
      uint8_t* ds = dring + static_cast<uint64_t>(slot) * W;
      auto uit = std::lower_bound(usegs.begin(), usegs.end(), lo,
                                  [](const dev::useg& u, uint64_t x) { return u.pos + u.len <= x; });
      if (uit != usegs.end() && uit->pos < hi) {
        const size_t ui = static_cast<size_t>(uit - usegs.begin());
        cudaEvent_t u0 = nullptr, u1 = nullptr;
        cudaEventCreate(&u0);
        cudaEventCreate(&u1);
        cudaEventRecord(u0, st);
        dev::launch_unpack(d_usegs + ui, static_cast<uint32_t>(usegs.size() - ui), lo, hi, ds, ctas, 512, st);
        cudaEventRecord(u1, st);
        unpack_ev.emplace_back(u0, u1);
        launches_a += 1;
        cuda_check(cudaGetLastError(), "unpack launch");
        win_unpacked[lo / W] = u1;
      }
      win_ready[lo / W] = 1;
      fnv_advance();
    }
    cuda_check(cudaLaunchHostFunc(st, [](void* a) {
                 auto* p = static_cast<host_cb_arg*>(a);
                 std::lock_guard<std::mutex> g(p->s->mu);
                 p->s->slot_busy[p->slot] = 0;
                 p->s->cv.notify_all();
               }, &cb_args[slot]), "cudaLaunchHostFunc");
  };
  struct wstate {
    uint64_t lo, hi;
    int slot;
    std::atomic<int> left{0};
  };
  // One part of a window is on its way to the device; the last one finishes it.
  auto part_done = [&](wstate& ws) {  // under cuda_mu
    if (--ws.left == 0) window_done(ws.lo, ws.hi, ws.slot);
  };
  // Pinned pieces: piece i of the restore uses buffer i % P; its mutex is held
  // from the pread to the H2D's event record, and the next user of the buffer
  // waits for that H2D.
  std::vector<std::mutex> pmu(P);
  std::vector<cudaEvent_t> pev(P, nullptr);
  std::vector<char> pused(P, 0);
  struct pev_guard {
    std::vector<cudaEvent_t>& v;
    ~pev_guard() {
      for (auto e : v)
        if (e) cudaEventDestroy(e);
    }
  } pev_g{pev};
  for (auto& e : pev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  std::atomic<uint64_t> piece_seq{0};

  double read_s = 0;
  rtrace("setup done", t_begin);
  const int64_t r0 = now_ns();
  {
    thread_pool pool(nthreads);
    cuda_check(cudaEventRecord(ev_a, st), "event");
    for (uint64_t lo = 0, w = 0; lo < img; lo += W, ++w) {
      const uint64_t hi = std::min(lo + W, img);
      const int slot = static_cast<int>(w % K);
      {
        std::unique_lock<std::mutex> g(S.mu);
        S.cv.wait(g, [&] { return S.slot_busy[slot] == 0 || S.err_status != TS_OK; });
        if (S.err_status != TS_OK) break;
        S.slot_busy[slot] = 1;
      }
      auto ws = std::make_shared<wstate>();
      ws->lo = lo;
      ws->hi = hi;
      ws->slot = slot;
      uint8_t* ds = dring + static_cast<uint64_t>(slot) * W;
      std::vector<std::tuple<size_t, uint64_t, uint64_t>> reads;
      std::vector<std::pair<uint64_t, uint64_t>> direct;  // ranges in page-locked files
      for (size_t k = 0; k < rc.files.size(); ++k) {
        const uint64_t a = std::max(lo, file_img[k].first);
        const uint64_t b = std::min(hi, file_img[k].first + file_img[k].second);
        if (b <= a) continue;
        if (regs.map[k]) {  // no pread: the copy engine reads the locked pages
          direct.push_back({a, b});
          continue;
        }
        for (uint64_t x = a; x < b; x += R) reads.emplace_back(k, x, std::min<uint64_t>(b, x + R));
      }
      ws->left = static_cast<int>(reads.size()) + 1;  // + this thread's part (page-locked ranges)
      for (const auto& rd : reads) {
        const size_t k = std::get<0>(rd);
        const uint64_t x = std::get<1>(rd), y = std::get<2>(rd);
        pool.submit([&, ws, k, x, y, ds] {
          const int pi = static_cast<int>(piece_seq.fetch_add(1) % static_cast<uint64_t>(P));
          try {
            std::lock_guard<std::mutex> pg(pmu[pi]);
            if (pused[pi]) cuda_check(cudaEventSynchronize(pev[pi]), "restore piece");
            uint8_t* hp = hring + static_cast<uint64_t>(pi) * R;
            bool ok = true;
            try {
              read_range(fds[k], hp, y - x, header_reserved + (x - file_img[k].first), rc.files[k].path,
                         &odirect_bytes);
              copy_host_tier(x, y, hp);
            } catch (const error& e) {
              set_err(e);
              ok = false;
            }
            std::lock_guard<std::mutex> g(cuda_mu);
            try {
              if (ok) {
                cuda_check(cudaMemcpyAsync(ds + (x - ws->lo), hp, y - x, cudaMemcpyHostToDevice, st),
                           "H2D piece");
                cuda_check(cudaEventRecord(pev[pi], st), "event");
                pused[pi] = 1;
              }
            } catch (const error& e) {
              set_err(e);
            }
            part_done(*ws);
          } catch (const error& e) {
            set_err(e);
          }
        });
      }
      try {
        for (const auto& [a, b] : direct) copy_host_tier(a, b, host_src(a, lo, nullptr));
        std::lock_guard<std::mutex> g(cuda_mu);
        try {
          for (const auto& [a, b] : direct)
            cuda_check(cudaMemcpyAsync(ds + (a - lo), host_src(a, lo, nullptr), b - a, cudaMemcpyHostToDevice, st),
                       "H2D window");
        } catch (const error& e) {
          set_err(e);
        }
        part_done(*ws);
      } catch (const error& e) {
        set_err(e);
      }
    }
  }  // pool joins: every read done, every window enqueued
  {
    std::unique_lock<std::mutex> g(S.mu);
    if (S.err_status == TS_OK) {
      S.cv.wait(g, [&] {
        if (S.err_status != TS_OK) return true;
        for (int k = 0; k < K; ++k)
          if (S.slot_busy[k]) return false;
        return true;
      });
    }
  }
  // (after a failure a window may never have been finished: drain the stream
  // so no copy still targets the staging)
  cudaStreamSynchronize(st);
  read_s = (now_ns() - r0) * 1e-9;
  uint32_t launches = launches_a.load();
  // Host-tier destinations: checksums over the restored host buffers, 4 chains per core.
  {
    std::vector<uint32_t> host_objs;
    for (uint32_t i = 0; i < objs.size(); ++i)
      if (objs[i].d->tier != TS_TIER_DEVICE) host_objs.push_back(i);
    for (uint32_t i : host_objs) {
      auto& o = objs[i];
      o.fnv = fnv1a64(o.d->data, o.size);
      o.hashed = o.size;
    }
  }
  cuda_check(cudaEventRecord(ev_b, st), "event");
  std::vector<uint64_t> dev_ck(dev_objs.size());
  if (S.err_status == TS_OK && next_fnv != nwin)
    fail(TS_ERR_GENERIC, "restore: device checksums did not cover every window");
  if (nf && S.err_status == TS_OK)
    cuda_check(cudaMemcpyAsync(dev_ck.data(), d_states, nf * 8ull, cudaMemcpyDeviceToHost, fst.s), "download");
  cuda_check(cudaStreamSynchronize(fst.s), "checksum stream");
  launches += launches_f.load();
  rtrace("pipeline done", t_begin);
  cuda_check(cudaStreamSynchronize(st), "restore stream");
  rtrace("device checksums done", t_begin);
  for (size_t i = 0; i < dev_objs.size(); ++i) {
    auto& o = objs[dev_objs[i]];
    o.fnv = dev_ck[i];
    o.hashed = o.size;
  }
  const float h2d_ms = elapsed_ms(ev_a, ev_b);
  float unpack_ms = 0;
  for (auto& ue : unpack_ev) unpack_ms += elapsed_ms(ue.first, ue.second);
  cudaEventDestroy(ev_a);
  cudaEventDestroy(ev_b);

  cudaStreamSynchronize(st);
  if (S.err_status != TS_OK) throw error(S.err_status, S.err, S.err_oid);
  rtrace("ring freed", t_begin);
  const int64_t t_verify = now_ns();
  for (const auto& o : objs)
    if (o.hashed != o.size || o.fnv != o.ck)
      fail(TS_ERR_CORRUPT_OBJECT, "checksum mismatch for object " + std::to_string(o.oid), static_cast<int64_t>(o.oid));

  // Structured objects: append-region pieces, checksum, decode (format.cpp:479-489).
  uint64_t ser_bytes = 0;
  for (size_t k = 0; k < rc.files.size(); ++k) {
    std::unordered_map<uint64_t, std::vector<const footer_entry*>> by_obj;
    for (const auto& e : rc.files[k].entries)
      if (e.kind != 0) by_obj[e.object_id].push_back(&e);
    for (auto& [oid, ps] : by_obj) {
      check_tiling(ps, oid);
      std::vector<uint8_t> bytes;
      for (const auto* e : ps) {
        const size_t at = bytes.size();
        bytes.resize(at + e->length);
        pread_all(fds[k].fd, bytes.data() + at, e->length, e->file_offset, rc.files[k].path);
      }
      if (fnv1a64(bytes.data(), bytes.size()) != ps.front()->checksum)
        fail(TS_ERR_CORRUPT_OBJECT, "checksum mismatch for object " + std::to_string(oid),
             static_cast<int64_t>(oid));
      try {
        rc.structured[oid] = decode(bytes.data(), bytes.size());
      } catch (const error& e) {
        fail(TS_ERR_CORRUPT_OBJECT, std::string("structured object does not decode: ") + e.what(),
             static_cast<int64_t>(oid));
      }
      ser_bytes += bytes.size();
    }
  }
  (void)mr;
  rtrace("structured done", t_begin);
  if (stats) {
    stats->bytes = raw_bytes + ser_bytes;
    stats->read_s = read_s;
    stats->verify_s = (now_ns() - t_verify) * 1e-9;
    stats->h2d_unpack_s = h2d_ms * 1e-3;
    stats->h2d_ms = h2d_ms;
    stats->direct_bytes = direct_bytes;
    stats->direct_io_bytes = odirect_bytes.load();
    stats->unpack_ms = unpack_ms;
    stats->total_s = (now_ns() - t_begin) * 1e-9;
    stats->kernel_launches = launches;
  }
}

// verify_checkpoint (format.cpp:496-529): full checksum pass, never throws.
void verify_checkpoint(const std::string& manifest_path, std::vector<std::pair<int, int64_t>>& issues,
                       uint64_t& files_checked, uint64_t& objects_checked) {
  files_checked = objects_checked = 0;
  manifest m;
  try {
    m = read_manifest(manifest_path);
  } catch (const error& e) {
    issues.push_back({e.status, e.object_id});
    return;
  }
  const auto slash = manifest_path.find_last_of('/');
  const std::string base = slash == std::string::npos ? "." : manifest_path.substr(0, slash);
  std::mutex mu;
  {
    thread_pool pool(static_cast<int>(std::min<unsigned>(16, std::max(2u, std::thread::hardware_concurrency()))));
    for (const auto& r : m.ranks) {
      for (const auto& mf : r.files) {
        pool.submit([&, path = base + "/" + mf.path, oids = mf.object_ids] {
          std::vector<std::pair<int, int64_t>> local;
          uint64_t nobj = 0;
          bool file_ok = false;
          try {
            uint64_t size = 0;
            auto entries = read_footer(path, &size);
            fd_holder fd;
            fd.fd = ::open(path.c_str(), O_RDONLY);
            if (fd.fd < 0) fail(TS_ERR_MISSING_FILE, "cannot open " + path);
            std::map<uint64_t, std::vector<const footer_entry*>> by_obj;
            for (const auto& e : entries) {
              if (e.file_offset + e.length > size)
                fail(TS_ERR_CORRUPT_FOOTER, "entry range outside the file", static_cast<int64_t>(e.object_id));
              by_obj[e.object_id].push_back(&e);
            }
            std::vector<uint8_t> buf(8ull << 20);
            for (auto& [oid, ps] : by_obj) {
              check_tiling(ps, oid);
              uint64_t h = fnv_seed;
              for (const auto* e : ps) {
                for (uint64_t x = 0; x < e->length; x += buf.size()) {
                  const uint64_t len = std::min<uint64_t>(buf.size(), e->length - x);
                  pread_all(fd.fd, buf.data(), len, e->file_offset + x, path);
                  h = fnv1a64(buf.data(), len, h);
                }
              }
              if (h != ps.front()->checksum)
                fail(TS_ERR_CORRUPT_OBJECT, "checksum mismatch for object " + std::to_string(oid),
                     static_cast<int64_t>(oid));
            }
            nobj = by_obj.size();
            file_ok = true;
            for (uint64_t oid : oids)
              if (!by_obj.count(oid)) local.push_back({TS_ERR_CORRUPT_FOOTER, static_cast<int64_t>(oid)});
          } catch (const error& e) {
            local.push_back({e.status, e.object_id});
          }
          std::lock_guard<std::mutex> g(mu);
          if (file_ok) {
            files_checked += 1;
            objects_checked += nobj;
          }
          issues.insert(issues.end(), local.begin(), local.end());
        });
      }
    }
  }
}

}  // namespace tsb
