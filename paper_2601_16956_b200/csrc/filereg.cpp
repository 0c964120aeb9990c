// Registry of page-locked checkpoint-file mappings (see filereg.hpp).
#include "filereg.hpp"
#include "core.hpp"

#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/vfs.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>

namespace tsb {

namespace {
const bool g_trace = std::getenv("TS_TRACE") != nullptr;
#define FTRACE(...)                        \
  do {                                     \
    if (g_trace) {                         \
      std::fprintf(stderr, "[ts filereg] "); \
      std::fprintf(stderr, __VA_ARGS__);   \
      std::fprintf(stderr, "\n");          \
    }                                      \
  } while (0)
struct file_stat {
  file_key key;
  int64_t size = -1, mtime_ns = -1, nlink = 0;
};
bool stat_fd(int fd, file_stat* s) {
  struct stat st;
  if (fd < 0 || ::fstat(fd, &st) != 0) return false;
  s->key.dev = static_cast<uint64_t>(st.st_dev);
  s->key.ino = static_cast<uint64_t>(st.st_ino);
  s->size = static_cast<int64_t>(st.st_size);
  s->mtime_ns = static_cast<int64_t>(st.st_mtim.tv_sec) * 1000000000ll + st.st_mtim.tv_nsec;
  s->nlink = static_cast<int64_t>(st.st_nlink);
  return true;
}
uint64_t page_up(uint64_t n) { return (n + 4095) & ~4095ull; }

// Locking populated every PTE of our (never CPU-touched) mapping; a truncation
// or hole punch by anyone zaps the PTEs of the dropped pages. So a registration
// is intact only while the sampled pages (first, last, 6 in between) are still
// present in /proc/self/pagemap (bit 63; needs no privilege). Truncating below
// len always drops the last page.
bool pages_present(const uint8_t* map, uint64_t maplen) {
  const int fd = ::open("/proc/self/pagemap", O_RDONLY);
  if (fd < 0) return true;  // no pagemap: size/mtime stamp only
  const uint64_t np = maplen / 4096;
  bool ok = true;
  for (int k = 0; k < 8 && ok; ++k) {
    const uint64_t pg = k == 7 ? np - 1 : np * k / 7;
    const uint64_t vpn = reinterpret_cast<uintptr_t>(map) / 4096 + pg;
    uint64_t e = 0;
    if (::pread(fd, &e, 8, static_cast<off_t>(vpn * 8)) == 8) ok = (e >> 63) & 1;
  }
  ::close(fd);
  return ok;
}
}  // namespace

file_registry& file_registry::get() {
  // Never destroyed: no CUDA calls from static destructors at process exit
  // (the OS releases locked pages with the process).
  static file_registry* r = new file_registry;
  return *r;
}

void file_registry::drop_locked(std::map<file_key, entry>::iterator it) {
  entry& e = it->second;
  if (e.map) {
    const int64_t t0 = now_ns();
    cudaHostUnregister(e.map);
    cudaGetLastError();
    ::munmap(e.map, e.maplen);
    stats_[3] += 1;
    stats_[4] += static_cast<uint64_t>(now_ns() - t0);
  }
  if (e.fd >= 0) ::close(e.fd);
  m_.erase(it);
}

uint8_t* file_registry::claim(int fd, uint64_t len, file_key* key) {
  file_stat s;
  if (!stat_fd(fd, &s)) return nullptr;
  *key = s.key;
  std::lock_guard<std::mutex> g(mu_);
  auto it = m_.find(s.key);
  if (it == m_.end()) return nullptr;
  entry& e = it->second;
  if (e.in_use || e.readers > 0) return nullptr;  // (a restore is reading it: leave it alone)
  if (e.pending) {
    FTRACE("claim ino=%llu pending", (unsigned long long)s.key.ino);
    // Still being registered: not usable now. Truncation to >= len keeps the
    // pages being locked; anything else makes the registration useless.
    if (e.len != len) e.stale = true;
    return nullptr;
  }
  const bool present = e.len == len && pages_present(e.map, e.maplen);
  if (e.len != len || e.size != s.size || e.mtime_ns != s.mtime_ns || !present) {
    FTRACE("claim ino=%llu dropped: len %llu/%llu size %lld/%lld mtime %lld/%lld present %d",
           (unsigned long long)s.key.ino, (unsigned long long)e.len, (unsigned long long)len, (long long)e.size,
           (long long)s.size, (long long)e.mtime_ns, (long long)s.mtime_ns, (int)present);
    drop_locked(it);
    return nullptr;
  }
  FTRACE("claim ino=%llu ok len=%llu", (unsigned long long)s.key.ino, (unsigned long long)len);
  e.in_use = true;
  return e.map;
}

const uint8_t* file_registry::acquire_read(int fd, uint64_t len, file_key* key) {
  file_stat s;
  if (!stat_fd(fd, &s)) return nullptr;
  *key = s.key;
  std::lock_guard<std::mutex> g(mu_);
  auto it = m_.find(s.key);
  if (it == m_.end()) return nullptr;
  entry& e = it->second;
  if (e.pending || e.in_use || e.len != len || e.size != s.size || e.mtime_ns != s.mtime_ns ||
      !pages_present(e.map, e.maplen))
    return nullptr;
  e.readers += 1;
  return e.map;
}

void file_registry::release_read(const file_key& key) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = m_.find(key);
  if (it != m_.end() && it->second.readers > 0) it->second.readers -= 1;
}

void file_registry::release(const file_key& key, int fd, bool ok) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = m_.find(key);
  if (it == m_.end()) return;
  entry& e = it->second;
  e.in_use = false;
  file_stat s;
  if (!ok || !stat_fd(fd, &s) || !(s.key.dev == key.dev && s.key.ino == key.ino)) {
    drop_locked(it);
    return;
  }
  e.size = s.size;
  e.mtime_ns = s.mtime_ns;
}

bool file_registry::want_register(int fd, uint64_t len, file_key* key) {
  file_stat s;
  if (!stat_fd(fd, &s)) return false;
  std::lock_guard<std::mutex> g(mu_);
  if (unsupported_dev_.count(s.key.dev)) return false;
  // Only shmem pages can be pinned long term for writing (disk filesystems
  // track dirty pages and refuse); do not even try elsewhere.
  struct statfs fs;
  constexpr long kTmpfsMagic = 0x01021994;
  if (::fstatfs(fd, &fs) != 0 || static_cast<long>(fs.f_type) != kTmpfsMagic) {
    unsupported_dev_.insert(s.key.dev);
    return false;
  }
  auto it = m_.find(s.key);
  if (it != m_.end()) {
    entry& e = it->second;
    if (e.in_use || e.readers > 0) return false;
    if (e.pending) {
      if (e.len != len) e.stale = true;
      else e.size = s.size, e.mtime_ns = s.mtime_ns;  // rewritten by us while being locked
      return false;
    }
    if (e.len == len) {  // written through the pool path this time: refresh the stamp
      e.size = s.size;
      e.mtime_ns = s.mtime_ns;
      return false;
    }
    drop_locked(it);
  }
  const int dfd = ::dup(fd);
  if (dfd < 0) return false;
  entry e;
  e.fd = dfd;
  e.len = len;
  e.pending = true;
  e.size = s.size;
  e.mtime_ns = s.mtime_ns;
  m_.emplace(s.key, e);
  *key = s.key;
  FTRACE("want_register ino=%llu len=%llu", (unsigned long long)s.key.ino, (unsigned long long)len);
  return true;
}

void file_registry::register_file(const file_key& key, int device) {
  int fd;
  uint64_t len;
  {
    std::lock_guard<std::mutex> g(mu_);
    auto it = m_.find(key);
    if (it == m_.end() || !it->second.pending) return;
    fd = it->second.fd;
    len = it->second.len;
  }
  cudaSetDevice(device);
  const uint64_t ml = page_up(len);
  file_stat s;
  // (a file cut below len meanwhile, e.g. recycled for a smaller layout, cannot be locked)
  bool ok = stat_fd(fd, &s) && static_cast<uint64_t>(s.size) >= len;
  void* m = ok ? ::mmap(nullptr, ml, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0) : MAP_FAILED;
  ok = m != MAP_FAILED;
  bool refused = false;
  const int64_t t_reg = now_ns();
  const bool reg_ok = ok && cudaHostRegister(m, ml, cudaHostRegisterPortable | cudaHostRegisterMapped) == cudaSuccess;
  if (ok) {
    stats_[0] += 1;
    stats_[1] += static_cast<uint64_t>(now_ns() - t_reg);
    if (reg_ok) stats_[2] += ml;
  }
  if (ok && !reg_ok) {
    cudaGetLastError();
    ::munmap(m, ml);
    ok = false;
    refused = stat_fd(fd, &s) && static_cast<uint64_t>(s.size) >= len;  // not explained by a truncation
  }
  FTRACE("register ino=%llu len=%llu ok=%d refused=%d", (unsigned long long)key.ino, (unsigned long long)len,
         (int)ok, (int)refused);
  std::lock_guard<std::mutex> g(mu_);
  auto it = m_.find(key);  // pending entries are only removed here
  entry& e = it->second;
  e.pending = false;
  if (!ok) {
    if (refused && !e.stale) unsupported_dev_.insert(key.dev);  // e.g. a disk filesystem
    drop_locked(it);
    return;
  }
  e.map = static_cast<uint8_t*>(m);
  e.maplen = ml;
  // Locking write-faults the shared mapping, which bumps mtime: stamp again
  // (the size must not have moved meanwhile).
  file_stat s2;
  if (e.stale || !stat_fd(fd, &s2) || s2.size != e.size) {
    drop_locked(it);
    return;
  }
  e.mtime_ns = s2.mtime_ns;
}

void file_registry::sweep() {
  std::lock_guard<std::mutex> g(mu_);
  for (auto it = m_.begin(); it != m_.end();) {
    auto cur = it++;
    const entry& e = cur->second;
    if (e.pending || e.in_use || e.readers > 0) continue;
    file_stat s;
    if (!stat_fd(e.fd, &s) || s.nlink == 0) drop_locked(cur);
  }
}

uint64_t file_registry::release_all() {
  std::lock_guard<std::mutex> g(mu_);
  uint64_t bytes = 0;
  for (auto it = m_.begin(); it != m_.end();) {
    auto cur = it++;
    if (cur->second.pending || cur->second.in_use || cur->second.readers > 0) continue;
    bytes += cur->second.maplen;
    drop_locked(cur);
  }
  return bytes;
}

uint64_t file_registry::registered_bytes() {
  std::lock_guard<std::mutex> g(mu_);
  uint64_t b = 0;
  for (const auto& kv : m_) b += kv.second.maplen;
  return b;
}

}  // namespace tsb

namespace tsb {
void file_registry::stats(uint64_t out[5]) {
  for (int i = 0; i < 5; ++i) out[i] = stats_[i].load();
}
}  // namespace tsb
