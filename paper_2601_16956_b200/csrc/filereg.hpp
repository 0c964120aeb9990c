// Copy-engine DMA straight into checkpoint files (B200-side addition).
//
// The reference stages every chunk in a host cache and pwrite()s it
// (engine.cpp:258-307, 388-434; format.cpp:20-32): two host copies per byte on
// top of the device->host transfer. On tmpfs (/dev/shm) the page-cache pages of
// a file can be page-locked for the copy engines: cudaHostRegister of a
// MAP_SHARED mapping of [0, tensor_region_end). Then the D2H windows land
// directly in the file (measured 57 GB/s, = the pinned-pool rate), and the host
// never touches the fixed region.
//
// Registering costs ~10 GB/s of one host thread, so registrations are cached
// per inode and reused when checkpoint rotation recycles a file
// (retire_checkpoint + spare directory): the steady state pays nothing.
// Safety rules (locked pages must never be dropped from the file):
//  * a registration covers exactly [0, len); a file is reused only when the new
//    checkpoint's tensor_region_end equals len (truncating to >= len keeps every
//    locked page) and its size/mtime still match the stamp taken at our last
//    finalize (nobody else truncated or rewrote it);
//  * every opened file passes through claim() BEFORE it is truncated: a
//    mismatching registration is dropped first;
//  * registrations of unlinked files are dropped by sweep();
//  * only tmpfs files are registered (disk filesystems refuse long-term pins).
#pragma once

#include <sys/types.h>

#include <condition_variable>
#include <cstdint>
#include <atomic>
#include <map>
#include <mutex>
#include <set>
#include <string>

namespace tsb {

struct file_key {
  uint64_t dev = 0, ino = 0;
  bool operator<(const file_key& o) const { return dev != o.dev ? dev < o.dev : ino < o.ino; }
  bool valid() const { return dev != 0 || ino != 0; }
};

class file_registry {
 public:
  static file_registry& get();

  // `fd`: a file just opened for a new checkpoint with fixed region [0, len),
  // before its header is written or it is truncated. Returns the locked
  // mapping (device-visible host pointer) when a valid registration of exactly
  // [0, len) exists and is idle (it is then in use until release()); otherwise
  // drops any registration of the inode that the truncation could invalidate
  // and returns nullptr.
  uint8_t* claim(int fd, uint64_t len, file_key* key);
  // The claimed file was finalized (`ok`: new stamp from `fd`) or abandoned
  // (registration dropped).
  void release(const file_key& key, int fd, bool ok);
  // A finalized, unregistered file: true if the caller should now run
  // register_file(key, device) (the entry is created pending, stamped from fd).
  bool want_register(int fd, uint64_t len, file_key* key);
  // mmap + cudaHostRegister (slow: run on a worker thread).
  void register_file(const file_key& key, int device);
  // Restore side: the locked mapping of a file whose registration covers
  // exactly [0, len) and is intact (same checks as claim), pinned against
  // claims and drops until release_read(); nullptr otherwise. The copy engines
  // then read the fixed region straight from the page cache.
  const uint8_t* acquire_read(int fd, uint64_t len, file_key* key);
  void release_read(const file_key& key);
  // Drop registrations of files that no longer have a name.
  void sweep();
  // Drop every idle registration; returns bytes released.
  uint64_t release_all();
  uint64_t registered_bytes();
  // [registrations, ns inside cudaHostRegister, bytes registered,
  //  unregistrations, ns inside cudaHostUnregister + munmap] since start
  void stats(uint64_t out[5]);

 private:
  struct entry {
    int fd = -1;
    uint8_t* map = nullptr;
    uint64_t len = 0, maplen = 0;
    bool pending = false, stale = false, in_use = false;
    int readers = 0;
    int64_t size = -1, mtime_ns = -1;
  };
  void drop_locked(std::map<file_key, entry>::iterator it);
  std::atomic<uint64_t> stats_[5] = {{0}, {0}, {0}, {0}, {0}};
  std::mutex mu_;
  std::map<file_key, entry> m_;
  std::set<uint64_t> unsupported_dev_;  // filesystems whose pages cannot be locked
};

}  // namespace tsb
