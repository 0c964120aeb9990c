// Minimal io_uring (raw io_uring_setup / io_uring_enter syscalls, no liburing)
// for the kernel-bypass flush and restore reads (the paper's
// engine uses liburing + O_DIRECT). One ring per thread: a
// flush worker submits the O_DIRECT body of a staging window as a batch of
// positional writes and reaps them together, so the device queue sees the
// whole window at once instead of one pwrite(2) at a time.
#pragma once

#include <cstddef>
#include <cstdint>

namespace tsb {

struct uring_op {
  int fd = -1;
  bool write = true;
  void* buf = nullptr;
  uint32_t len = 0;
  uint64_t off = 0;
  int64_t res = 0;  // bytes transferred, or -errno
};

class uring {
 public:
  explicit uring(unsigned entries);
  ~uring();
  uring(const uring&) = delete;
  uring& operator=(const uring&) = delete;
  bool ok() const { return fd_ >= 0; }
  unsigned depth() const { return sq_entries_; }
  // Submits every op (in batches of at most depth()) and waits for all of
  // them; fills res. Returns false when the ring itself failed (ops not run).
  bool run(uring_op* ops, size_t n);

 private:
  int fd_ = -1;
  unsigned sq_entries_ = 0;
  void* sq_ring_ = nullptr;
  void* cq_ring_ = nullptr;
  void* sqes_ = nullptr;
  size_t sq_ring_sz_ = 0, cq_ring_sz_ = 0, sqes_sz_ = 0;
  unsigned *sq_head_ = nullptr, *sq_tail_ = nullptr, *sq_mask_ = nullptr, *sq_array_ = nullptr;
  unsigned *cq_head_ = nullptr, *cq_tail_ = nullptr, *cq_mask_ = nullptr;
  void* cqes_ = nullptr;
};

// This thread's ring (created on first use), or nullptr when io_uring is not
// available here (seccomp, io_uring_disabled, old kernel): callers fall back
// to pread/pwrite.
uring* thread_uring();

// Positional write / read of [off, off+n) through the thread's ring, cut in
// `piece`-byte requests all in flight together. Returns the bytes done in
// order from the start (short on the first failed or short request), or -1
// when no ring is available.
int64_t uring_pwrite(int fd, const void* p, uint64_t n, uint64_t off, uint64_t piece);
int64_t uring_pread(int fd, void* p, uint64_t n, uint64_t off, uint64_t piece);

// Requests submitted through any ring of the process (diagnostics / tests).
uint64_t uring_ops();
bool uring_available();

}  // namespace tsb
