#include "uring.hpp"

#include <linux/io_uring.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <cstring>
#include <memory>
#include <vector>

namespace tsb {

std::atomic<uint64_t> g_uring_ops{0};

namespace {
int sys_setup(unsigned entries, io_uring_params* p) {
  return static_cast<int>(::syscall(__NR_io_uring_setup, entries, p));
}
int sys_enter(int fd, unsigned to_submit, unsigned min_complete, unsigned flags) {
  return static_cast<int>(::syscall(__NR_io_uring_enter, fd, to_submit, min_complete, flags, nullptr, 0));
}
template <class T>
T* at(void* base, uint32_t off) {
  return reinterpret_cast<T*>(static_cast<uint8_t*>(base) + off);
}
}  // namespace

uring::uring(unsigned entries) {
  io_uring_params p;
  std::memset(&p, 0, sizeof p);
  const int fd = sys_setup(entries, &p);
  if (fd < 0) return;
  sq_entries_ = p.sq_entries;
  sq_ring_sz_ = p.sq_off.array + p.sq_entries * sizeof(unsigned);
  cq_ring_sz_ = p.cq_off.cqes + p.cq_entries * sizeof(io_uring_cqe);
  const bool single = (p.features & IORING_FEAT_SINGLE_MMAP) != 0;
  if (single) sq_ring_sz_ = cq_ring_sz_ = std::max(sq_ring_sz_, cq_ring_sz_);
  sq_ring_ = ::mmap(nullptr, sq_ring_sz_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, IORING_OFF_SQ_RING);
  if (sq_ring_ == MAP_FAILED) {
    sq_ring_ = nullptr;
    ::close(fd);
    return;
  }
  if (single) {
    cq_ring_ = sq_ring_;
  } else {
    cq_ring_ = ::mmap(nullptr, cq_ring_sz_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, IORING_OFF_CQ_RING);
    if (cq_ring_ == MAP_FAILED) {
      cq_ring_ = nullptr;
      ::munmap(sq_ring_, sq_ring_sz_);
      sq_ring_ = nullptr;
      ::close(fd);
      return;
    }
  }
  sqes_sz_ = p.sq_entries * sizeof(io_uring_sqe);
  sqes_ = ::mmap(nullptr, sqes_sz_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, IORING_OFF_SQES);
  if (sqes_ == MAP_FAILED) {
    sqes_ = nullptr;
    if (cq_ring_ != sq_ring_) ::munmap(cq_ring_, cq_ring_sz_);
    ::munmap(sq_ring_, sq_ring_sz_);
    sq_ring_ = cq_ring_ = nullptr;
    ::close(fd);
    return;
  }
  sq_head_ = at<unsigned>(sq_ring_, p.sq_off.head);
  sq_tail_ = at<unsigned>(sq_ring_, p.sq_off.tail);
  sq_mask_ = at<unsigned>(sq_ring_, p.sq_off.ring_mask);
  sq_array_ = at<unsigned>(sq_ring_, p.sq_off.array);
  cq_head_ = at<unsigned>(cq_ring_, p.cq_off.head);
  cq_tail_ = at<unsigned>(cq_ring_, p.cq_off.tail);
  cq_mask_ = at<unsigned>(cq_ring_, p.cq_off.ring_mask);
  cqes_ = at<void>(cq_ring_, p.cq_off.cqes);
  fd_ = fd;
}

uring::~uring() {
  if (sqes_) ::munmap(sqes_, sqes_sz_);
  if (cq_ring_ && cq_ring_ != sq_ring_) ::munmap(cq_ring_, cq_ring_sz_);
  if (sq_ring_) ::munmap(sq_ring_, sq_ring_sz_);
  if (fd_ >= 0) ::close(fd_);
}

bool uring::run(uring_op* ops, size_t n) {
  if (fd_ < 0) return false;
  auto* sqes = static_cast<io_uring_sqe*>(sqes_);
  auto* cqes = static_cast<io_uring_cqe*>(cqes_);
  size_t next = 0;
  while (next < n) {
    // one batch: fill up to depth() submission entries, submit, reap them all
    const unsigned batch = static_cast<unsigned>(std::min<size_t>(sq_entries_, n - next));
    unsigned tail = __atomic_load_n(sq_tail_, __ATOMIC_RELAXED);
    const unsigned mask = *sq_mask_;
    for (unsigned k = 0; k < batch; ++k) {
      const uring_op& o = ops[next + k];
      const unsigned idx = tail & mask;
      io_uring_sqe& e = sqes[idx];
      std::memset(&e, 0, sizeof e);
      e.opcode = o.write ? IORING_OP_WRITE : IORING_OP_READ;
      e.fd = o.fd;
      e.addr = reinterpret_cast<uint64_t>(o.buf);
      e.len = o.len;
      e.off = o.off;
      e.user_data = next + k;
      sq_array_[idx] = idx;
      ++tail;
    }
    __atomic_store_n(sq_tail_, tail, __ATOMIC_RELEASE);
    g_uring_ops.fetch_add(batch, std::memory_order_relaxed);
    unsigned reaped = 0, submitted = 0;
    while (reaped < batch) {
      const unsigned want_submit = batch - submitted;
      const int r = sys_enter(fd_, want_submit, 1, IORING_ENTER_GETEVENTS);
      if (r < 0) {
        if (errno == EINTR || errno == EAGAIN || errno == EBUSY) continue;
        return false;  // (the ring is unusable; ops not reaped are left unrun)
      }
      submitted += static_cast<unsigned>(r);
      unsigned head = __atomic_load_n(cq_head_, __ATOMIC_RELAXED);
      const unsigned ctail = __atomic_load_n(cq_tail_, __ATOMIC_ACQUIRE);
      for (; head != ctail; ++head, ++reaped) {
        const io_uring_cqe& c = cqes[head & *cq_mask_];
        ops[c.user_data].res = c.res;
      }
      __atomic_store_n(cq_head_, head, __ATOMIC_RELEASE);
    }
    next += batch;
  }
  return true;
}

uring* thread_uring() {
  static std::atomic<bool> unavailable{false};
  if (unavailable.load(std::memory_order_relaxed)) return nullptr;
  thread_local std::unique_ptr<uring> r;
  if (!r) {
    r = std::make_unique<uring>(32);
    if (!r->ok()) {
      r.reset();
      unavailable = true;
      return nullptr;
    }
  }
  return r.get();
}

namespace {
int64_t uring_rw(bool write, int fd, uint8_t* p, uint64_t n, uint64_t off, uint64_t piece) {
  uring* r = thread_uring();
  if (!r) return -1;
  piece = std::max<uint64_t>(4096, std::min<uint64_t>(piece, 1ull << 30));
  std::vector<uring_op> ops;
  ops.reserve(static_cast<size_t>((n + piece - 1) / piece));
  for (uint64_t d = 0; d < n; d += piece) {
    uring_op o;
    o.fd = fd;
    o.write = write;
    o.buf = p + d;
    o.len = static_cast<uint32_t>(std::min(piece, n - d));
    o.off = off + d;
    ops.push_back(o);
  }
  if (!r->run(ops.data(), ops.size())) return -1;
  int64_t done = 0;
  for (const auto& o : ops) {
    if (o.res < 0) break;
    done += o.res;
    if (static_cast<uint64_t>(o.res) < o.len) break;
  }
  return done;
}
}  // namespace

int64_t uring_pwrite(int fd, const void* p, uint64_t n, uint64_t off, uint64_t piece) {
  return uring_rw(true, fd, static_cast<uint8_t*>(const_cast<void*>(p)), n, off, piece);
}

int64_t uring_pread(int fd, void* p, uint64_t n, uint64_t off, uint64_t piece) {
  return uring_rw(false, fd, static_cast<uint8_t*>(p), n, off, piece);
}


uint64_t uring_ops() { return g_uring_ops.load(); }
bool uring_available() { return thread_uring() != nullptr; }

}  // namespace tsb
