// Worker thread pool and the bounded pinned staging pool (staging.cpp:10-115
// semantics over cudaHostAlloc memory). See engine.hpp.
#include <algorithm>
#include <chrono>
#include <cstdio>

#include "engine.hpp"

namespace tsb {

namespace {
std::chrono::steady_clock::time_point to_tp(int64_t ns) {
  return std::chrono::steady_clock::time_point(std::chrono::nanoseconds(ns));
}
}  // namespace

// ---------------------------------------------------------------------------
// thread pool

thread_pool::thread_pool(int n, std::function<void()> init) {
  for (int i = 0; i < std::max(1, n); ++i)
    threads_.emplace_back([this, init] {
      if (init) init();
      for (;;) {
        std::function<void()> f;
        {
          std::unique_lock<std::mutex> g(mu_);
          cv_.wait(g, [&] { return stop_ || !q_.empty(); });
          if (q_.empty()) return;
          f = std::move(q_.front());
          q_.pop_front();
        }
        f();
      }
    });
}

thread_pool::~thread_pool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : threads_) t.join();
}

void thread_pool::submit(std::function<void()> f) {
  {
    std::lock_guard<std::mutex> g(mu_);
    q_.push_back([f = std::move(f)] {
      try {
        f();
      } catch (const std::exception& e) {
        std::fprintf(stderr, "ts_b200: uncaught exception in worker task: %s\n", e.what());
      }
    });
  }
  cv_.notify_one();
}

// ---------------------------------------------------------------------------
// pinned pool (staging.cpp:10-115 semantics over cudaHostAlloc memory)

pinned_pool::pinned_pool(uint64_t capacity) : capacity_(capacity) {
  if (capacity == 0) fail(TS_ERR_GENERIC, "staging cache: zero capacity");
  void* p = nullptr;
  cuda_check(cudaHostAlloc(&p, capacity, cudaHostAllocPortable | cudaHostAllocMapped),
             "cudaHostAlloc(staging pool)");
  base_ = static_cast<uint8_t*>(p);
}

pinned_pool::~pinned_pool() {
  if (base_) cudaFreeHost(base_);
}

bool pinned_pool::find_locked(uint64_t size, uint64_t* off) const {
  auto free_at = [&](uint64_t start) {
    if (start + size > capacity_) return false;
    auto it = live_.lower_bound(start);
    if (it != live_.end() && it->first < start + size) return false;
    if (it != live_.begin()) {
      auto prev = std::prev(it);
      if (prev->first + prev->second > start) return false;
    }
    return true;
  };
  if (free_at(bump_)) return *off = bump_, true;
  if (free_at(0)) return *off = 0, true;
  uint64_t cursor = 0;
  for (const auto& [o, l] : live_) {
    if (o >= cursor && o - cursor >= size) return *off = cursor, true;
    cursor = std::max(cursor, o + l);
  }
  if (capacity_ - cursor >= size) return *off = cursor, true;
  return false;
}

pinned_pool::region pinned_pool::acquire(uint64_t size, int64_t deadline_ns) {
  if (size == 0) fail(TS_ERR_GENERIC, "staging cache: zero-size acquire");
  if (size > capacity_) fail(TS_ERR_GENERIC, "staging cache: oversized request");
  std::unique_lock<std::mutex> g(mu_);
  const uint64_t token = next_token_++;
  waiters_.push_back(token);
  for (;;) {
    uint64_t off;
    if (waiters_.front() == token && find_locked(size, &off)) {
      waiters_.pop_front();
      live_.emplace(off, size);
      allocated_ += size;
      peak_ = std::max(peak_, allocated_);
      bump_ = (off + size) % capacity_;
      cv_.notify_all();
      return {next_id_++, off, size};
    }
    if (deadline_ns >= 0) {
      if (now_ns() >= deadline_ns) {
        waiters_.erase(std::find(waiters_.begin(), waiters_.end(), token));
        cv_.notify_all();
        fail(TS_ERR_CACHE_TIMEOUT, "staging cache: acquire deadline exceeded");
      }
      cv_.wait_until(g, to_tp(deadline_ns));
    } else {
      cv_.wait(g);
    }
  }
}

void pinned_pool::release(const region& r) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = live_.find(r.offset);
  if (it == live_.end()) fail(TS_ERR_GENERIC, "staging cache: release of unknown or freed region");
  allocated_ -= it->second;
  live_.erase(it);
  cv_.notify_all();
}

}  // namespace tsb
