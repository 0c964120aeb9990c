// Host file-write microbenchmark for the flush path (run on the GPU box):
// how fast can staged bytes land in one checkpoint file on tmpfs / local disk?
//   g++ -O2 -pthread tools/io_bench.cpp -o /tmp/io_bench && /tmp/io_bench /dev/shm 8
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/dev/shm";
  const size_t gb = argc > 2 ? std::stoul(argv[2]) : 8;
  const size_t total = gb << 30, chunk = 64 << 20;
  std::vector<char> src(total);
  for (size_t i = 0; i < total; i += 4096) src[i] = static_cast<char>(i);
  std::memset(src.data(), 7, total);
  auto path = [&](int k) { return dir + "/io_bench_" + std::to_string(k) + ".bin"; };
  auto report = [&](const char* what, int threads, double t) {
    std::printf("{\"test\": \"%s\", \"threads\": %d, \"GBps\": %.2f}\n", what, threads, total / t / 1e9);
    std::fflush(stdout);
  };
  for (int T : {1, 2, 4, 8, 16}) {
    // T threads pwrite disjoint ranges of ONE file
    int fd = open(path(0).c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
    if (ftruncate(fd, total) != 0) return 1;
    double t0 = now();
    std::vector<std::thread> th;
    for (int k = 0; k < T; ++k)
      th.emplace_back([&, k] {
        for (size_t off = k * chunk; off < total; off += T * chunk)
          if (pwrite(fd, src.data() + off, chunk, off) != (ssize_t)chunk) std::abort();
      });
    for (auto& x : th) x.join();
    report("pwrite_one_file", T, now() - t0);
    close(fd);
    unlink(path(0).c_str());
    // T threads memcpy into one MAP_SHARED mapping
    fd = open(path(0).c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
    if (ftruncate(fd, total) != 0) return 1;
    char* m = static_cast<char*>(mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
    t0 = now();
    th.clear();
    for (int k = 0; k < T; ++k)
      th.emplace_back([&, k] {
        for (size_t off = k * chunk; off < total; off += T * chunk) std::memcpy(m + off, src.data() + off, chunk);
      });
    for (auto& x : th) x.join();
    report("mmap_memcpy_one_file", T, now() - t0);
    munmap(m, total);
    close(fd);
    unlink(path(0).c_str());
    // T threads, one file each
    t0 = now();
    th.clear();
    for (int k = 0; k < T; ++k)
      th.emplace_back([&, k] {
        int f = open(path(k + 1).c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
        for (size_t off = k * chunk; off < total; off += T * chunk)
          if (pwrite(f, src.data() + off, chunk, off) != (ssize_t)chunk) std::abort();
        close(f);
      });
    for (auto& x : th) x.join();
    report("pwrite_file_per_thread", T, now() - t0);
    for (int k = 0; k < T; ++k) unlink(path(k + 1).c_str());
  }
  // page-cache read back speed (restore side): T threads pread
  {
    int fd = open(path(0).c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
    for (size_t off = 0; off < total; off += chunk) pwrite(fd, src.data() + off, chunk, off);
    for (int T : {1, 4, 16}) {
      double t0 = now();
      std::vector<std::thread> th;
      for (int k = 0; k < T; ++k)
        th.emplace_back([&, k] {
          for (size_t off = k * chunk; off < total; off += T * chunk) pread(fd, src.data() + off, chunk, off);
        });
      for (auto& x : th) x.join();
      report("pread_one_file", T, now() - t0);
    }
    close(fd);
    unlink(path(0).c_str());
  }
  return 0;
}
