// Host memory-bandwidth probe: what bounds the page-cache restore path
// (pread from tmpfs into the pinned ring = a kernel memcpy) on this box.
//   g++ -O2 -pthread tools/membw_probe.cpp -o tools/membw_probe && tools/membw_probe [GiB]
// Prints one JSON line per (kind, threads): memcpy between two private
// buffers, and pread of a tmpfs file into a buffer.
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const size_t gib = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 8;
  const size_t n = gib << 30;
  auto* a = static_cast<unsigned char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_POPULATE, -1, 0));
  auto* b = static_cast<unsigned char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_POPULATE, -1, 0));
  if (a == MAP_FAILED || b == MAP_FAILED) return 1;
  std::memset(a, 1, n);
  std::memset(b, 2, n);
  const char* path = "/dev/shm/membw_probe.bin";
  int fd = open(path, O_RDWR | O_CREAT | O_TRUNC, 0644);
  if (fd < 0 || ftruncate(fd, static_cast<off_t>(n)) != 0) return 2;
  for (size_t o = 0; o < n; o += 1 << 26) pwrite(fd, a + o, 1 << 26, static_cast<off_t>(o));
  for (int kind = 0; kind < 2; ++kind) {
    for (int t : {1, 2, 4, 8, 12, 16}) {
      const size_t per = n / t;
      std::vector<std::thread> th;
      const double t0 = now();
      for (int i = 0; i < t; ++i)
        th.emplace_back([&, i] {
          const size_t lo = per * i;
          for (size_t o = 0; o < per; o += 16 << 20) {
            const size_t k = std::min<size_t>(16 << 20, per - o);
            if (kind == 0) std::memcpy(b + lo + o, a + lo + o, k);
            else if (pread(fd, b + lo + o, k, static_cast<off_t>(lo + o)) != static_cast<ssize_t>(k)) std::abort();
          }
        });
      for (auto& x : th) x.join();
      const double dt = now() - t0;
      std::printf("{\"kind\": \"%s\", \"threads\": %d, \"gb\": %.1f, \"gbps\": %.2f}\n",
                  kind == 0 ? "memcpy" : "pread_tmpfs", t, n / 1e9, n / dt / 1e9);
      std::fflush(stdout);
    }
  }
  close(fd);
  unlink(path);
  return 0;
}
