// Probe: H2D straight from a pageable mapping of a tmpfs file (no pread, no
// registration): how fast does the driver's pageable path go, with 1-4 streams?
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/pageable_h2d_probe.cu -o tools/pageable_h2d_probe
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

int main() {
  const size_t n = 8ull << 30, chunk = 64 << 20;
  const char* path = "/dev/shm/pageable_probe.bin";
  int fd = ::open(path, O_RDWR | O_CREAT | O_TRUNC, 0644);
  if (ftruncate(fd, n) != 0) return 1;
  char* m = static_cast<char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
  std::memset(m, 3, n);
  cudaSetDevice(0);
  void* d;
  cudaMalloc(&d, n);
  for (int ns : {1, 2, 4}) {
    for (int rep = 0; rep < 2; ++rep) {
      std::vector<cudaStream_t> st(ns);
      for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int k = 0; k < ns; ++k)
        th.emplace_back([&, k] {
          cudaSetDevice(0);
          for (size_t o = k * chunk; o < n; o += ns * chunk)
            cudaMemcpyAsync(static_cast<char*>(d) + o, m + o, chunk, cudaMemcpyHostToDevice, st[k]);
          cudaStreamSynchronize(st[k]);
        });
      for (auto& t : th) t.join();
      const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::printf("{\"streams\": %d, \"rep\": %d, \"pageable_h2d_gbps\": %.1f}\n", ns, rep, n / s / 1e9);
      for (auto& x : st) cudaStreamDestroy(x);
    }
  }
  munmap(m, n);
  close(fd);
  unlink(path);
  return 0;
}
