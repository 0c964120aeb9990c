// Probe: does cudaHostRegister of a tmpfs file mapping scale with threads
// (disjoint ranges registered concurrently), and does a read-only registration
// (for restore: H2D straight from the page cache) cost less? JSON lines.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/reg_scaling_probe.cu -o tools/reg_scaling_probe
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t G = 1ull << 30, n = 16 * G;
  cudaSetDevice(0);
  cudaFree(nullptr);
  const char* path = "/dev/shm/reg_probe.bin";
  int fd = ::open(path, O_RDWR | O_CREAT | O_TRUNC, 0644);
  if (ftruncate(fd, n) != 0) return 1;
  {
    void* m = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    std::memset(m, 1, n);  // populate the page cache
    munmap(m, n);
  }
  void* dbuf;
  cudaMalloc(&dbuf, n);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int threads : {1, 2, 4, 8, 16}) {
    for (int ro = 0; ro < 2; ++ro) {
      void* m = mmap(nullptr, n, ro ? PROT_READ : PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      const unsigned flags = cudaHostRegisterPortable | (ro ? cudaHostRegisterReadOnly : 0);
      const size_t part = n / threads;
      std::vector<std::thread> th;
      std::vector<int> ok(threads, 0);
      const double t0 = now();
      for (int k = 0; k < threads; ++k)
        th.emplace_back([&, k] {
          cudaSetDevice(0);
          ok[k] = cudaHostRegister(static_cast<char*>(m) + k * part, part, flags) == cudaSuccess;
        });
      for (auto& t : th) t.join();
      const double dt = now() - t0;
      int good = 0;
      for (int v : ok) good += v;
      double h2d = 0;
      if (good == threads) {  // H2D from the registered page cache
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (size_t o = 0; o < n; o += 64 << 20)
          cudaMemcpyAsync(static_cast<char*>(dbuf) + o, static_cast<char*>(m) + o, 64 << 20, cudaMemcpyHostToDevice, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        h2d = n / (ms / 1e3) / 1e9;
      }
      const double u0 = now();
      for (int k = 0; k < threads; ++k) cudaHostUnregister(static_cast<char*>(m) + k * part);
      const double du = now() - u0;
      cudaGetLastError();
      munmap(m, n);
      std::printf("{\"threads\": %d, \"read_only\": %d, \"ok\": %d, \"register_s\": %.3f, \"register_gbps\": %.1f, "
                  "\"h2d_gbps\": %.1f, \"unregister_s\": %.3f}\n",
                  threads, ro, good, dt, n / dt / 1e9, h2d, du);
      std::fflush(stdout);
    }
  }
  close(fd);
  unlink(path);
  return 0;
}
