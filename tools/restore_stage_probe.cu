// Probe: restore staging, tmpfs page cache -> pinned -> H2D, two shapes.
//   windows: the restore's current shape — K pinned windows of W bytes, 16
//            threads pread each window in 16 MiB pieces, then one H2D per
//            window (the DMA reads the window from DRAM: it was written long
//            before).
//   pieces:  a small pool of P pinned pieces of R bytes (P*R well inside the
//            60 MiB L3); each thread preads a piece and enqueues its H2D at
//            once, so the copy engine may read it from the LLC (PCIe reads
//            are coherent) instead of DRAM: host DRAM traffic 2 passes
//            instead of 3.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/restore_stage_probe.cu -o tools/restore_stage_probe
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static void pread_all(int fd, char* p, size_t n, size_t off) {
  while (n) {
    ssize_t r = ::pread(fd, p, n, off);
    if (r <= 0) { std::perror("pread"); std::exit(1); }
    p += r; n -= r; off += r;
  }
}

int main(int argc, char** argv) {
  const size_t n = (argc > 1 ? std::atoll(argv[1]) : 16) << 30;
  const char* path = "/dev/shm/restore_stage_probe.bin";
  int fd = ::open(path, O_RDWR | O_CREAT | O_TRUNC, 0644);
  {
    std::vector<char> buf(64 << 20, 7);
    for (size_t o = 0; o < n; o += buf.size()) {
      for (size_t k = 0; k < buf.size(); k += 4096) buf[k] = static_cast<char>(o >> 20);
      if (::pwrite(fd, buf.data(), buf.size(), o) != static_cast<ssize_t>(buf.size())) return 1;
    }
  }
  cudaSetDevice(0);
  char* d;
  if (cudaMalloc(&d, n) != cudaSuccess) return 2;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int nth = 16;

  // windows
  for (int rep = 0; rep < 2; ++rep) {
    const size_t W = 1ull << 30, piece = 16 << 20;
    const int K = 4;
    char* h;
    cudaHostAlloc(reinterpret_cast<void**>(&h), W * K, cudaHostAllocDefault);
    std::vector<cudaEvent_t> ev(K);
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    std::vector<int> used(K, 0);
    const double t0 = now();
    for (size_t lo = 0, w = 0; lo < n; lo += W, ++w) {
      const int s = w % K;
      if (used[s]) cudaEventSynchronize(ev[s]);
      used[s] = 1;
      char* hs = h + s * W;
      std::atomic<size_t> next{lo};
      std::vector<std::thread> th;
      for (int t = 0; t < nth; ++t)
        th.emplace_back([&] {
          for (;;) {
            size_t x = next.fetch_add(piece);
            if (x >= lo + W || x >= n) return;
            pread_all(fd, hs + (x - lo), std::min(piece, std::min(lo + W, n) - x), x);
          }
        });
      for (auto& x : th) x.join();
      cudaMemcpyAsync(d + lo, hs, std::min(W, n - lo), cudaMemcpyHostToDevice, st);
      cudaEventRecord(ev[s], st);
    }
    cudaStreamSynchronize(st);
    const double dt = now() - t0;
    std::printf("{\"shape\": \"windows\", \"W_mb\": 1024, \"K\": 4, \"rep\": %d, \"gbps\": %.2f}\n", rep, n / dt / 1e9);
    std::fflush(stdout);
    for (auto& e : ev) cudaEventDestroy(e);
    cudaFreeHost(h);
  }

  // pieces
  for (size_t R : {512ull << 10, 1ull << 20, 2ull << 20, 4ull << 20}) {
    for (int P : {16, 32, 64}) {
      char* h;
      cudaHostAlloc(reinterpret_cast<void**>(&h), R * P, cudaHostAllocDefault);
      // piece k serves chunks k, k+P, ...: its mutex is held from acquire to
      // the H2D's event record; the next user waits for that event
      std::vector<std::mutex> pmu(P);
      std::vector<cudaEvent_t> pev(P);
      for (auto& e : pev) {
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        cudaEventRecord(e, st);
      }
      std::mutex cuda_mu;
      std::atomic<size_t> next{0};
      const double t0 = now();
      std::vector<std::thread> th;
      for (int t = 0; t < nth; ++t)
        th.emplace_back([&] {
          cudaSetDevice(0);
          for (;;) {
            const size_t i = next.fetch_add(1);
            const size_t x = i * R;
            if (x >= n) return;
            const int k = static_cast<int>(i % P);
            std::lock_guard<std::mutex> pg(pmu[k]);
            cudaEventSynchronize(pev[k]);
            const size_t len = std::min(R, n - x);
            pread_all(fd, h + k * R, len, x);
            std::lock_guard<std::mutex> g(cuda_mu);
            cudaMemcpyAsync(d + x, h + k * R, len, cudaMemcpyHostToDevice, st);
            cudaEventRecord(pev[k], st);
          }
        });
      for (auto& x : th) x.join();
      cudaStreamSynchronize(st);
      const double dt = now() - t0;
      std::printf("{\"shape\": \"pieces\", \"R_mb\": %zu, \"P\": %d, \"inflight_mb\": %zu, \"gbps\": %.2f}\n", R >> 20, P,
                  (R * P) >> 20, n / dt / 1e9);
      std::fflush(stdout);
      for (auto& e : pev) cudaEventDestroy(e);
      cudaFreeHost(h);
    }
  }
  // check a few bytes
  char probe[2];
  cudaMemcpy(probe, d + (n / 2), 1, cudaMemcpyDeviceToHost);
  cudaFree(d);
  ::close(fd);
  ::unlink(path);
  return 0;
}
