// Probe: pinned D2H bandwidth with 1, 2, 4 concurrent streams (copy engines).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/d2h_streams_probe.cu -o tools/d2h_streams_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

int main() {
  const size_t n = 8ull << 30, chunk = 64 << 20;
  cudaSetDevice(0);
  void *d, *h;
  cudaMalloc(&d, n);
  cudaHostAlloc(&h, n, cudaHostAllocPortable);
  cudaMemset(d, 1, n);
  cudaDeviceSynchronize();
  for (int dir = 0; dir < 2; ++dir)
    for (int ns : {1, 2, 4}) {
      std::vector<cudaStream_t> st(ns);
      for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaDeviceSynchronize();
        cudaEventRecord(a, st[0]);
        for (int k = 1; k < ns; ++k) cudaStreamWaitEvent(st[k], a, 0);
        size_t i = 0;
        for (size_t o = 0; o < n; o += chunk, ++i) {
          if (dir == 0)
            cudaMemcpyAsync(static_cast<char*>(h) + o, static_cast<char*>(d) + o, chunk, cudaMemcpyDeviceToHost, st[i % ns]);
          else
            cudaMemcpyAsync(static_cast<char*>(d) + o, static_cast<char*>(h) + o, chunk, cudaMemcpyHostToDevice, st[i % ns]);
        }
        for (int k = 1; k < ns; ++k) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          cudaEventRecord(e, st[k]);
          cudaStreamWaitEvent(st[0], e, 0);
        }
        cudaEventRecord(b, st[0]);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) std::printf("{\"dir\": \"%s\", \"streams\": %d, \"gbps\": %.1f}\n", dir ? "h2d" : "d2h", ns, n / (ms / 1e3) / 1e9);
      }
    }
  return 0;
}
