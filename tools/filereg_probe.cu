// Probe: can the copy engine DMA straight into the page cache of a checkpoint
// file on tmpfs (cudaHostRegister of a MAP_SHARED mapping), and what do
// registration and D2H cost? Prints one JSON line per measurement.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/filereg_probe.cu -o tools/filereg_probe
//   tools/filereg_probe /dev/shm/probe.bin 8
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::printf("{\"error\": \"%s\", \"at\": \"%s\"}\n", cudaGetErrorString(e_), #x); \
    }                                                                              \
  } while (0)

static double d2h(void* dst, const void* src, size_t n, size_t chunk, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (size_t o = 0; o < n; o += chunk)
    CK(cudaMemcpyAsync((char*)dst + o, (const char*)src + o, std::min(chunk, n - o), cudaMemcpyDeviceToHost, s));
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return n / (ms / 1e3) / 1e9;
}

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "/dev/shm/probe.bin";
  const size_t gib = argc > 2 ? std::atoi(argv[2]) : 8;
  const size_t n = gib << 30, chunk = 64 << 20;
  cudaSetDevice(0);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  void* dsrc;
  CK(cudaMalloc(&dsrc, n));
  CK(cudaMemset(dsrc, 0x5a, n));
  cudaDeviceSynchronize();

  // reference: cudaHostAlloc pool
  void* pin;
  double t = now();
  CK(cudaHostAlloc(&pin, n, cudaHostAllocPortable | cudaHostAllocMapped));
  std::printf("{\"what\": \"cudaHostAlloc\", \"s\": %.3f, \"gbps_alloc\": %.2f}\n", now() - t, n / (now() - t) / 1e9);
  d2h(pin, dsrc, n, chunk, s);
  std::printf("{\"what\": \"d2h_hostalloc\", \"gbps\": %.2f}\n", d2h(pin, dsrc, n, chunk, s));

  for (int round = 0; round < 3; ++round) {
    int fd = ::open(path, O_RDWR | O_CREAT, 0644);
    if (round == 0) ftruncate(fd, 0);
    ftruncate(fd, n);
    void* m = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    t = now();
    int pr = madvise(m, n, MADV_POPULATE_WRITE);
    const double tpop = now() - t;
    t = now();
    cudaError_t e = cudaHostRegister(m, n, cudaHostRegisterPortable);
    const double treg = now() - t;
    std::printf("{\"what\": \"register_file_mapping\", \"round\": %d, \"populate_rc\": %d, \"populate_s\": %.3f, "
                "\"register\": \"%s\", \"register_s\": %.3f, \"register_gbps\": %.2f}\n",
                round, pr, tpop, cudaGetErrorString(e), treg, n / treg / 1e9);
    if (e == cudaSuccess) {
      double g1 = d2h(m, dsrc, n, chunk, s);
      double g2 = d2h(m, dsrc, n, chunk, s);
      // check the bytes reached the file
      unsigned char buf[16];
      pread(fd, buf, 16, n - 16);
      std::printf("{\"what\": \"d2h_into_file_pages\", \"round\": %d, \"gbps\": [%.2f, %.2f], \"tail_ok\": %d}\n", round,
                  g1, g2, buf[0] == 0x5a && buf[15] == 0x5a);
      t = now();
      cudaHostUnregister(m);
      std::printf("{\"what\": \"unregister\", \"s\": %.3f}\n", now() - t);
    } else {
      cudaGetLastError();
      // pageable fallback: driver-staged copy into the mapping
      std::printf("{\"what\": \"d2h_pageable_mapping\", \"gbps\": %.2f}\n", d2h(m, dsrc, n, chunk, s));
    }
    t = now();
    munmap(m, n);
    std::printf("{\"what\": \"munmap\", \"s\": %.3f}\n", now() - t);
    close(fd);
  }
  // memcpy reference: pinned -> file mapping (the current flush)
  {
    int fd = ::open(path, O_RDWR);
    void* m = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    t = now();
    std::memcpy(m, pin, n);
    std::printf("{\"what\": \"memcpy_1thread_pinned_to_file\", \"gbps\": %.2f}\n", n / (now() - t) / 1e9);
    munmap(m, n);
    close(fd);
  }
  unlink(path);
  cudaFreeHost(pin);
  cudaFree(dsrc);
  return 0;
}
