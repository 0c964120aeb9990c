// Probe: device-to-device cudaMemcpyAsync — copy engine or SMs, and at what rate?
// Measures (1) D2D rate alone, (2) D2D concurrent with D2H windows, and
// (3) the slowdown a D2D stream inflicts on an SM-saturating compute kernel,
// compared with an SM copy kernel moving the same bytes. JSON lines.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/ce_probe.cu -o tools/ce_probe
#include <cuda_runtime.h>

#include <cstdio>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) std::printf("{\"error\": \"%s\", \"at\": \"%s\"}\n", cudaGetErrorString(e_), #x); \
  } while (0)

__global__ void burn(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0001f;
  for (int i = 0; i < iters; ++i) a = fmaf(a, b, 1e-7f);
  if (a == 12345.f) out[blockIdx.x] = a;
}

__global__ void smcopy(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) d[i] = s[i];
}

static float ms_between(cudaEvent_t a, cudaEvent_t b) {
  float m = 0;
  cudaEventElapsedTime(&m, a, b);
  return m;
}

int main() {
  cudaSetDevice(0);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t G = 1ull << 30, N = 16;
  char *src, *dst;
  CK(cudaMalloc(&src, N * G));
  CK(cudaMalloc(&dst, N * G));
  void* pin;
  CK(cudaHostAlloc(&pin, 4 * G, cudaHostAllocDefault));
  float* fo;
  CK(cudaMalloc(&fo, 4096 * 4));
  cudaStream_t s1, s2, s3;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking);
  cudaEvent_t a, b, c, d, e, f;
  for (cudaEvent_t* x : {&a, &b, &c, &d, &e, &f}) cudaEventCreate(x);
  CK(cudaMemset(src, 1, N * G));
  cudaDeviceSynchronize();

  // (1) D2D alone, 1 GiB copies
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, s1);
    for (size_t i = 0; i < N; ++i) CK(cudaMemcpyAsync(dst + i * G, src + i * G, G, cudaMemcpyDeviceToDevice, s1));
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
  }
  std::printf("{\"what\": \"d2d_alone\", \"gbps_rw\": %.1f}\n", 2.0 * N * G / (ms_between(a, b) / 1e3) / 1e9);
  // SM copy alone
  cudaEventRecord(a, s1);
  smcopy<<<sms * 2, 512, 0, s1>>>((const uint4*)src, (uint4*)dst, N * G / 16);
  cudaEventRecord(b, s1);
  cudaEventSynchronize(b);
  std::printf("{\"what\": \"smcopy_alone\", \"gbps_rw\": %.1f}\n", 2.0 * N * G / (ms_between(a, b) / 1e3) / 1e9);

  // (2) D2D with concurrent D2H (64 MiB windows, 4 GiB)
  cudaEventRecord(a, s1);
  cudaEventRecord(c, s2);
  for (size_t i = 0; i < N; ++i) CK(cudaMemcpyAsync(dst + i * G, src + i * G, G, cudaMemcpyDeviceToDevice, s1));
  for (size_t o = 0; o < 4 * G; o += 64 << 20)
    CK(cudaMemcpyAsync((char*)pin + o, src + o, 64 << 20, cudaMemcpyDeviceToHost, s2));
  cudaEventRecord(b, s1);
  cudaEventRecord(d, s2);
  cudaDeviceSynchronize();
  std::printf("{\"what\": \"d2d_with_d2h\", \"d2d_gbps_rw\": %.1f, \"d2h_gbps\": %.1f}\n",
              2.0 * N * G / (ms_between(a, b) / 1e3) / 1e9, 4.0 * G / (ms_between(c, d) / 1e3) / 1e9);

  // (3) interference with an SM-saturating kernel (4 CTAs/SM, ~0.2 s)
  const int iters = 12000000;
  auto burn_ms = [&](int variant) {
    cudaDeviceSynchronize();
    cudaEventRecord(e, s3);
    burn<<<sms * 8, 256, 0, s3>>>(fo, iters);
    cudaEventRecord(f, s3);
    if (variant == 1)
      for (size_t i = 0; i < N; ++i) cudaMemcpyAsync(dst + i * G, src + i * G, G, cudaMemcpyDeviceToDevice, s1);
    if (variant == 2) smcopy<<<sms * 2, 512, 0, s1>>>((const uint4*)src, (uint4*)dst, N * G / 16);
    cudaDeviceSynchronize();
    return ms_between(e, f);
  };
  burn_ms(0);
  const float base = burn_ms(0), with_ce = burn_ms(1), with_sm = burn_ms(2);
  std::printf("{\"what\": \"interference\", \"burn_ms\": %.2f, \"burn_with_d2d_ms\": %.2f, \"burn_with_smcopy_ms\": %.2f}\n",
              base, with_ce, with_sm);
  // priority variant: smcopy on a high-priority stream
  int lo, hi;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t sh;
  cudaStreamCreateWithPriority(&sh, cudaStreamNonBlocking, hi);
  cudaDeviceSynchronize();
  cudaEventRecord(e, s3);
  burn<<<sms * 8, 256, 0, s3>>>(fo, iters);
  cudaEventRecord(f, s3);
  cudaEventRecord(a, sh);
  smcopy<<<sms * 2, 512, 0, sh>>>((const uint4*)src, (uint4*)dst, N * G / 16);
  cudaEventRecord(b, sh);
  cudaDeviceSynchronize();
  std::printf("{\"what\": \"interference_hiprio_smcopy\", \"burn_ms\": %.2f, \"smcopy_ms\": %.2f}\n", ms_between(e, f),
              ms_between(a, b));
  cudaDeviceSynchronize();
  cudaEventRecord(e, s3);
  burn<<<sms * 8, 256, 0, s3>>>(fo, iters);
  cudaEventRecord(f, s3);
  cudaEventRecord(a, s1);
  for (size_t i = 0; i < N; ++i) cudaMemcpyAsync(dst + i * G, src + i * G, G, cudaMemcpyDeviceToDevice, s1);
  cudaEventRecord(b, s1);
  cudaDeviceSynchronize();
  std::printf("{\"what\": \"interference_d2d_timing\", \"burn_ms\": %.2f, \"d2d_ms\": %.2f}\n", ms_between(e, f),
              ms_between(a, b));
  return 0;
}
