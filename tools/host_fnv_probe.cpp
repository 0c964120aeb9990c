// Host FNV-1a-64 throughput on this box: how many GB/s can the host workers
// take off the GPU's FNV kernels? Scalar chains interleaved 1/4/8 per thread
// (the engine's fnv_lockstep uses 4) and SIMD lanes of independent objects
// (AVX2: 4 x 64-bit lanes per ymm, AVX-512: 8 per zmm; h*P = (h << 40) + h*0x1b3
// with 32x32->64 multiplies, no 64-bit vector multiply needed), all checked
// against the scalar reference chain.
//   g++ -O3 -pthread tools/host_fnv_probe.cpp -o tools/host_fnv_probe && tools/host_fnv_probe
#include <immintrin.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static constexpr uint64_t kSeed = 14695981039346656037ull, kP = 1099511628211ull;

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static uint64_t fnv1(const uint8_t* p, size_t n, uint64_t h = kSeed) {
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * kP;
  return h;
}

template <int K>
static void fnv_k(const uint8_t* const* p, size_t n, uint64_t* out) {
  uint64_t h[K];
  for (int k = 0; k < K; ++k) h[k] = kSeed;
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < K; ++k) h[k] = (h[k] ^ p[k][i]) * kP;
  for (int k = 0; k < K; ++k) out[k] = h[k];
}

__attribute__((target("avx2"))) static inline __m256i mulp256(__m256i h) {
  const __m256i q = _mm256_set1_epi64x(0x1b3);
  const __m256i lo = _mm256_mul_epu32(h, q);                         // (h & 0xffffffff) * q
  const __m256i hi = _mm256_mul_epu32(_mm256_srli_epi64(h, 32), q);  // (h >> 32) * q
  return _mm256_add_epi64(_mm256_add_epi64(lo, _mm256_slli_epi64(hi, 32)), _mm256_slli_epi64(h, 40));
}
__attribute__((target("avx512f"))) static inline __m512i mulp512(__m512i h) {
  const __m512i q = _mm512_set1_epi64(0x1b3);
  const __m512i lo = _mm512_mul_epu32(h, q);
  const __m512i hi = _mm512_mul_epu32(_mm512_srli_epi64(h, 32), q);
  return _mm512_add_epi64(_mm512_add_epi64(lo, _mm512_slli_epi64(hi, 32)), _mm512_slli_epi64(h, 40));
}

// 8 streams, 2 ymm accumulators of 4 lanes: per 8 input bytes of every
// stream, one 64-bit load per stream, then 8 byte steps.
__attribute__((target("avx2"))) static void fnv_avx2_8(const uint8_t* const* p, size_t n, uint64_t* out) {
  __m256i h0 = _mm256_set1_epi64x(static_cast<long long>(kSeed)), h1 = h0;
  const __m256i m8 = _mm256_set1_epi64x(0xff);
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w[8];
    for (int k = 0; k < 8; ++k) std::memcpy(&w[k], p[k] + i, 8);
    __m256i a = _mm256_setr_epi64x(w[0], w[1], w[2], w[3]);
    __m256i b = _mm256_setr_epi64x(w[4], w[5], w[6], w[7]);
    for (int j = 0; j < 8; ++j) {
      h0 = mulp256(_mm256_xor_si256(h0, _mm256_and_si256(a, m8)));
      h1 = mulp256(_mm256_xor_si256(h1, _mm256_and_si256(b, m8)));
      a = _mm256_srli_epi64(a, 8);
      b = _mm256_srli_epi64(b, 8);
    }
  }
  alignas(32) uint64_t r[8];
  _mm256_store_si256(reinterpret_cast<__m256i*>(r), h0);
  _mm256_store_si256(reinterpret_cast<__m256i*>(r + 4), h1);
  for (int k = 0; k < 8; ++k) out[k] = fnv1(p[k] + i, n - i, r[k]);
}

// 16 streams, 2 zmm accumulators of 8 lanes.
__attribute__((target("avx512f"))) static void fnv_avx512_16(const uint8_t* const* p, size_t n, uint64_t* out) {
  __m512i h0 = _mm512_set1_epi64(static_cast<long long>(kSeed)), h1 = h0;
  const __m512i m8 = _mm512_set1_epi64(0xff);
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w[16];
    for (int k = 0; k < 16; ++k) std::memcpy(&w[k], p[k] + i, 8);
    __m512i a = _mm512_loadu_si512(w), b = _mm512_loadu_si512(w + 8);
    for (int j = 0; j < 8; ++j) {
      h0 = mulp512(_mm512_xor_si512(h0, _mm512_and_si512(a, m8)));
      h1 = mulp512(_mm512_xor_si512(h1, _mm512_and_si512(b, m8)));
      a = _mm512_srli_epi64(a, 8);
      b = _mm512_srli_epi64(b, 8);
    }
  }
  alignas(64) uint64_t r[16];
  _mm512_store_si512(r, h0);
  _mm512_store_si512(r + 8, h1);
  for (int k = 0; k < 16; ++k) out[k] = fnv1(p[k] + i, n - i, r[k]);
}

int main(int argc, char** argv) {
  const size_t per = (argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 64) << 20;  // MiB per stream
  const int streams = 256;
  std::vector<uint8_t> buf(per * 16 + 64);
  for (size_t i = 0; i < buf.size(); ++i) buf[i] = static_cast<uint8_t>((i * 2654435761u) >> 13);
  // 256 streams over a 16-stream-wide buffer (offsets differ: distinct data)
  std::vector<const uint8_t*> ps(streams);
  for (int s = 0; s < streams; ++s) ps[s] = buf.data() + (s % 16) * per + (s / 16) % 64;
  const size_t n = per - 64;
  std::vector<uint64_t> ref(streams);
  for (int s = 0; s < 16; ++s) ref[s] = fnv1(ps[s], n);
  const bool has_avx2 = __builtin_cpu_supports("avx2"), has_avx512 = __builtin_cpu_supports("avx512f");
  struct variant {
    const char* name;
    int width;
    void (*fn)(const uint8_t* const*, size_t, uint64_t*);
    bool ok;
  } vs[] = {{"scalar1", 1, fnv_k<1>, true},          {"scalar4", 4, fnv_k<4>, true},
            {"scalar8", 8, fnv_k<8>, true},          {"avx2_8", 8, fnv_avx2_8, has_avx2},
            {"avx512_16", 16, fnv_avx512_16, has_avx512}};
  for (const auto& v : vs) {
    if (!v.ok) {
      std::printf("{\"variant\": \"%s\", \"supported\": false}\n", v.name);
      continue;
    }
    uint64_t out[16];
    v.fn(ps.data(), n, out);
    bool exact = true;
    for (int k = 0; k < v.width; ++k) exact &= out[k] == ref[k];
    for (int threads : {1, 16}) {
      const int groups = streams / v.width / (threads == 1 ? 16 : 1);
      std::vector<std::thread> th;
      const double t0 = now();
      for (int t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
          uint64_t o[16];
          for (int g = t; g < groups; g += threads) v.fn(ps.data() + g * v.width, n, o);
        });
      for (auto& x : th) x.join();
      const double dt = now() - t0;
      std::printf("{\"variant\": \"%s\", \"threads\": %d, \"exact\": %s, \"gbps\": %.2f}\n", v.name, threads,
                  exact ? "true" : "false", static_cast<double>(groups) * v.width * n / dt / 1e9);
      std::fflush(stdout);
    }
  }
  return 0;
}
