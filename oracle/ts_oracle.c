/* CPU restatement of the reference's byte/integer arithmetic on the snapshot path.
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the checker. Each function cites the reference
 * file:line it restates (paths relative to /root/reference/proj). */
#include "ts_oracle.h"

#include <stdlib.h>

/* include/tierstream/common.hpp:44-51 — 64-bit FNV-1a, byte at a time. */
uint64_t tso_fnv1a64(const uint8_t* data, size_t n, uint64_t state) {
  const uint64_t prime = 1099511628211ull;
  for (size_t i = 0; i < n; ++i) {
    state ^= (uint64_t)data[i];
    state *= prime;
  }
  return state;
}

/* include/tierstream/pattern.hpp:26-33 */
uint64_t tso_mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

/* pattern.hpp:35-40 */
static uint64_t pattern_base(uint64_t seed, uint64_t space, uint64_t it) {
  uint64_t h = tso_mix64(seed + 0x9e3779b97f4a7c15ull);
  h = tso_mix64(h ^ space);
  h = tso_mix64(h ^ it);
  return h | 1;
}

/* pattern.hpp:42-51 */
static uint64_t pattern_word(uint64_t base, uint64_t block) {
  uint64_t x = base + block * 0x9e3779b97f4a7c15ull;
  x ^= x >> 32;
  x *= 0xd6e8feb86659fd93ull;
  x ^= x >> 32;
  x *= 0xd6e8feb86659fd93ull;
  x ^= x >> 32;
  return x;
}

/* pattern.hpp:57-69: byte p of the space is byte (p % 8) of pattern_word(base, p / 8). */
void tso_fill_pattern(uint8_t* out, size_t n, uint64_t seed, uint64_t space, uint64_t iteration,
                      uint64_t offset) {
  const uint64_t base = pattern_base(seed, space, iteration);
  uint64_t pos = offset;
  size_t i = 0;
  while (i < n) {
    const uint64_t w = pattern_word(base, pos / 8);
    for (unsigned b = (unsigned)(pos % 8); b < 8 && i < n; ++b, ++i, ++pos)
      out[i] = (uint8_t)((w >> (8 * b)) & 0xff);
  }
}

/* pattern.hpp:72-81 */
int64_t tso_match_pattern(const uint8_t* data, size_t n, uint64_t seed, uint64_t space,
                          uint64_t iteration, uint64_t offset) {
  const uint64_t base = pattern_base(seed, space, iteration);
  uint64_t pos = offset;
  for (size_t i = 0; i < n; ++i, ++pos) {
    const uint64_t w = pattern_word(base, pos / 8);
    if (data[i] != (uint8_t)((w >> (8 * (pos % 8))) & 0xff)) return (int64_t)i;
  }
  return -1;
}

/* src/provider.cpp:54-71 — raw objects of one file sorted by (size desc, id asc),
 * each placed at align_up(cursor, alignment) starting at the 4096-byte header. */
static const uint64_t* g_ids;
static const uint64_t* g_sizes;
static int cmp_plan(const void* a, const void* b) {
  size_t i = *(const size_t*)a, j = *(const size_t*)b;
  if (g_sizes[i] != g_sizes[j]) return g_sizes[i] > g_sizes[j] ? -1 : 1;
  if (g_ids[i] != g_ids[j]) return g_ids[i] < g_ids[j] ? -1 : 1;
  return 0;
}

uint64_t tso_plan_file(const uint64_t* ids, const uint64_t* sizes, size_t n, uint64_t alignment,
                       uint64_t* offsets_out, size_t* order_out) {
  for (size_t i = 0; i < n; ++i) order_out[i] = i;
  g_ids = ids;
  g_sizes = sizes;
  qsort(order_out, n, sizeof(size_t), cmp_plan);
  uint64_t cursor = 4096; /* header_reserved_bytes, provider.hpp:22 */
  for (size_t k = 0; k < n; ++k) {
    size_t i = order_out[k];
    if (alignment) cursor = (cursor + alignment - 1) / alignment * alignment; /* common.hpp:35-38 */
    offsets_out[i] = cursor;
    cursor += sizes[i];
  }
  return cursor;
}

/* ------------------------------------------------------------------------
 * Bulk checkers for full-size parity (tests/test_gpu_large.py): the same
 * FNV-1a (common.hpp:44-51) and pattern (pattern.hpp:57-69) as above, over many
 * objects on host threads. A thread advances four independent chains in
 * lock-step so one core runs ~4 multiply chains at once; nothing here changes
 * the byte order inside an object. */
#include <pthread.h>
#include <stdatomic.h>
#include <string.h>

#define TSO_BLK 16384

typedef struct {
  size_t n;
  /* pattern mode */
  const uint64_t *seed, *space, *iter, *offset;
  /* range mode */
  const uint8_t* const* ptrs;
  const uint64_t* lens;
  uint64_t* out;
  atomic_size_t next;
} tso_many_job;

/* Fills `out` with the pattern bytes [pos, pos + n) of `base`, a word at a time. */
static void fill_fast(uint8_t* out, size_t n, uint64_t base, uint64_t pos) {
  size_t i = 0;
  while (i < n && (pos & 7)) {
    out[i++] = (uint8_t)(pattern_word(base, pos / 8) >> (8 * (pos & 7)));
    ++pos;
  }
  for (; i + 8 <= n; i += 8, pos += 8) {
    const uint64_t w = pattern_word(base, pos / 8);
    memcpy(out + i, &w, 8);
  }
  for (; i < n; ++i, ++pos) out[i] = (uint8_t)(pattern_word(base, pos / 8) >> (8 * (pos & 7)));
}

static void* many_worker(void* arg) {
  tso_many_job* J = (tso_many_job*)arg;
  const uint64_t P = 1099511628211ull;
  uint8_t* buf = (uint8_t*)malloc(4 * TSO_BLK);
  size_t obj[4];
  uint64_t h[4], done[4], len[4], base[4];
  int act = 0;
  for (;;) {
    while (act < 4) { /* refill the lanes */
      const size_t k = atomic_fetch_add(&J->next, 1);
      if (k >= J->n) break;
      obj[act] = k;
      h[act] = TSO_FNV_SEED;
      done[act] = 0;
      len[act] = J->ptrs ? J->lens[k] : J->lens[k];
      base[act] = J->ptrs ? 0 : pattern_base(J->seed[k], J->space[k], J->iter[k]);
      ++act;
    }
    if (act == 0) break;
    const uint8_t* p[4];
    uint64_t m = TSO_BLK;
    for (int a = 0; a < act; ++a) {
      const uint64_t r = len[a] - done[a];
      if (r < m) m = r;
    }
    for (int a = 0; a < act; ++a) {
      if (J->ptrs) {
        p[a] = J->ptrs[obj[a]] + done[a];
      } else {
        fill_fast(buf + a * TSO_BLK, (size_t)m, base[a], J->offset[obj[a]] + done[a]);
        p[a] = buf + a * TSO_BLK;
      }
    }
    if (act == 4) {
      uint64_t a0 = h[0], a1 = h[1], a2 = h[2], a3 = h[3];
      for (uint64_t i = 0; i < m; ++i) {
        a0 = (a0 ^ p[0][i]) * P;
        a1 = (a1 ^ p[1][i]) * P;
        a2 = (a2 ^ p[2][i]) * P;
        a3 = (a3 ^ p[3][i]) * P;
      }
      h[0] = a0, h[1] = a1, h[2] = a2, h[3] = a3;
    } else {
      for (int a = 0; a < act; ++a) h[a] = tso_fnv1a64(p[a], (size_t)m, h[a]);
    }
    for (int a = 0; a < act;) {
      done[a] += m;
      if (done[a] == len[a]) { /* object finished: publish, compact the lanes */
        J->out[obj[a]] = h[a];
        --act;
        obj[a] = obj[act], h[a] = h[act], done[a] = done[act], len[a] = len[act], base[a] = base[act];
      } else {
        ++a;
      }
    }
  }
  free(buf);
  return NULL;
}

static void run_many(tso_many_job* J, int threads) {
  if (threads < 1) threads = 1;
  atomic_init(&J->next, 0);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, many_worker, J);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
}

void tso_fnv_pattern_many(size_t n, const uint64_t* seed, const uint64_t* space, const uint64_t* iter,
                          const uint64_t* offset, const uint64_t* size, int threads, uint64_t* out) {
  tso_many_job J;
  memset(&J, 0, sizeof J);
  J.n = n, J.seed = seed, J.space = space, J.iter = iter, J.offset = offset, J.lens = size, J.out = out;
  run_many(&J, threads);
}

void tso_fnv_ranges_many(size_t n, const uint8_t* const* ptrs, const uint64_t* lens, int threads, uint64_t* out) {
  tso_many_job J;
  memset(&J, 0, sizeof J);
  J.n = n, J.ptrs = ptrs, J.lens = lens, J.out = out;
  run_many(&J, threads);
}
