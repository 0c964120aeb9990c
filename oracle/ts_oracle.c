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
