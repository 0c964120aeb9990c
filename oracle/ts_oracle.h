/* CPU restatement of the reference's byte/integer arithmetic on the snapshot path.
 * TEST INFRASTRUCTURE ONLY (checker + cpu_baseline "port"); never linked by the
 * product. Parity pinned against oracle/_ref (the compiled reference) and the
 * golden trees under tests/golden/. */
#ifndef TS_ORACLE_H
#define TS_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#define TSO_FNV_SEED 14695981039346656037ull

/* common.hpp:44-51 */
uint64_t tso_fnv1a64(const uint8_t* data, size_t n, uint64_t state);
/* pattern.hpp:57-69 */
void tso_fill_pattern(uint8_t* out, size_t n, uint64_t seed, uint64_t space, uint64_t iteration,
                      uint64_t offset);
/* pattern.hpp:72-81; returns index of first mismatch or -1 */
int64_t tso_match_pattern(const uint8_t* data, size_t n, uint64_t seed, uint64_t space,
                          uint64_t iteration, uint64_t offset);
/* pattern.hpp:26-33 */
uint64_t tso_mix64(uint64_t x);

/* provider.cpp:37-72 for ONE file: raw sizes/ids in, offsets out (in the input order);
 * returns tensor_region_end. order_out receives the planned order (indices). */
uint64_t tso_plan_file(const uint64_t* ids, const uint64_t* sizes, size_t n, uint64_t alignment,
                       uint64_t* offsets_out, size_t* order_out);
/* Bulk checkers (threaded; same arithmetic as above): FNV-1a of each object's
 * pattern bytes, and FNV-1a of each [ptrs[i], ptrs[i] + lens[i]) range. */
void tso_fnv_pattern_many(size_t n, const uint64_t* seed, const uint64_t* space, const uint64_t* iter,
                          const uint64_t* offset, const uint64_t* size, int threads, uint64_t* out);
void tso_fnv_ranges_many(size_t n, const uint8_t* const* ptrs, const uint64_t* lens, int threads, uint64_t* out);
#endif
