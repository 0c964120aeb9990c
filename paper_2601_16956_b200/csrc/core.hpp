// Host core of the B200 snapshot engine: errors, FNV-1a, little-endian packing,
// the synthetic pattern (host side, for metadata blobs) and the TLV value model.
//
// Byte-level contracts follow the reference (paths relative to
// /root/reference/proj): FNV-1a-64 common.hpp:44-51, LE packing common.hpp:54-72,
// pattern pattern.hpp:18-69, TLV tlv.hpp:16-22 / tlv.cpp:39-203.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "../../include/ts_b200.h"

namespace tsb {

// ---------------------------------------------------------------------------
// Errors: one exception type carrying the C-ABI status (reference kinds map 1:1).

class error : public std::runtime_error {
 public:
  error(ts_status s, const std::string& what, int64_t object_id = -1)
      : std::runtime_error(what), status(s), object_id(object_id) {}
  ts_status status;
  int64_t object_id;
};

[[noreturn]] inline void fail(ts_status s, const std::string& what, int64_t oid = -1) {
  throw error(s, what, oid);
}

// ---------------------------------------------------------------------------
// FNV-1a-64 (common.hpp:44-51).

constexpr uint64_t fnv_seed = 14695981039346656037ull;
constexpr uint64_t fnv_prime = 1099511628211ull;

inline uint64_t fnv1a64(const void* p, size_t n, uint64_t h = fnv_seed) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= fnv_prime;
  }
  return h;
}

// Four independent FNV chains advanced in lock-step: the serial multiply chain
// of one object is latency bound (~4 cycles/byte), so interleaving objects
// gives the core ILP. Each chain is exactly fnv1a64 of its own range.
void fnv1a64_x4(const uint8_t* const p[4], const size_t n[4], uint64_t h[4]);

inline uint64_t align_up(uint64_t v, uint64_t a) { return a == 0 ? v : (v + a - 1) / a * a; }

inline void put_u64(uint8_t* o, uint64_t v) {
  for (int i = 0; i < 8; ++i) o[i] = static_cast<uint8_t>(v >> (8 * i));
}
inline void put_u32(uint8_t* o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o[i] = static_cast<uint8_t>(v >> (8 * i));
}
inline uint64_t get_u64(const uint8_t* in) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(in[i]) << (8 * i);
  return v;
}
inline uint32_t get_u32(const uint8_t* in) {
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(in[i]) << (8 * i);
  return v;
}

// ---------------------------------------------------------------------------
// Synthetic pattern (pattern.hpp:26-69), host side. The device side lives in
// kernels.cu; both are the same integer functions.

inline uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}
inline uint64_t pattern_base(uint64_t seed, uint64_t space, uint64_t it) {
  uint64_t h = mix64(seed + 0x9e3779b97f4a7c15ull);
  h = mix64(h ^ space);
  h = mix64(h ^ it);
  return h | 1;
}
inline uint64_t pattern_word(uint64_t base, uint64_t block) {
  uint64_t x = base + block * 0x9e3779b97f4a7c15ull;
  x ^= x >> 32;
  x *= 0xd6e8feb86659fd93ull;
  x ^= x >> 32;
  x *= 0xd6e8feb86659fd93ull;
  x ^= x >> 32;
  return x;
}
void fill_pattern_host(uint8_t* out, size_t n, uint64_t seed, uint64_t space, uint64_t it,
                       uint64_t offset);

inline uint64_t pack_space(uint64_t role, uint64_t layer, uint64_t tp_idx) {
  return (role << 56) | (layer << 16) | tp_idx;  // model.cpp:17-19
}

// ---------------------------------------------------------------------------
// TLV value (tlv.hpp:24-66): null | int64 | f64 | utf8 | bytes | list | map.
// Maps keep keys sorted (std::map<std::string>) so encodings are canonical.

struct value;
using vlist = std::vector<value>;
using vmap = std::map<std::string, value>;
using vbytes = std::vector<uint8_t>;

struct value {
  std::variant<std::monostate, int64_t, double, std::string, vbytes, vlist, vmap> v;
  value() = default;
  template <class T>
  explicit value(T x) : v(std::move(x)) {}
  int type() const { return static_cast<int>(v.index()); }
};

bool is_valid_utf8(const char* s, size_t n);
size_t encoded_size(const value& v);
// Appends the canonical encoding of v to out (tlv.cpp:39-77).
void encode_into(const value& v, uint8_t* out, size_t* pos);
std::vector<uint8_t> encode(const value& v);
value decode(const uint8_t* p, size_t n);  // strict (tlv.cpp:104-151, 198-203)

value make_metadata_value(int rank_id, int tp, int pp, int dp, uint64_t seed,
                          uint64_t metadata_bytes, uint64_t iteration);

// Monotonic ns clock.
int64_t now_ns();

}  // namespace tsb

// The opaque C handle ts_value* is a reinterpret_cast of tsb::value* (never defined).
inline tsb::value* V(ts_value* h) { return reinterpret_cast<tsb::value*>(h); }
inline const tsb::value* V(const ts_value* h) { return reinterpret_cast<const tsb::value*>(h); }
inline ts_value* H(tsb::value* v) { return reinterpret_cast<ts_value*>(v); }
inline const ts_value* H(const tsb::value* v) { return reinterpret_cast<const ts_value*>(v); }
