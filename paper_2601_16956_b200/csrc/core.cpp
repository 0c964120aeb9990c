// Host core: FNV chains, host pattern, TLV codec, metadata value.
#include "core.hpp"

#include <chrono>

namespace tsb {

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

void fnv1a64_x4(const uint8_t* const p[4], const size_t n[4], uint64_t h[4]) {
  uint64_t a = h[0], b = h[1], c = h[2], d = h[3];
  size_t m = std::min(std::min(n[0], n[1]), std::min(n[2], n[3]));
  const uint8_t *pa = p[0], *pb = p[1], *pc = p[2], *pd = p[3];
  for (size_t i = 0; i < m; ++i) {
    a = (a ^ pa[i]) * fnv_prime;
    b = (b ^ pb[i]) * fnv_prime;
    c = (c ^ pc[i]) * fnv_prime;
    d = (d ^ pd[i]) * fnv_prime;
  }
  h[0] = fnv1a64(pa + m, n[0] - m, a);
  h[1] = fnv1a64(pb + m, n[1] - m, b);
  h[2] = fnv1a64(pc + m, n[2] - m, c);
  h[3] = fnv1a64(pd + m, n[3] - m, d);
}

// pattern.hpp:57-69: byte p of a space = byte (p % 8) of pattern_word(base, p / 8).
void fill_pattern_host(uint8_t* out, size_t n, uint64_t seed, uint64_t space, uint64_t it,
                       uint64_t offset) {
  const uint64_t base = pattern_base(seed, space, it);
  uint64_t pos = offset;
  size_t i = 0;
  while (i < n && (pos & 7)) {
    out[i++] = static_cast<uint8_t>(pattern_word(base, pos / 8) >> (8 * (pos & 7)));
    ++pos;
  }
  for (; i + 8 <= n; i += 8, pos += 8) {
    const uint64_t w = pattern_word(base, pos / 8);
    std::memcpy(out + i, &w, 8);  // little-endian host (x86-64)
  }
  for (; i < n; ++i, ++pos)
    out[i] = static_cast<uint8_t>(pattern_word(base, pos / 8) >> (8 * (pos & 7)));
}

// ---------------------------------------------------------------------------
// TLV. Tags and layout: tlv.hpp:16-22; strict decoder: tlv.cpp:104-151.

bool is_valid_utf8(const char* s, size_t n) {
  size_t i = 0;
  while (i < n) {
    const auto c = static_cast<uint8_t>(s[i]);
    size_t len;
    if (c < 0x80) len = 1;
    else if ((c >> 5) == 0x6) len = 2;
    else if ((c >> 4) == 0xe) len = 3;
    else if ((c >> 3) == 0x1e) len = 4;
    else return false;
    if (i + len > n) return false;
    for (size_t k = 1; k < len; ++k)
      if ((static_cast<uint8_t>(s[i + k]) >> 6) != 0x2) return false;
    i += len;
  }
  return true;
}

size_t encoded_size(const value& v) {
  switch (v.type()) {
    case 0: return 1;
    case 1:
    case 2: return 9;
    case 3: return 9 + std::get<std::string>(v.v).size();
    case 4: return 9 + std::get<vbytes>(v.v).size();
    case 5: {
      size_t s = 9;
      for (const auto& x : std::get<vlist>(v.v)) s += encoded_size(x);
      return s;
    }
    default: {
      size_t s = 9;
      for (const auto& [k, x] : std::get<vmap>(v.v)) s += 9 + k.size() + encoded_size(x);
      return s;
    }
  }
}

namespace {
void put_tag_len(uint8_t* out, size_t* pos, uint8_t tag, uint64_t len) {
  out[(*pos)++] = tag;
  put_u64(out + *pos, len);
  *pos += 8;
}
void put_str(uint8_t* out, size_t* pos, const std::string& s, const std::string& path) {
  if (!is_valid_utf8(s.data(), s.size()))
    fail(TS_ERR_TLV, "tlv: non-utf8 string at " + (path.empty() ? std::string("$") : path));
  put_tag_len(out, pos, 3, s.size());
  std::memcpy(out + *pos, s.data(), s.size());
  *pos += s.size();
}
void encode_rec(const value& v, uint8_t* out, size_t* pos, std::string& path) {
  switch (v.type()) {
    case 0: out[(*pos)++] = 0; break;
    case 1: put_tag_len(out, pos, 1, static_cast<uint64_t>(std::get<int64_t>(v.v))); break;
    case 2: {
      uint64_t bits;
      const double d = std::get<double>(v.v);
      std::memcpy(&bits, &d, 8);
      put_tag_len(out, pos, 2, bits);
      break;
    }
    case 3: put_str(out, pos, std::get<std::string>(v.v), path); break;
    case 4: {
      const auto& b = std::get<vbytes>(v.v);
      put_tag_len(out, pos, 4, b.size());
      if (!b.empty()) std::memcpy(out + *pos, b.data(), b.size());
      *pos += b.size();
      break;
    }
    case 5: {
      const auto& l = std::get<vlist>(v.v);
      put_tag_len(out, pos, 5, l.size());
      const size_t mark = path.size();
      for (size_t i = 0; i < l.size(); ++i) {
        path += "[" + std::to_string(i) + "]";
        encode_rec(l[i], out, pos, path);
        path.resize(mark);
      }
      break;
    }
    default: {
      const auto& m = std::get<vmap>(v.v);
      put_tag_len(out, pos, 6, m.size());
      const size_t mark = path.size();
      for (const auto& [k, x] : m) {
        path += "." + k;
        put_str(out, pos, k, path);
        encode_rec(x, out, pos, path);
        path.resize(mark);
      }
    }
  }
}

struct reader {
  const uint8_t* p;
  size_t n, pos = 0;
  void need(size_t k) const {
    if (k > n - pos) fail(TS_ERR_TLV, "tlv: truncated input");
  }
  uint8_t u8() {
    need(1);
    return p[pos++];
  }
  uint64_t u64() {
    need(8);
    uint64_t v = get_u64(p + pos);
    pos += 8;
    return v;
  }
};

value decode_rec(reader& r, int depth) {
  if (depth > 256) fail(TS_ERR_TLV, "tlv: nesting too deep");
  switch (r.u8()) {
    case 0: return value();
    case 1: return value(static_cast<int64_t>(r.u64()));
    case 2: {
      uint64_t bits = r.u64();
      double d;
      std::memcpy(&d, &bits, 8);
      return value(d);
    }
    case 3: {
      const uint64_t k = r.u64();
      r.need(k);
      std::string s(reinterpret_cast<const char*>(r.p + r.pos), k);
      r.pos += k;
      if (!is_valid_utf8(s.data(), s.size())) fail(TS_ERR_TLV, "tlv: invalid utf8 string");
      return value(std::move(s));
    }
    case 4: {
      const uint64_t k = r.u64();
      r.need(k);
      vbytes b(r.p + r.pos, r.p + r.pos + k);
      r.pos += k;
      return value(std::move(b));
    }
    case 5: {
      const uint64_t k = r.u64();
      vlist l;
      l.reserve(std::min<uint64_t>(k, 4096));
      for (uint64_t i = 0; i < k; ++i) l.push_back(decode_rec(r, depth + 1));
      return value(std::move(l));
    }
    case 6: {
      const uint64_t k = r.u64();
      vmap m;
      for (uint64_t i = 0; i < k; ++i) {
        value key = decode_rec(r, depth + 1);
        if (key.type() != 3) fail(TS_ERR_TLV, "tlv: map key is not a string");
        value x = decode_rec(r, depth + 1);
        m.emplace(std::move(std::get<std::string>(key.v)), std::move(x));
      }
      return value(std::move(m));
    }
    default: fail(TS_ERR_TLV, "tlv: unknown tag");
  }
}
}  // namespace

void encode_into(const value& v, uint8_t* out, size_t* pos) {
  std::string path;
  encode_rec(v, out, pos, path);
}

std::vector<uint8_t> encode(const value& v) {
  std::vector<uint8_t> out(encoded_size(v));
  size_t pos = 0;
  encode_into(v, out.data(), &pos);
  return out;
}

value decode(const uint8_t* p, size_t n) {
  reader r{p, n};
  value v = decode_rec(r, 0);
  if (r.pos != n) fail(TS_ERR_TLV, "tlv: trailing bytes after value");
  return v;
}

// model.cpp:206-231: fixed fields plus a pattern blob of metadata_bytes - 256
// bytes (16 when smaller), pattern space (3 << 56 | rank_id << 16).
value make_metadata_value(int rank_id, int tp, int pp, int dp, uint64_t seed,
                          uint64_t metadata_bytes, uint64_t iteration) {
  vmap m;
  m.emplace("iteration", value(static_cast<int64_t>(iteration)));
  m.emplace("rank_id", value(static_cast<int64_t>(rank_id)));
  m.emplace("tp_idx", value(static_cast<int64_t>(tp)));
  m.emplace("pp_idx", value(static_cast<int64_t>(pp)));
  m.emplace("dp_idx", value(static_cast<int64_t>(dp)));
  m.emplace("rng_seed",
            value(static_cast<int64_t>(mix64(seed ^ iteration ^ static_cast<uint64_t>(rank_id)))));
  m.emplace("framework", value(std::string("tierstream")));
  const uint64_t filler = metadata_bytes > 256 ? metadata_bytes - 256 : 16;
  vbytes b(filler);
  fill_pattern_host(b.data(), b.size(), seed, pack_space(3, static_cast<uint64_t>(rank_id), 0),
                    iteration, 0);
  m.emplace("state_blob", value(std::move(b)));
  return value(std::move(m));
}

}  // namespace tsb
