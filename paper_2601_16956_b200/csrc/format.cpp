// Layout planner, file format and manifest (see format.hpp for the contract).
#include "format.hpp"
#include "uring.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/statvfs.h>
#include <sys/vfs.h>
#include <unistd.h>

#include <dirent.h>

#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <unordered_set>

namespace tsb {

const file_plan& layout_plan::file(uint32_t fid) const {
  for (const auto& f : files)
    if (f.file_id == fid) return f;
  fail(TS_ERR_GENERIC, "layout plan: unknown file id");
}

// provider.cpp:37-72. Files: every object's file id. Raw objects per file are
// placed largest-first (ties by id) at align_up(cursor) from 4096.
layout_plan plan_layout(const ts_object_desc* objs, size_t n, uint64_t alignment) {
  layout_plan p;
  p.alignment = alignment;
  std::unordered_set<uint64_t> seen;
  seen.reserve(n * 2);
  std::vector<uint32_t> fids;
  fids.reserve(n);
  std::vector<size_t> raw;
  raw.reserve(n);
  for (size_t i = 0; i < n; ++i) {
    if (!seen.insert(objs[i].object_id).second)
      fail(TS_ERR_GENERIC, "plan_layout: duplicate object id " + std::to_string(objs[i].object_id));
    fids.push_back(objs[i].file_id);
    if (objs[i].kind == TS_KIND_RAW) {
      if (objs[i].size_bytes == 0) fail(TS_ERR_GENERIC, "plan_layout: raw buffer without a known size");
      raw.push_back(i);
    }
  }
  std::sort(fids.begin(), fids.end());
  fids.erase(std::unique(fids.begin(), fids.end()), fids.end());
  p.files.resize(fids.size());
  for (size_t k = 0; k < fids.size(); ++k) p.files[k].file_id = fids[k];
  std::sort(raw.begin(), raw.end(), [&](size_t a, size_t b) {
    if (objs[a].file_id != objs[b].file_id) return objs[a].file_id < objs[b].file_id;
    if (objs[a].size_bytes != objs[b].size_bytes) return objs[a].size_bytes > objs[b].size_bytes;
    return objs[a].object_id < objs[b].object_id;
  });
  size_t k = 0;
  for (auto& f : p.files) {
    uint64_t cursor = header_reserved;
    while (k < raw.size() && objs[raw[k]].file_id == f.file_id) {
      cursor = align_up(cursor, alignment);
      f.fixed.push_back({objs[raw[k]].object_id, cursor, objs[raw[k]].size_bytes});
      cursor += objs[raw[k]].size_bytes;
      ++k;
    }
    f.tensor_region_end = cursor;
  }
  p.hash = compute_plan_hash(p);
  return p;
}

// provider.cpp:17-35: FNV-1a over LE u64s.
uint64_t compute_plan_hash(const layout_plan& p) {
  size_t words = 1;
  for (const auto& f : p.files) words += 2 + 3 * f.fixed.size();
  std::vector<uint8_t> buf(words * 8);
  size_t o = 0;
  auto push = [&](uint64_t v) {
    put_u64(buf.data() + o, v);
    o += 8;
  };
  push(p.alignment);
  for (const auto& f : p.files) {
    push(f.file_id);
    push(f.tensor_region_end);
    for (const auto& a : f.fixed) {
      push(a.object_id);
      push(a.file_offset);
      push(a.length);
    }
  }
  return fnv1a64(buf.data(), buf.size());
}

// format.cpp:176-199
std::vector<uint8_t> footer_blob(const std::vector<footer_entry>& entries) {
  const size_t table_len = 8 + entries.size() * entry_wire;
  std::vector<uint8_t> blob(table_len + 16);
  put_u64(blob.data(), entries.size());
  for (size_t i = 0; i < entries.size(); ++i) {
    uint8_t* o = blob.data() + 8 + i * entry_wire;
    const auto& e = entries[i];
    put_u64(o, e.object_id);
    o[8] = e.kind;
    put_u64(o + 9, e.file_offset);
    put_u64(o + 17, e.length);
    put_u64(o + 25, e.object_offset_base);
    put_u64(o + 33, e.checksum);
  }
  put_u64(blob.data() + table_len, fnv1a64(blob.data(), table_len));
  put_u64(blob.data() + table_len + 8, table_len + 8);
  return blob;
}

// format.cpp:95-121
void validate_entries(const std::vector<footer_entry>& entries, uint64_t tre) {
  std::vector<std::pair<uint64_t, uint64_t>> spans;
  spans.reserve(entries.size());
  for (const auto& e : entries) {
    const int64_t oid = static_cast<int64_t>(e.object_id);
    if (e.length == 0) fail(TS_ERR_INVALID_ENTRIES, "zero-length entry", oid);
    if (e.file_offset < header_reserved) fail(TS_ERR_INVALID_ENTRIES, "entry inside reserved header", oid);
    if (e.kind == 0 && e.file_offset + e.length > tre)
      fail(TS_ERR_INVALID_ENTRIES, "raw entry above the tensor region", oid);
    if (e.kind == 1 && e.file_offset < tre)
      fail(TS_ERR_INVALID_ENTRIES, "structured entry below the tensor region", oid);
    spans.emplace_back(e.file_offset, e.file_offset + e.length);
  }
  std::sort(spans.begin(), spans.end());
  for (size_t i = 1; i < spans.size(); ++i)
    if (spans[i].first < spans[i - 1].second)
      fail(TS_ERR_INVALID_ENTRIES, "overlapping footer entries");
}

namespace {
void pwrite_all(int fd, const uint8_t* p, size_t n, uint64_t off, const std::string& path) {
  size_t done = 0;
  while (done < n) {
    const ssize_t k = ::pwrite(fd, p + done, n - done, static_cast<off_t>(off + done));
    if (k < 0) {
      if (errno == EINTR) continue;
      fail(TS_ERR_IO, "write failed at " + path + ": " + std::strerror(errno));
    }
    done += static_cast<size_t>(k);
  }
}
}  // namespace

void pread_all(int fd, void* p, size_t n, uint64_t off, const std::string& path) {
  size_t done = 0;
  auto* b = static_cast<uint8_t*>(p);
  while (done < n) {
    const ssize_t k = ::pread(fd, b + done, n - done, static_cast<off_t>(off + done));
    if (k < 0) {
      if (errno == EINTR) continue;
      fail(TS_ERR_IO, "read failed at " + path + ": " + std::strerror(errno));
    }
    if (k == 0) fail(TS_ERR_INCOMPLETE_FILE, "unexpected end of file: " + path);
    done += static_cast<size_t>(k);
  }
}

// format.cpp:125-147: header block, pre-size to tensor_region_end.
file_writer::file_writer(const std::string& path, uint64_t tre, uint64_t plan_hash, bool overwrite,
                         bool io, const std::string& recycled, const std::function<bool(int)>& on_open)
    : path_(path), tre_(tre), io_(io) {
  if (!io_) return;
  if (!overwrite && ::access(path.c_str(), F_OK) == 0) fail(TS_ERR_IO, "file exists: " + path);
  if (!recycled.empty() && ::rename(recycled.c_str(), path.c_str()) == 0) {
    fd_ = ::open(path.c_str(), O_RDWR);
    reused_ = fd_ >= 0;
  }
  bool fresh = false;
  if (fd_ < 0) {
    fd_ = ::open(path.c_str(), O_RDWR | O_CREAT, 0644);
    fresh = true;
  }
  if (fd_ < 0) fail(TS_ERR_IO, "cannot create " + path + ": " + std::strerror(errno));
  const bool keep = on_open ? on_open(fd_) : false;
  // (O_TRUNC semantics for a new file, after on_open had its look at the inode)
  if (fresh && !keep && ::ftruncate(fd_, 0) != 0)
    fail(TS_ERR_IO, "cannot truncate " + path + ": " + std::strerror(errno));
  uint8_t header[header_reserved] = {};
  std::memcpy(header, "TSCKPT01", 8);
  put_u32(header + 8, 1);
  put_u64(header + 12, plan_hash);
  pwrite_all(fd_, header, sizeof header, 0, path_);
  if (::ftruncate(fd_, static_cast<off_t>(tre_)) != 0)
    fail(TS_ERR_IO, "cannot pre-size " + path + ": " + std::strerror(errno));
}

file_writer::~file_writer() {
  if (map_) ::munmap(map_, tre_);
  if (dfd_ >= 0) ::close(dfd_);
  if (fd_ >= 0) ::close(fd_);
}

bool file_writer::open_direct() {
  if (!io_ || dfd_ >= 0 || map_) return dfd_ >= 0;
  // tmpfs accepts O_DIRECT (Linux >= 6.6) but serves it from its page cache:
  // nothing to bypass, keep the buffered path (and honest direct_io_bytes)
  struct statfs fs;
  if (::fstatfs(fd_, &fs) == 0 && static_cast<unsigned long>(fs.f_type) == 0x01021994ul) return false;
  dfd_ = ::open(path_.c_str(), O_WRONLY | O_DIRECT);
  return dfd_ >= 0;
}

void file_writer::release_mapping() {
  if (map_) ::munmap(map_, tre_);
  map_ = nullptr;
}

void file_writer::map_fixed_region() {
  if (!io_ || map_ || tre_ <= header_reserved) return;
  // A fault on a full filesystem raises SIGBUS instead of returning ENOSPC:
  // only map when the space is there, else keep positional writes.
  struct statvfs vs;
  if (::fstatvfs(fd_, &vs) != 0 || static_cast<uint64_t>(vs.f_bavail) * vs.f_frsize < tre_ + (64ull << 20)) return;
  // (a recycled file's pages exist: its faults only map them)
  void* m = ::mmap(nullptr, tre_, PROT_READ | PROT_WRITE, MAP_SHARED, fd_, 0);
  if (m == MAP_FAILED) return;  // fall back to positional writes
  map_ = static_cast<uint8_t*>(m);
}

#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
void file_writer::populate(uint64_t off, uint64_t n) {
  if (!map_ || off >= tre_) return;
  n = std::min<uint64_t>(n, tre_ - off);
  const uint64_t a = off & ~4095ull;
  ::madvise(map_ + a, n + (off - a), MADV_POPULATE_WRITE);  // best effort
}

void file_writer::write_fixed(uint64_t off, const void* p, size_t n) {
  if (!io_ || n == 0) return;
  if (off < header_reserved || off + n > tre_) fail(TS_ERR_IO, "fixed write outside the tensor region");
  if (map_) {
    // Reserve the range before touching the mapping: a write fault on a full
    // filesystem is a SIGBUS, a failed fallocate is an error we can report
    // (the positional write below then returns ENOSPC as a format error, the
    // reference's pwrite behaviour). Filesystems without fallocate keep the
    // free-space check made at map time.
    if (::fallocate(fd_, 0, static_cast<off_t>(off), static_cast<off_t>(n)) == 0 || errno == EOPNOTSUPP ||
        errno == ENOSYS) {
      std::memcpy(map_ + off, p, n);
      return;
    }
  }
  const auto* b = static_cast<const uint8_t*>(p);
  constexpr uint64_t blk = 4096;
  // O_DIRECT needs file offset, length and buffer aligned: only when the
  // buffer and the file offset share their offset within a block
  if (dfd_ >= 0 && ((reinterpret_cast<uintptr_t>(b) - off) & (blk - 1)) == 0) {
    const uint64_t a = (off + blk - 1) & ~(blk - 1), e = (off + n) & ~(blk - 1);
    if (e > a) {
      if (a > off) pwrite_all(fd_, b, a - off, off, path_);
      const int64_t k = uring_ ? uring_pwrite(dfd_, b + (a - off), e - a, a, 4ull << 20)
                               : static_cast<int64_t>(::pwrite(dfd_, b + (a - off), e - a, static_cast<off_t>(a)));
      if (k == static_cast<int64_t>(e - a)) {
        direct_bytes_ += e - a;
        if (off + n > e) pwrite_all(fd_, b + (e - off), off + n - e, e, path_);
        return;
      }
      // short or refused direct write: finish the whole range buffered
      // (the bytes are all in the window; rewriting them is idempotent)
    }
  }
  pwrite_all(fd_, b, n, off, path_);
}

void file_writer::write_at(uint64_t off, const void* p, size_t n) {
  if (!io_ || n == 0) return;
  pwrite_all(fd_, static_cast<const uint8_t*>(p), n, off, path_);
}

void file_writer::finalize_at(uint64_t off, const std::vector<footer_entry>& entries) {
  validate_entries(entries, tre_);
  if (!io_) return;
  const auto blob = footer_blob(entries);
  pwrite_all(fd_, blob.data(), blob.size(), off, path_);
}

namespace {
struct fd_guard {
  int fd;
  ~fd_guard() {
    if (fd >= 0) ::close(fd);
  }
};
int open_ro(const std::string& path) {
  int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0)
    fail(errno == ENOENT ? TS_ERR_MISSING_FILE : TS_ERR_IO,
         "cannot open " + path + ": " + std::strerror(errno));
  return fd;
}
uint64_t fd_size(int fd) {
  struct stat st;
  if (::fstat(fd, &st) != 0) return 0;
  return static_cast<uint64_t>(st.st_size);
}
}  // namespace

// format.cpp:201-216
file_header read_header(const std::string& path) {
  fd_guard g{open_ro(path)};
  if (fd_size(g.fd) < header_reserved)
    fail(TS_ERR_INCOMPLETE_FILE, "file shorter than the reserved header: " + path);
  uint8_t h[20];
  pread_all(g.fd, h, 20, 0, path);
  if (std::memcmp(h, "TSCKPT01", 8) != 0) fail(TS_ERR_INCOMPLETE_FILE, "bad magic: " + path);
  file_header fh{get_u32(h + 8), get_u64(h + 12)};
  if (fh.version != 1) fail(TS_ERR_INCOMPLETE_FILE, "unsupported format version in " + path);
  return fh;
}

// format.cpp:218-245
std::vector<footer_entry> read_footer(const std::string& path, uint64_t* file_size) {
  read_header(path);
  fd_guard g{open_ro(path)};
  const uint64_t size = fd_size(g.fd);
  if (file_size) *file_size = size;
  if (size < header_reserved + 16) fail(TS_ERR_INCOMPLETE_FILE, "no room for a footer: " + path);
  uint8_t t[8];
  pread_all(g.fd, t, 8, size - 8, path);
  const uint64_t blob_len = get_u64(t);
  if (blob_len < 16 || blob_len + 8 > size)
    fail(TS_ERR_INCOMPLETE_FILE, "implausible footer length, file incomplete: " + path);
  std::vector<uint8_t> blob(blob_len);
  pread_all(g.fd, blob.data(), blob_len, size - 8 - blob_len, path);
  const size_t table_len = blob_len - 8;
  if (get_u64(blob.data() + table_len) != fnv1a64(blob.data(), table_len))
    fail(TS_ERR_INCOMPLETE_FILE, "footer checksum mismatch, file incomplete: " + path);
  const uint64_t count = get_u64(blob.data());
  if (8 + count * entry_wire != table_len)
    fail(TS_ERR_CORRUPT_FOOTER, "footer entry count disagrees with table size: " + path);
  std::vector<footer_entry> out(count);
  for (uint64_t i = 0; i < count; ++i) {
    const uint8_t* e = blob.data() + 8 + i * entry_wire;
    out[i] = {get_u64(e), e[8], get_u64(e + 9), get_u64(e + 17), get_u64(e + 25), get_u64(e + 33)};
  }
  return out;
}

namespace {
std::string spare_name(const std::string& spare_dir, const std::string& name, int k) {
  return spare_dir + "/" + name + (k ? "." + std::to_string(k) : std::string());
}
}  // namespace

std::string spare_take(const std::string& spare_dir, const std::string& name) {
  for (int k = 0; k < kMaxSpares; ++k) {
    const std::string p = spare_name(spare_dir, name, k);
    if (::access(p.c_str(), F_OK) == 0) return p;
  }
  return {};
}

std::string spare_put_name(const std::string& spare_dir, const std::string& name) {
  for (int k = 0; k < kMaxSpares; ++k) {
    const std::string p = spare_name(spare_dir, name, k);
    if (::access(p.c_str(), F_OK) != 0) return p;
  }
  return spare_name(spare_dir, name, 0);  // full: replace the first
}

void retire_checkpoint(const std::string& dir, const std::string& spare_dir) {
  ::mkdir(spare_dir.c_str(), 0755);
  if (::unlink((dir + "/MANIFEST.tlv").c_str()) != 0 && errno != ENOENT)
    fail(TS_ERR_IO, "cannot retire " + dir + ": " + std::strerror(errno));
  DIR* d = ::opendir(dir.c_str());
  if (!d) fail(TS_ERR_MISSING_FILE, "cannot open " + dir);
  std::vector<std::string> ranks;
  while (dirent* e = ::readdir(d))
    if (std::strncmp(e->d_name, "rank_", 5) == 0) ranks.push_back(e->d_name);
  ::closedir(d);
  for (const auto& r : ranks) {
    const std::string rd = dir + "/" + r;
    DIR* rdh = ::opendir(rd.c_str());
    if (!rdh) continue;
    std::vector<std::string> files;
    while (dirent* e = ::readdir(rdh))
      if (std::strncmp(e->d_name, "file_", 5) == 0) files.push_back(e->d_name);
    ::closedir(rdh);
    for (const auto& f : files) {
      const std::string dst = spare_put_name(spare_dir, r + "_" + f);
      if (::rename((rd + "/" + f).c_str(), dst.c_str()) != 0)
        fail(TS_ERR_IO, "cannot recycle " + rd + "/" + f + ": " + std::strerror(errno));
    }
    ::rmdir(rd.c_str());
  }
  ::rmdir(dir.c_str());
}

// ---------------------------------------------------------------------------
// Manifest TLV (format.cpp:292-396)

std::string rank_dir_name(int rank_id) {
  char b[32];
  std::snprintf(b, sizeof b, "rank_%04d", rank_id);
  return b;
}

namespace {
value I(int64_t v) { return value(v); }
int64_t need_int(const vmap& m, const char* k) {
  auto it = m.find(k);
  if (it == m.end() || it->second.type() != TS_V_INT)
    fail(TS_ERR_BAD_MANIFEST, std::string("manifest missing field: ") + k);
  return std::get<int64_t>(it->second.v);
}
const value& need(const vmap& m, const char* k, int type) {
  auto it = m.find(k);
  if (it == m.end() || it->second.type() != type)
    fail(TS_ERR_BAD_MANIFEST, std::string("manifest missing field: ") + k);
  return it->second;
}
}  // namespace

value rank_to_value(const manifest_rank& r) {
  vmap rm;
  rm.emplace("rank_id", I(r.rank_id));
  rm.emplace("tp_idx", I(r.tp_idx));
  rm.emplace("pp_idx", I(r.pp_idx));
  rm.emplace("dp_idx", I(r.dp_idx));
  vlist files;
  for (const auto& f : r.files) {
    vmap fm;
    fm.emplace("file_id", I(f.file_id));
    fm.emplace("path", value(f.path));
    vlist oids;
    oids.reserve(f.object_ids.size());
    for (uint64_t o : f.object_ids) oids.push_back(I(static_cast<int64_t>(o)));
    fm.emplace("object_ids", value(std::move(oids)));
    files.push_back(value(std::move(fm)));
  }
  rm.emplace("files", value(std::move(files)));
  vlist objs;
  objs.reserve(r.objects.size());
  for (const auto& o : r.objects) {
    vmap om;
    om.emplace("object_id", I(static_cast<int64_t>(o.object_id)));
    om.emplace("kind", I(o.kind));
    om.emplace("tier", I(o.tier));
    om.emplace("precision", I(o.precision));
    om.emplace("file_id", I(o.file_id));
    objs.push_back(value(std::move(om)));
  }
  rm.emplace("objects", value(std::move(objs)));
  return value(std::move(rm));
}

manifest_rank rank_from_value(const value& v) {
  if (v.type() != TS_V_MAP) fail(TS_ERR_BAD_MANIFEST, "rank entry is not a map");
  const auto& rm = std::get<vmap>(v.v);
  manifest_rank r;
  r.rank_id = static_cast<int>(need_int(rm, "rank_id"));
  r.tp_idx = static_cast<int>(need_int(rm, "tp_idx"));
  r.pp_idx = static_cast<int>(need_int(rm, "pp_idx"));
  r.dp_idx = static_cast<int>(need_int(rm, "dp_idx"));
  for (const auto& fv : std::get<vlist>(need(rm, "files", TS_V_LIST).v)) {
    if (fv.type() != TS_V_MAP) fail(TS_ERR_BAD_MANIFEST, "file entry is not a map");
    const auto& fm = std::get<vmap>(fv.v);
    manifest_file f;
    f.file_id = static_cast<uint32_t>(need_int(fm, "file_id"));
    f.path = std::get<std::string>(need(fm, "path", TS_V_STRING).v);
    for (const auto& o : std::get<vlist>(need(fm, "object_ids", TS_V_LIST).v)) {
      if (o.type() != TS_V_INT) fail(TS_ERR_BAD_MANIFEST, "object id is not an int");
      f.object_ids.push_back(static_cast<uint64_t>(std::get<int64_t>(o.v)));
    }
    r.files.push_back(std::move(f));
  }
  for (const auto& ov : std::get<vlist>(need(rm, "objects", TS_V_LIST).v)) {
    if (ov.type() != TS_V_MAP) fail(TS_ERR_BAD_MANIFEST, "object entry is not a map");
    const auto& om = std::get<vmap>(ov.v);
    manifest_object o;
    o.object_id = static_cast<uint64_t>(need_int(om, "object_id"));
    o.kind = static_cast<uint8_t>(need_int(om, "kind"));
    o.tier = static_cast<uint8_t>(need_int(om, "tier"));
    o.precision = static_cast<uint8_t>(need_int(om, "precision"));
    o.file_id = static_cast<uint32_t>(need_int(om, "file_id"));
    r.objects.push_back(o);
  }
  return r;
}

value manifest_to_value(const manifest& m) {
  vmap v;
  v.emplace("checkpoint_id", I(static_cast<int64_t>(m.checkpoint_id)));
  v.emplace("iteration", I(static_cast<int64_t>(m.iteration)));
  v.emplace("tp", I(m.tp));
  v.emplace("pp", I(m.pp));
  v.emplace("dp", I(m.dp));
  v.emplace("zero1", I(m.zero1 ? 1 : 0));
  v.emplace("seed", I(static_cast<int64_t>(m.seed)));
  v.emplace("n_params", I(static_cast<int64_t>(m.n_params)));
  v.emplace("layers", I(m.layers));
  v.emplace("metadata_bytes", I(static_cast<int64_t>(m.metadata_bytes)));
  v.emplace("complete", I(m.complete ? 1 : 0));
  vlist ranks;
  for (const auto& r : m.ranks) ranks.push_back(rank_to_value(r));
  v.emplace("ranks", value(std::move(ranks)));
  return value(std::move(v));
}

manifest manifest_from_value(const value& v) {
  if (v.type() != TS_V_MAP) fail(TS_ERR_BAD_MANIFEST, "manifest is not a map");
  const auto& m = std::get<vmap>(v.v);
  manifest out;
  out.checkpoint_id = static_cast<uint64_t>(need_int(m, "checkpoint_id"));
  out.iteration = static_cast<uint64_t>(need_int(m, "iteration"));
  out.tp = static_cast<int>(need_int(m, "tp"));
  out.pp = static_cast<int>(need_int(m, "pp"));
  out.dp = static_cast<int>(need_int(m, "dp"));
  out.zero1 = need_int(m, "zero1") != 0;
  out.seed = static_cast<uint64_t>(need_int(m, "seed"));
  out.n_params = static_cast<uint64_t>(need_int(m, "n_params"));
  out.layers = static_cast<int>(need_int(m, "layers"));
  out.metadata_bytes = static_cast<uint64_t>(need_int(m, "metadata_bytes"));
  out.complete = need_int(m, "complete") != 0;
  auto it = m.find("ranks");
  if (it == m.end() || it->second.type() != TS_V_LIST) fail(TS_ERR_BAD_MANIFEST, "manifest missing ranks");
  for (const auto& rv : std::get<vlist>(it->second.v)) out.ranks.push_back(rank_from_value(rv));
  return out;
}

// format.cpp:398-405 (written to a temp name and renamed: same bytes, atomic commit)
void write_manifest(const std::string& path, const manifest& m) {
  const auto bytes = encode(manifest_to_value(m));
  const std::string tmp = path + ".tmp";
  int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) fail(TS_ERR_IO, "cannot write manifest: " + path);
  size_t done = 0;
  while (done < bytes.size()) {
    ssize_t k = ::write(fd, bytes.data() + done, bytes.size() - done);
    if (k < 0) {
      if (errno == EINTR) continue;
      ::close(fd);
      fail(TS_ERR_IO, "manifest write failed: " + path);
    }
    done += static_cast<size_t>(k);
  }
  ::close(fd);
  if (::rename(tmp.c_str(), path.c_str()) != 0) fail(TS_ERR_IO, "manifest rename failed: " + path);
}

// format.cpp:407-428
manifest read_manifest(const std::string& path) {
  int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) fail(TS_ERR_MISSING_FILE, "cannot open manifest: " + path);
  fd_guard g{fd};
  const uint64_t size = fd_size(fd);
  std::vector<uint8_t> bytes(size);
  if (size) pread_all(fd, bytes.data(), size, 0, path);
  value v;
  try {
    v = decode(bytes.data(), bytes.size());
  } catch (const error& e) {
    fail(TS_ERR_BAD_MANIFEST, std::string("manifest does not decode: ") + e.what());
  }
  manifest m = manifest_from_value(v);
  if (!m.complete) fail(TS_ERR_BAD_MANIFEST, "manifest not marked complete: " + path);
  return m;
}

}  // namespace tsb
