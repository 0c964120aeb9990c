// Layout planner, checkpoint file format and manifest.
//
// Byte contract (reference paths relative to /root/reference/proj):
//   plan_layout / plan_hash        provider.cpp:17-72
//   file = 4096-B header ("TSCKPT01", u32 1, u64 plan hash) | fixed region |
//          append region | u64 n | n x 41-B entries | u64 fnv(table) | u64 len
//                                  format.hpp:19-29, format.cpp:66-199
//   MANIFEST.tlv                   format.cpp:292-405
#pragma once

#include <atomic>
#include <functional>
#include <string>
#include <vector>

#include "core.hpp"

namespace tsb {

constexpr uint64_t header_reserved = 4096;  // provider.hpp:22
constexpr size_t entry_wire = 41;           // format.cpp:76

struct fixed_assignment {
  uint64_t object_id, file_offset, length;
};
struct file_plan {
  uint32_t file_id = 0;
  uint64_t tensor_region_end = header_reserved;
  std::vector<fixed_assignment> fixed;  // plan order (size desc, id asc)
};
struct layout_plan {
  uint64_t alignment = 4096;
  std::vector<file_plan> files;  // ascending file id
  uint64_t hash = 0;
  const file_plan& file(uint32_t fid) const;
};

// O(n log n) planner: objects grouped per file with one sort, no per-object scans
// (the reference's raw_chunk_source ctor is O(n^2), provider.cpp:78-85).
layout_plan plan_layout(const ts_object_desc* objs, size_t n, uint64_t alignment);
uint64_t compute_plan_hash(const layout_plan& p);

struct footer_entry {
  uint64_t object_id = 0;
  uint8_t kind = 0;
  uint64_t file_offset = 0, length = 0, object_offset_base = 0, checksum = 0;
};

std::vector<uint8_t> footer_blob(const std::vector<footer_entry>& entries);
void validate_entries(const std::vector<footer_entry>& entries, uint64_t tensor_region_end);

// Positional writer: header + ftruncate at open, concurrent pwrite at disjoint
// offsets, footer at finalize (format.cpp:125-199).
class file_writer {
 public:
  // `recycled`: a file of a retired checkpoint to take over (rename) instead of
  // creating a fresh one: its page-cache pages are reused, every byte the
  // checkpoint needs is rewritten (header, whole fixed region incl. zero gaps,
  // appends, footer; the old tail is truncated away).
  // `on_open(fd)` runs right after open, before the header is written or the
  // file is truncated; it returns true when the file's existing pages in
  // [0, tensor_region_end) must be kept (a page-locked registration of them is
  // in use, filereg.hpp): the file is then only re-sized, never emptied first.
  file_writer(const std::string& path, uint64_t tensor_region_end, uint64_t plan_hash,
              bool overwrite, bool io, const std::string& recycled = "",
              const std::function<bool(int)>& on_open = {});
  ~file_writer();
  void write_at(uint64_t off, const void* p, size_t n);
  // Fixed-region writes through a shared mapping of [0, tensor_region_end):
  // a page-cache file accepts one writer at a time through write(2) (the inode
  // lock), but page faults and copies into a shared mapping proceed in
  // parallel, so many flush threads can fill one file concurrently.
  void map_fixed_region();
  bool mapped() const { return map_ != nullptr; }
  // Kernel-bypass fixed-region writes (the reference's flush path with the
  // page cache taken out): a second descriptor opened O_DIRECT;
  // write_fixed sends the 4 KiB-aligned body of a write through it straight
  // from the pinned staging window (DMA from the pool, no page-cache copy)
  // and only the ragged head/tail through pwrite(2). Returns false (positional
  // buffered writes stay) where the filesystem refuses O_DIRECT (tmpfs).
  bool open_direct();
  bool direct() const { return dfd_ >= 0; }
  // O_DIRECT bodies go through this thread's io_uring (flush_mmap = 3): each
  // window body as a batch of 4 MiB writes in flight together.
  void use_uring(bool on) { uring_ = on; }
  uint64_t direct_bytes() const { return direct_bytes_.load(); }
  // Pre-faults [off, off+n) of the mapping (MADV_POPULATE_WRITE): page
  // allocation for the file overlaps the device-side capture and D2H.
  void populate(uint64_t off, uint64_t n);
  void write_fixed(uint64_t off, const void* p, size_t n);
  void finalize_at(uint64_t off, const std::vector<footer_entry>& entries);
  // Drops the fixed-region mapping (page-table teardown of a multi-GB mapping
  // is not free: done after the file is reported persisted).
  void release_mapping();
  const std::string& path() const { return path_; }
  int fd() const { return fd_; }

 private:
  std::string path_;
  int fd_ = -1;
  int dfd_ = -1;
  bool uring_ = false;
  std::atomic<uint64_t> direct_bytes_{0};  // (flush threads of one file write concurrently)
  uint64_t tre_;
  bool io_;
  bool reused_ = false;
  uint8_t* map_ = nullptr;
};

// Retires a checkpoint (MANIFEST.tlv removed first, so it is no longer
// restorable) and moves its rank files into `spare_dir` for reuse by later
// checkpoints (see file_writer's `recycled`). Checkpoint rotation without
// freeing and re-faulting the page cache.
void retire_checkpoint(const std::string& dir, const std::string& spare_dir);

// Spare files of one name ("rank_0000_file_1.bin") may exist in up to
// kMaxSpares copies (suffixes .1, .2, ...): retire adds one (the oldest surplus
// is overwritten), an issue takes one, provisioning creates them ahead of time.
constexpr int kMaxSpares = 4;
std::string spare_take(const std::string& spare_dir, const std::string& name);  // "" if none
std::string spare_put_name(const std::string& spare_dir, const std::string& name);

struct file_header {
  uint32_t version;
  uint64_t plan_hash;
};
file_header read_header(const std::string& path);
std::vector<footer_entry> read_footer(const std::string& path, uint64_t* file_size = nullptr);

// Reads `n` bytes at `off` (pread loop); throws io / incomplete_file.
void pread_all(int fd, void* p, size_t n, uint64_t off, const std::string& path);

// ---------------------------------------------------------------------------
// Manifest (format.hpp:118-153).

struct manifest_file {
  uint32_t file_id = 0;
  std::string path;
  std::vector<uint64_t> object_ids;
};
struct manifest_object {
  uint64_t object_id = 0;
  uint8_t kind = 0, tier = 0, precision = 0;
  uint32_t file_id = 0;
};
struct manifest_rank {
  int rank_id = 0, tp_idx = 0, pp_idx = 0, dp_idx = 0;
  std::vector<manifest_file> files;
  std::vector<manifest_object> objects;
};
struct manifest {
  uint64_t checkpoint_id = 0, iteration = 0;
  int tp = 1, pp = 1, dp = 1;
  bool zero1 = false;
  uint64_t seed = 0, n_params = 0;
  int layers = 1;
  uint64_t metadata_bytes = 0;
  bool complete = false;
  std::vector<manifest_rank> ranks;
};

value rank_to_value(const manifest_rank& r);
manifest_rank rank_from_value(const value& v);
value manifest_to_value(const manifest& m);
manifest manifest_from_value(const value& v);
void write_manifest(const std::string& path, const manifest& m);
manifest read_manifest(const std::string& path);  // requires complete=1 (format.cpp:424-426)

std::string rank_dir_name(int rank_id);

}  // namespace tsb
