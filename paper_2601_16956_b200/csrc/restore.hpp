// Restore / verify (format.cpp:201-529) on the B200 path.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <unordered_map>
#include <vector>

#include "format.hpp"

namespace tsb {

struct restore_handle {
  struct file_info {
    uint32_t file_id = 0;
    std::string path;
    uint64_t size = 0, region_end = header_reserved;
    std::vector<footer_entry> entries;
  };
  struct rank_cache {
    bool loaded = false;
    std::vector<file_info> files;
    std::unordered_map<uint64_t, uint64_t> sizes;
    std::unordered_map<uint64_t, uint8_t> kinds;
    std::unordered_map<uint64_t, value> structured;
  };
  manifest m;
  std::string base;
  std::vector<rank_cache> ranks;
  // Files page-locked by this process (file_dma rotation) are read by the copy
  // engines straight from their page cache instead of pread into pinned memory.
  bool use_file_cache = true;
  // Reads from disk O_DIRECT into the pinned windows (page cache bypassed):
  // 1 always, 0 never, -1 (default) for files mostly not in the page cache.
  int direct_io = -1;

  explicit restore_handle(const std::string& manifest_path);
  ~restore_handle();
  restore_handle(const restore_handle&) = delete;
  restore_handle& operator=(const restore_handle&) = delete;
  void load_rank(int index);
  void restore_rank(int index, const ts_object_desc* dst, size_t n, int device, cudaStream_t st,
                    ts_restore_stats* stats);
};

// Frees the process-wide restore staging (pinned ring, per-device window ring,
// scratch); returns the bytes freed. Also done when the last handle closes.
uint64_t restore_release_staging();

void verify_checkpoint(const std::string& manifest_path, std::vector<std::pair<int, int64_t>>& issues,
                       uint64_t& files_checked, uint64_t& objects_checked);

}  // namespace tsb
