// checkpoint_session (engine.cpp:35-117): per-rank manifest info, manifest-last
// commit once every rank persisted. See engine.hpp.
#include <algorithm>
#include <unordered_map>

#include "engine.hpp"

namespace tsb {

// ---------------------------------------------------------------------------
// session (engine.cpp:35-117): manifest written last, ranks sorted by id.

manifest_rank make_rank_info(const ts_rank_info& rank, const ts_object_desc* objs, size_t n) {
  manifest_rank info;
  info.rank_id = rank.rank_id;
  info.tp_idx = rank.tp_idx;
  info.pp_idx = rank.pp_idx;
  info.dp_idx = rank.dp_idx;
  std::vector<uint32_t> fids;
  for (size_t i = 0; i < n; ++i) fids.push_back(objs[i].file_id);
  std::sort(fids.begin(), fids.end());
  fids.erase(std::unique(fids.begin(), fids.end()), fids.end());
  std::unordered_map<uint32_t, size_t> at;
  for (uint32_t f : fids) {
    at.emplace(f, info.files.size());
    manifest_file mf;
    mf.file_id = f;
    mf.path = rank_dir_name(rank.rank_id) + "/file_" + std::to_string(f) + ".bin";
    info.files.push_back(std::move(mf));
  }
  for (size_t i = 0; i < n; ++i) {
    info.files[at.at(objs[i].file_id)].object_ids.push_back(objs[i].object_id);
    info.objects.push_back({objs[i].object_id, objs[i].kind, objs[i].tier, objs[i].precision,
                            objs[i].file_id});
  }
  return info;
}

session::session(const std::string& dir, uint64_t ckpt_id, uint64_t iteration,
                 const ts_manifest_echo* echo, int n_ranks, bool writes)
    : dir_(dir), n_ranks_(n_ranks), writes_(writes) {
  m_.checkpoint_id = ckpt_id;
  m_.iteration = iteration;
  if (echo) {
    m_.tp = echo->tp;
    m_.pp = echo->pp;
    m_.dp = echo->dp;
    m_.zero1 = echo->zero1 != 0;
    m_.seed = echo->seed;
    m_.n_params = echo->n_params;
    m_.layers = echo->layers;
    m_.metadata_bytes = echo->metadata_bytes;
  }
  if (writes_ || !dir_.empty()) mkdirs(dir_);
}

void session::register_rank(manifest_rank info) {
  std::lock_guard<std::mutex> g(mu_);
  const int id = info.rank_id;
  ranks_[id] = std::move(info);
  persisted_.emplace(id, false);
}

std::vector<uint8_t> session::rank_blob(int rank_id) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = ranks_.find(rank_id);
  if (it == ranks_.end()) fail(TS_ERR_INVALID_ARG, "session: unknown rank");
  return encode(rank_to_value(it->second));
}

void session::add_remote_rank(const uint8_t* blob, size_t n) {
  manifest_rank r = rank_from_value(decode(blob, n));
  std::unique_lock<std::mutex> g(mu_);
  const int id = r.rank_id;
  ranks_[id] = std::move(r);
  persisted_[id] = true;
  maybe_commit_locked(g);
}

void session::rank_persisted(int rank_id) {
  std::unique_lock<std::mutex> g(mu_);
  persisted_[rank_id] = true;
  maybe_commit_locked(g);
}

void session::maybe_commit_locked(std::unique_lock<std::mutex>& g) {
  int done = 0;
  for (const auto& [id, p] : persisted_) done += p ? 1 : 0;
  if (complete_ || committing_) return;
  if (!writes_) {
    if (done == static_cast<int>(persisted_.size())) {
      complete_ = true;
      cv_.notify_all();
    }
    return;
  }
  if (done < n_ranks_) return;
  committing_ = true;
  manifest m = m_;
  m.complete = true;
  for (const auto& [id, r] : ranks_) m.ranks.push_back(r);
  g.unlock();
  std::string err;
  try {
    write_manifest(dir_ + "/MANIFEST.tlv", m);
  } catch (const error& e) {
    err = e.what();
  }
  g.lock();
  commit_error_ = err;
  complete_ = true;
  cv_.notify_all();
  if (!err.empty()) fail(TS_ERR_IO, err);
}

bool session::wait_complete(int64_t timeout_ns) {
  std::unique_lock<std::mutex> g(mu_);
  if (timeout_ns < 0) cv_.wait(g, [&] { return complete_; });
  else cv_.wait_for(g, std::chrono::nanoseconds(timeout_ns), [&] { return complete_; });
  if (complete_ && !commit_error_.empty()) fail(TS_ERR_IO, commit_error_);
  return complete_;
}

bool session::complete() {
  std::lock_guard<std::mutex> g(mu_);
  return complete_;
}

}  // namespace tsb
