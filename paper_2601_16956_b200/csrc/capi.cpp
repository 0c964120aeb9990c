// extern "C" boundary (include/ts_b200.h). Exceptions never cross it: every
// entry point maps tsb::error to its ts_status and records the message.
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>

#include "engine.hpp"
#include "restore.hpp"
#include "uring.hpp"

using namespace tsb;

namespace {
thread_local std::string t_err;
thread_local int64_t t_err_oid = -1;

template <class F>
ts_status guard(F&& f) {
  try {
    f();
    t_err.clear();
    t_err_oid = -1;
    return TS_OK;
  } catch (const error& e) {
    t_err = e.what();
    t_err_oid = e.object_id;
    return e.status;
  } catch (const std::bad_alloc&) {
    t_err = "out of host memory";
    t_err_oid = -1;
    return TS_ERR_GENERIC;
  } catch (const std::exception& e) {
    t_err = e.what();
    t_err_oid = -1;
    return TS_ERR_GENERIC;
  }
}
}  // namespace

struct ts_engine {
  std::unique_ptr<engine> e;
};
struct ts_session {
  std::shared_ptr<session> s;  // shared with the jobs issued on it
};
struct ts_ticket {
  std::shared_ptr<ticket_state> t;
};
struct ts_restore {
  std::unique_ptr<restore_handle> r;
};

extern "C" {

const char* ts_last_error(void) { return t_err.c_str(); }
int64_t ts_last_error_object(void) { return t_err_oid; }
int ts_abi_version(void) { return TS_ABI_VERSION; }

// --- TLV -------------------------------------------------------------------

ts_value* ts_value_null(void) { return H(new value()); }
ts_value* ts_value_int(int64_t v) { return H(new value(v)); }
ts_value* ts_value_float(double v) { return H(new value(v)); }
ts_value* ts_value_string(const char* s, size_t n) { return H(new value(std::string(s, n))); }
ts_value* ts_value_bytes(const void* p, size_t n) {
  const auto* b = static_cast<const uint8_t*>(p);
  return H(new value(vbytes(b, b + n)));
}
ts_value* ts_value_list(void) { return H(new value(vlist{})); }
ts_value* ts_value_map(void) { return H(new value(vmap{})); }

ts_status ts_value_list_append(ts_value* list, ts_value* item) {
  return guard([&] {
    if (!list || !item || V(list)->type() != TS_V_LIST) fail(TS_ERR_INVALID_ARG, "not a list");
    std::unique_ptr<value> it(V(item));
    std::get<vlist>(V(list)->v).push_back(std::move(*it));
  });
}

ts_status ts_value_map_set(ts_value* map, const char* k, size_t kn, ts_value* v) {
  return guard([&] {
    if (!map || !v || V(map)->type() != TS_V_MAP) fail(TS_ERR_INVALID_ARG, "not a map");
    std::unique_ptr<value> it(V(v));
    std::get<vmap>(V(map)->v)[std::string(k, kn)] = std::move(*it);
  });
}

void ts_value_free(ts_value* v) { delete V(v); }
int ts_value_type(const ts_value* v) { return v ? V(v)->type() : -1; }
int64_t ts_value_as_int(const ts_value* v) {
  return v && V(v)->type() == TS_V_INT ? std::get<int64_t>(V(v)->v) : 0;
}
double ts_value_as_float(const ts_value* v) {
  return v && V(v)->type() == TS_V_FLOAT ? std::get<double>(V(v)->v) : 0.0;
}
const uint8_t* ts_value_data(const ts_value* v, size_t* n) {
  if (!v) return nullptr;
  if (V(v)->type() == TS_V_STRING) {
    const auto& s = std::get<std::string>(V(v)->v);
    *n = s.size();
    return reinterpret_cast<const uint8_t*>(s.data());
  }
  if (V(v)->type() == TS_V_BYTES) {
    const auto& b = std::get<vbytes>(V(v)->v);
    *n = b.size();
    return b.data();
  }
  *n = 0;
  return nullptr;
}
size_t ts_value_len(const ts_value* v) {
  if (!v) return 0;
  if (V(v)->type() == TS_V_LIST) return std::get<vlist>(V(v)->v).size();
  if (V(v)->type() == TS_V_MAP) return std::get<vmap>(V(v)->v).size();
  return 0;
}
const ts_value* ts_value_list_get(const ts_value* v, size_t i) {
  if (!v || V(v)->type() != TS_V_LIST) return nullptr;
  const auto& l = std::get<vlist>(V(v)->v);
  return i < l.size() ? H(&l[i]) : nullptr;
}
const ts_value* ts_value_map_key(const ts_value* v, size_t i, size_t* kn, const char** k) {
  if (!v || V(v)->type() != TS_V_MAP) return nullptr;
  const auto& m = std::get<vmap>(V(v)->v);
  if (i >= m.size()) return nullptr;
  auto it = m.begin();
  std::advance(it, static_cast<long>(i));
  *kn = it->first.size();
  *k = it->first.data();
  return H(&it->second);
}
size_t ts_value_encoded_size(const ts_value* v) { return v ? encoded_size(*V(v)) : 0; }
ts_status ts_value_encode(const ts_value* v, uint8_t* buf, size_t cap, size_t* len) {
  return guard([&] {
    if (!v) fail(TS_ERR_INVALID_ARG, "null value");
    const size_t need = encoded_size(*V(v));
    if (len) *len = need;
    if (cap < need) fail(TS_ERR_INVALID_ARG, "tlv: output buffer too small");
    size_t pos = 0;
    encode_into(*V(v), buf, &pos);
  });
}
ts_status ts_value_decode(const uint8_t* buf, size_t n, ts_value** out) {
  return guard([&] { *out = H(new value(decode(buf, n))); });
}
ts_value* ts_make_metadata_value(int rank_id, int tp_idx, int pp_idx, int dp_idx, uint64_t seed,
                                 uint64_t metadata_bytes, uint64_t iteration) {
  return H(new value(make_metadata_value(rank_id, tp_idx, pp_idx, dp_idx, seed, metadata_bytes, iteration)));
}

// --- planner / checksum ----------------------------------------------------

ts_status ts_plan_layout(const ts_object_desc* objs, size_t n, uint64_t alignment,
                         uint32_t* files_out, uint64_t* ends_out, size_t* n_files,
                         ts_fixed_assignment* fixed_out, uint32_t* fixed_file_out, size_t* n_fixed,
                         uint64_t* hash) {
  return guard([&] {
    const layout_plan p = plan_layout(objs, n, alignment);
    size_t k = 0;
    for (size_t f = 0; f < p.files.size(); ++f) {
      if (files_out) files_out[f] = p.files[f].file_id;
      if (ends_out) ends_out[f] = p.files[f].tensor_region_end;
      for (const auto& a : p.files[f].fixed) {
        if (fixed_out) fixed_out[k] = {a.object_id, a.file_offset, a.length};
        if (fixed_file_out) fixed_file_out[k] = p.files[f].file_id;
        ++k;
      }
    }
    if (n_files) *n_files = p.files.size();
    if (n_fixed) *n_fixed = k;
    if (hash) *hash = p.hash;
  });
}

uint64_t ts_fnv1a64(const void* p, size_t n, uint64_t state) { return fnv1a64(p, n, state); }

// --- engine / session / ticket ---------------------------------------------

void ts_engine_config_default(ts_engine_config* c) {
  std::memset(c, 0, sizeof *c);
  c->strategy = TS_STRATEGY_LAZY;
  c->lazy_serialize_overlap = 1;
  c->staging_capacity_bytes = 256ull << 20;
  c->flush_workers = 4;
  c->raw_chunk_bytes = 16ull << 20;
  c->serialized_chunk_bytes = 1ull << 20;
  c->alignment = 4096;
  c->cache_acquire_timeout_ns = 300ll * 1000000000ll;
  c->overwrite = 1;
  c->d2h_mode = TS_D2H_HYBRID;
  c->device_staging_bytes = 2ull << 30;
  c->hybrid_direct_min_bytes = 1ull << 20;
  c->pack_ctas = 0;
  c->pack_threads = 512;
  c->pack_priority = 1;
  c->write_files = 1;
  c->checksum_on_gpu = 1;
  c->flush_mmap = 1;
  c->pack_kernel = 1;
  c->bulk_min_bytes = 1ull << 20;
  c->file_dma = 1;
  c->checksum_priority = -1;
  c->checksum_host_frac = -1.0;
  c->ring_chunk_bytes = 0;
  c->numa_bind = 1;
  c->worker_nice = 19;
  c->helper_mask = 0;
  c->helper_share = 0.0;
  c->checksum_lane_max_bytes = 0;
}

ts_status ts_engine_create(const ts_engine_config* cfg, int rank_id, int device, ts_engine** out) {
  return guard([&] {
    ts_engine_config c;
    if (cfg) c = *cfg;
    else ts_engine_config_default(&c);
    auto* h = new ts_engine;
    try {
      h->e = std::make_unique<engine>(c, rank_id, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

ts_status ts_retire_checkpoint(const char* ckpt_dir, const char* spare_dir) {
  return guard([&] { retire_checkpoint(ckpt_dir, spare_dir); });
}

ts_status ts_engine_set_spare_dir(ts_engine* e, const char* spare_dir) {
  return guard([&] { e->e->set_spare_dir(spare_dir ? spare_dir : ""); });
}

uint64_t ts_file_cache_bytes(void) { return file_registry::get().registered_bytes(); }
void ts_file_cache_stats(uint64_t out[5]) { file_registry::get().stats(out); }

ts_status ts_file_cache_release_all(uint64_t* released_bytes) {
  return guard([&] {
    const uint64_t b = file_registry::get().release_all();
    if (released_bytes) *released_bytes = b;
  });
}

ts_status ts_engine_provision_spares(ts_engine* e, const char* spare_dir, const ts_rank_info* rank,
                                     const ts_object_desc* objs, size_t n, int copies,
                                     uint64_t* locked_bytes) {
  return guard([&] {
    const uint64_t b = e->e->provision_spares(spare_dir ? spare_dir : "", *rank, objs, n, copies);
    if (locked_bytes) *locked_bytes = b;
  });
}

int ts_engine_numa_node(ts_engine* e) { return e && e->e ? e->e->numa_node() : -1; }

ts_status ts_engine_destroy(ts_engine* e) {
  return guard([&] { delete e; });
}

ts_status ts_session_create(const char* dir, uint64_t checkpoint_id, uint64_t iteration,
                            const ts_manifest_echo* echo, int n_ranks, int writes_manifest,
                            ts_session** out) {
  return guard([&] {
    auto* h = new ts_session;
    h->s = std::make_shared<session>(dir ? dir : "", checkpoint_id, iteration, echo, n_ranks,
                                     writes_manifest != 0);
    *out = h;
  });
}

ts_status ts_session_destroy(ts_session* s) {
  return guard([&] { delete s; });
}

ts_status ts_session_rank_blob(ts_session* s, int rank_id, uint8_t* buf, size_t cap, size_t* len) {
  return guard([&] {
    const auto b = s->s->rank_blob(rank_id);
    if (len) *len = b.size();
    if (cap < b.size()) fail(TS_ERR_INVALID_ARG, "session: blob buffer too small");
    std::memcpy(buf, b.data(), b.size());
  });
}

ts_status ts_session_add_remote_rank(ts_session* s, const uint8_t* blob, size_t len) {
  return guard([&] { s->s->add_remote_rank(blob, len); });
}

ts_status ts_session_register_rank(ts_session* s, const ts_rank_info* rank, const ts_object_desc* objs,
                                   size_t n) {
  return guard([&] {
    if (!s || !rank || (!objs && n)) fail(TS_ERR_INVALID_ARG, "null argument");
    s->s->register_rank(make_rank_info(*rank, objs, n));
  });
}

ts_status ts_session_rank_persisted(ts_session* s, int rank_id) {
  return guard([&] { s->s->rank_persisted(rank_id); });
}

ts_status ts_session_wait_complete(ts_session* s, int64_t timeout_ns) {
  return guard([&] {
    if (!s->s->wait_complete(timeout_ns)) fail(TS_ERR_TICKET, "session: commit timed out");
  });
}

int ts_session_complete(ts_session* s) { return s->s->complete() ? 1 : 0; }

ts_status ts_issue(ts_engine* e, ts_session* s, const ts_rank_info* rank, const ts_object_desc* objs,
                   size_t n, uint64_t iteration, void* producer_stream, ts_ticket** out) {
  return guard([&] {
    if (!e || !s || !rank || (!objs && n)) fail(TS_ERR_INVALID_ARG, "ts_issue: null argument");
    auto t = e->e->issue(s->s, *rank, objs, n, iteration, static_cast<cudaStream_t>(producer_stream));
    *out = new ts_ticket{std::move(t)};
  });
}

ts_status ts_pre_update_barrier(ts_engine* e, ts_ticket* t, void* optimizer_stream, int host_block,
                                int64_t* blocked_ns) {
  return guard([&] {
    const int64_t dt = e->e->pre_update_barrier(t ? t->t : nullptr,
                                                static_cast<cudaStream_t>(optimizer_stream), host_block);
    if (blocked_ns) *blocked_ns = dt;
  });
}

ts_status ts_ticket_wait_captured(ts_ticket* t, int64_t* blocked_ns) {
  return guard([&] {
    const int64_t t0 = now_ns();
    t->t->wait_until([&] { return t->t->capture_recorded; });
    cuda_check(cudaSetDevice(t->t->device), "cudaSetDevice");
    cuda_check(cudaEventSynchronize(t->t->ev_capture), "cudaEventSynchronize(capture)");
    if (blocked_ns) *blocked_ns = now_ns() - t0;
  });
}

ts_status ts_ticket_wait_snapshot(ts_ticket* t, int64_t* blocked_ns) {
  return guard([&] {
    const int64_t dt = t->t->wait_until([&] { return t->t->snapshot; });
    if (blocked_ns) *blocked_ns = dt;
  });
}

ts_status ts_ticket_wait_persisted(ts_ticket* t, int64_t* blocked_ns) {
  return guard([&] {
    const int64_t dt = t->t->wait_until([&] { return t->t->persisted; });
    if (blocked_ns) *blocked_ns = dt;
  });
}

ts_status ts_ticket_stats_get(ts_ticket* t, ts_ticket_stats* o) {
  return guard([&] {
    auto& s = *t->t;
    std::lock_guard<std::mutex> g(s.mu);
    std::memset(o, 0, sizeof *o);
    o->checkpoint_id = s.checkpoint_id;
    o->total_bytes = s.total_bytes;
    o->raw_bytes = s.raw_bytes;
    o->serialized_bytes = s.serialized_bytes;
    o->image_bytes = s.image_bytes;
    o->issue_block_ns = s.issue_block_ns;
    o->barrier_block_ns = s.barrier_block_ns;
    o->t_captured_ns = s.t_captured;
    o->t_snapshot_ns = s.t_snapshot;
    o->t_persisted_ns = s.t_persisted;
    o->pack_ms = s.pack_ms;
    o->d2h_ms = s.d2h_ms;
    o->kernel_launches = s.kernel_launches;
    o->copies = s.copies;
    o->snapshot_done = s.snapshot;
    o->persisted_done = s.persisted;
    o->failed = s.failed;
    o->file_dma_bytes = s.file_dma_bytes;
    o->host_checksum_bytes = s.host_checksum_bytes;
    o->helper_bytes = s.helper_bytes;
    o->direct_io_bytes = s.direct_io_bytes;
    o->lane_checksum_bytes = s.lane_checksum_bytes;
    o->lane_ms = s.lane_ms;
    o->packed_bytes = s.packed_bytes;
  });
}

ts_status ts_ticket_object_checksum(ts_ticket* t, uint64_t object_id, uint64_t* out) {
  return guard([&] {
    std::lock_guard<std::mutex> g(t->t->mu);
    auto it = t->t->checksums.find(object_id);
    if (it == t->t->checksums.end()) fail(TS_ERR_INVALID_ARG, "no checksum for object", static_cast<int64_t>(object_id));
    *out = it->second;
  });
}

void ts_ticket_release(ts_ticket* t) { delete t; }

ts_status ts_ticket_adopt_values(ts_ticket* t, ts_value* const* values, size_t n) {
  return guard([&] {
    if (!t || (n && !values)) fail(TS_ERR_INVALID_ARG, "adopt_values: null argument");
    std::lock_guard<std::mutex> g(t->t->mu);
    for (size_t i = 0; i < n; ++i)
      if (values[i]) t->t->owned_values.emplace_back(V(values[i]));
  });
}

// --- restore / verify --------------------------------------------------------

ts_status ts_restore_set_file_cache(ts_restore* r, int use) {
  return guard([&] { r->r->use_file_cache = use != 0; });
}

ts_status ts_restore_set_direct_io(ts_restore* r, int use) {
  return guard([&] { r->r->direct_io = use < 0 ? -1 : use >= 2 ? 2 : use != 0; });
}

ts_status ts_restore_open(const char* manifest_path, ts_restore** out) {
  return guard([&] {
    auto* h = new ts_restore;
    try {
      h->r = std::make_unique<restore_handle>(manifest_path);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void ts_restore_close(ts_restore* r) { delete r; }
uint64_t ts_restore_release_staging(void) { return restore_release_staging(); }
int ts_io_uring_available(void) { return uring_available() ? 1 : 0; }
uint64_t ts_io_uring_ops(void) { return uring_ops(); }
int ts_restore_n_ranks(ts_restore* r) { return static_cast<int>(r->r->m.ranks.size()); }

ts_status ts_restore_rank_info(ts_restore* r, int index, ts_rank_info* out) {
  return guard([&] {
    const auto& mr = r->r->m.ranks.at(static_cast<size_t>(index));
    *out = {mr.rank_id, mr.tp_idx, mr.pp_idx, mr.dp_idx};
  });
}

ts_status ts_restore_rank_objects(ts_restore* r, int index, ts_restore_object* out, size_t cap,
                                  size_t* n) {
  return guard([&] {
    r->r->load_rank(index);
    const auto& mr = r->r->m.ranks.at(static_cast<size_t>(index));
    auto& rc = r->r->ranks[static_cast<size_t>(index)];
    if (n) *n = mr.objects.size();
    if (!out) return;
    if (cap < mr.objects.size()) fail(TS_ERR_INVALID_ARG, "restore: object buffer too small");
    for (size_t i = 0; i < mr.objects.size(); ++i) {
      const auto& o = mr.objects[i];
      out[i] = {o.object_id, o.kind, o.tier, o.precision, 0, o.file_id, rc.sizes.at(o.object_id)};
    }
  });
}

ts_status ts_restore_rank(ts_restore* r, int index, const ts_object_desc* dst, size_t n, int device,
                          void* stream, ts_restore_stats* stats) {
  return guard([&] {
    r->r->restore_rank(index, dst, n, device, static_cast<cudaStream_t>(stream), stats);
  });
}

ts_status ts_restore_structured(ts_restore* r, int index, uint64_t object_id, ts_value** out) {
  return guard([&] {
    auto& rc = r->r->ranks.at(static_cast<size_t>(index));
    auto it = rc.structured.find(object_id);
    if (it == rc.structured.end())
      fail(TS_ERR_INVALID_ARG, "restore: structured object not restored", static_cast<int64_t>(object_id));
    *out = H(new value(it->second));
  });
}

ts_status ts_verify(const char* manifest_path, ts_verify_report* rep, ts_verify_issue* issues, size_t cap) {
  return guard([&] {
    std::vector<std::pair<int, int64_t>> iss;
    uint64_t files = 0, objects = 0;
    verify_checkpoint(manifest_path, iss, files, objects);
    rep->ok = iss.empty() ? 1 : 0;
    rep->n_issues = static_cast<int32_t>(iss.size());
    rep->files_checked = files;
    rep->objects_checked = objects;
    for (size_t i = 0; i < iss.size() && i < cap; ++i) issues[i] = {iss[i].first, 0, iss[i].second};
  });
}

// --- device kernels of the synthetic state ----------------------------------

namespace {
struct pseg_table {
  std::vector<dev::pseg> h;
  uint64_t total = 0;
};
pseg_table make_psegs(const ts_pattern_desc* d, size_t n) {
  pseg_table t;
  t.h.reserve(n);
  for (size_t i = 0; i < n; ++i) {
    if (d[i].size == 0) continue;
    t.h.push_back({t.total, d[i].size, static_cast<uint8_t*>(d[i].data), d[i].space, d[i].offset});
    t.total += d[i].size;
  }
  return t;
}
void require_device() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(TS_ERR_CUDA, "no CUDA device: the B200 kernels have no CPU fallback");
  // The small per-call tables below come from the stream-ordered allocator: keep
  // its memory cached instead of unmapping it at every synchronization.
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = 256ull << 20;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.push_back(dev);
}
}  // namespace

ts_status ts_pattern_fill(const ts_pattern_desc* d, size_t n, uint64_t seed, uint64_t iteration, void* stream) {
  return guard([&] {
    require_device();
    auto t = make_psegs(d, n);
    if (t.h.empty()) return;
    auto st = static_cast<cudaStream_t>(stream);
    int dev = 0;
    cudaGetDevice(&dev);
    dev::pseg* p = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p), t.h.size() * sizeof(dev::pseg), st), "alloc");
    cuda_check(cudaMemcpyAsync(p, t.h.data(), t.h.size() * sizeof(dev::pseg), cudaMemcpyHostToDevice, st), "upload");
    dev::launch_pattern_fill(p, static_cast<uint32_t>(t.h.size()), t.total, seed, iteration,
                             dev::sm_count(dev) * 2, 512, st);
    cuda_check(cudaGetLastError(), "pattern fill launch");
    cuda_check(cudaFreeAsync(p, st), "free");
  });
}

ts_status ts_pattern_verify(const ts_pattern_desc* d, size_t n, uint64_t seed, uint64_t iteration,
                            void* stream, uint64_t* mismatched) {
  return guard([&] {
    require_device();
    auto t = make_psegs(d, n);
    *mismatched = 0;
    if (t.h.empty()) return;
    auto st = static_cast<cudaStream_t>(stream);
    int dev = 0;
    cudaGetDevice(&dev);
    dev::pseg* p = nullptr;
    unsigned long long* cnt = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p), t.h.size() * sizeof(dev::pseg), st), "alloc");
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&cnt), sizeof *cnt, st), "alloc");
    cuda_check(cudaMemsetAsync(cnt, 0, sizeof *cnt, st), "memset");
    cuda_check(cudaMemcpyAsync(p, t.h.data(), t.h.size() * sizeof(dev::pseg), cudaMemcpyHostToDevice, st), "upload");
    dev::launch_pattern_verify(p, static_cast<uint32_t>(t.h.size()), t.total, seed, iteration, cnt,
                               dev::sm_count(dev) * 2, 512, st);
    cuda_check(cudaGetLastError(), "pattern verify launch");
    unsigned long long h = 0;
    cuda_check(cudaMemcpyAsync(&h, cnt, sizeof h, cudaMemcpyDeviceToHost, st), "download");
    cuda_check(cudaFreeAsync(p, st), "free");
    cuda_check(cudaFreeAsync(cnt, st), "free");
    cuda_check(cudaStreamSynchronize(st), "sync");
    *mismatched = h;
  });
}

ts_status ts_pack(const void* const* srcs, const uint64_t* sizes, const uint64_t* dst_offsets, size_t n,
                  void* dst, uint64_t dst_len, int ctas, int threads, void* stream) {
  return guard([&] {
    require_device();
    auto st = static_cast<cudaStream_t>(stream);
    std::vector<size_t> order(n);
    for (size_t i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return dst_offsets[a] < dst_offsets[b]; });
    std::vector<dev::seg> segs;
    uint64_t cur = 0;
    for (size_t i : order) {
      if (sizes[i] == 0) continue;
      if (dst_offsets[i] < cur || dst_offsets[i] + sizes[i] > dst_len)
        fail(TS_ERR_INVALID_ARG, "ts_pack: overlapping or out-of-range destination");
      if (dst_offsets[i] > cur) segs.push_back({cur, dst_offsets[i] - cur, nullptr});
      segs.push_back({dst_offsets[i], sizes[i], static_cast<const uint8_t*>(srcs[i])});
      cur = dst_offsets[i] + sizes[i];
    }
    if (dst_len > cur) segs.push_back({cur, dst_len - cur, nullptr});
    if (segs.empty()) return;
    int dev = 0;
    cudaGetDevice(&dev);
    dev::seg* p = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p), segs.size() * sizeof(dev::seg), st), "alloc");
    cuda_check(cudaMemcpyAsync(p, segs.data(), segs.size() * sizeof(dev::seg), cudaMemcpyHostToDevice, st), "upload");
    dev::launch_pack(p, static_cast<uint32_t>(segs.size()), 0, dst_len, static_cast<uint8_t*>(dst),
                     ctas > 0 ? ctas : dev::sm_count(dev) * 2, threads > 0 ? threads : 512, st);
    cuda_check(cudaGetLastError(), "pack launch");
    cuda_check(cudaFreeAsync(p, st), "free");
  });
}

ts_status ts_unpack(const void* src, const uint64_t* src_offsets, void* const* dsts, const uint64_t* sizes,
                    size_t n, int ctas, int threads, void* stream) {
  return guard([&] {
    require_device();
    auto st = static_cast<cudaStream_t>(stream);
    std::vector<dev::useg> segs;
    uint64_t hi = 0;
    for (size_t i = 0; i < n; ++i) {
      if (sizes[i] == 0) continue;
      segs.push_back({src_offsets[i], sizes[i], static_cast<uint8_t*>(dsts[i])});
      hi = std::max(hi, src_offsets[i] + sizes[i]);
    }
    std::sort(segs.begin(), segs.end(), [](const dev::useg& a, const dev::useg& b) { return a.pos < b.pos; });
    for (size_t i = 1; i < segs.size(); ++i)
      if (segs[i].pos < segs[i - 1].pos + segs[i - 1].len) fail(TS_ERR_INVALID_ARG, "ts_unpack: overlapping sources");
    if (segs.empty()) return;
    int dev = 0;
    cudaGetDevice(&dev);
    dev::useg* p = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p), segs.size() * sizeof(dev::useg), st), "alloc");
    cuda_check(cudaMemcpyAsync(p, segs.data(), segs.size() * sizeof(dev::useg), cudaMemcpyHostToDevice, st), "upload");
    dev::launch_unpack(p, static_cast<uint32_t>(segs.size()), 0, hi, static_cast<const uint8_t*>(src),
                       ctas > 0 ? ctas : dev::sm_count(dev) * 2, threads > 0 ? threads : 512, st);
    cuda_check(cudaGetLastError(), "unpack launch");
    cuda_check(cudaFreeAsync(p, st), "free");
  });
}

uint64_t ts_kernel_launch_count(void) { return dev::launches(); }

ts_status ts_fnv1a64_device(const void* const* ptrs, const uint64_t* sizes, size_t n, const uint64_t* init,
                            uint64_t* out, void* stream) {
  return guard([&] {
    require_device();
    if (n == 0) return;
    auto st = static_cast<cudaStream_t>(stream);
    std::vector<dev::fnv_obj> objs(n);
    std::vector<uint64_t> states(n);
    for (size_t i = 0; i < n; ++i) {
      objs[i] = {static_cast<const uint8_t*>(ptrs[i]), sizes[i], 0, 0, i};
      states[i] = init ? init[i] : fnv_seed;
    }
    uint64_t nchunk = 0;
    const uint64_t nseg = dev::fnv_prepare(objs.data(), static_cast<uint32_t>(n), &nchunk);
    const uint64_t tb = dev::align_up_dev(n * sizeof(dev::fnv_obj), 256), sb = dev::align_up_dev(n * 8, 256);
    uint8_t* buf = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&buf),
                               tb + sb + dev::fnv_scratch_bytes(nseg, nchunk, static_cast<uint32_t>(n)), st), "alloc");
    cuda_check(cudaMemcpyAsync(buf, objs.data(), n * sizeof(dev::fnv_obj), cudaMemcpyHostToDevice, st), "upload");
    cuda_check(cudaMemcpyAsync(buf + tb, states.data(), n * 8, cudaMemcpyHostToDevice, st), "upload");
    dev::launch_fnv(reinterpret_cast<dev::fnv_obj*>(buf), static_cast<uint32_t>(n), nseg, nchunk,
                    reinterpret_cast<uint64_t*>(buf + tb), buf + tb + sb, st);
    cuda_check(cudaGetLastError(), "fnv launch");
    cuda_check(cudaMemcpyAsync(out, buf + tb, n * 8, cudaMemcpyDeviceToHost, st), "download");
    cuda_check(cudaFreeAsync(buf, st), "free");
    cuda_check(cudaStreamSynchronize(st), "sync");
  });
}

ts_status ts_fnv1a64_device_lanes(const void* const* ptrs, const uint64_t* sizes, size_t n, const uint64_t* init,
                                  uint64_t* out, void* stream) {
  return guard([&] {
    require_device();
    if (n == 0) return;
    auto st = static_cast<cudaStream_t>(stream);
    std::vector<dev::fnv_lane_obj> objs(n);
    for (size_t i = 0; i < n; ++i)
      objs[i] = {static_cast<const uint8_t*>(ptrs[i]), sizes[i], init ? init[i] : fnv_seed, i};
    std::stable_sort(objs.begin(), objs.end(), [](const auto& a, const auto& b) { return a.len > b.len; });
    const uint64_t tb = dev::align_up_dev(n * sizeof(dev::fnv_lane_obj), 256);
    uint8_t* buf = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&buf), tb + n * 8, st), "alloc");
    cuda_check(cudaMemcpyAsync(buf, objs.data(), n * sizeof(dev::fnv_lane_obj), cudaMemcpyHostToDevice, st),
               "upload");
    dev::launch_fnv_lanes(reinterpret_cast<dev::fnv_lane_obj*>(buf), static_cast<uint32_t>(n),
                          reinterpret_cast<uint64_t*>(buf + tb), st);
    cuda_check(cudaGetLastError(), "fnv lane launch");
    cuda_check(cudaMemcpyAsync(out, buf + tb, n * 8, cudaMemcpyDeviceToHost, st), "download");
    cuda_check(cudaFreeAsync(buf, st), "free");
    cuda_check(cudaStreamSynchronize(st), "sync");
  });
}

}  // extern "C"
