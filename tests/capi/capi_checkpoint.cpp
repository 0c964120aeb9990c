// End-to-end use of the engine through the C-ABI alone (include/ts_b200.h):
// what a C++ caller of the reference's checkpoint_engine (engine.hpp:92-153)
// binds. No Python, no torch: device state from cudaMalloc, filled by
// ts_pattern_fill; one lazy checkpoint of every rank of a recipe through
// ts_issue; restore into fresh device buffers and a bit-exact check with
// ts_pattern_verify; ts_verify over the written tree.
//
//   capi_checkpoint <spec file> <out dir>
// spec (written by tests/test_gpu_capi.py from a golden recipe):
//   checkpoint <id> <iteration>
//   pattern_iteration <it>
//   echo <tp> <pp> <dp> <zero1> <seed> <n_params> <layers> <metadata_bytes>   (optional)
//   rank <id> <tp> <pp> <dp> <seed> <metadata_bytes>
//   raw <id> <file> <precision> <tier> <size> <space> <offset>
//   meta <id> <file>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "ts_b200.h"

namespace {
#define CHECK(x)                                                                 \
  do {                                                                           \
    const ts_status s_ = (x);                                                    \
    if (s_ != TS_OK) {                                                           \
      std::fprintf(stderr, "%s failed: %d %s\n", #x, s_, ts_last_error());       \
      std::exit(2);                                                              \
    }                                                                            \
  } while (0)

struct obj {
  uint64_t id = 0, size = 0, space = 0, offset = 0;
  uint32_t file = 0;
  int kind = 0, tier = 0, precision = 0;
  void* data = nullptr;
  ts_value* value = nullptr;
};
struct rank {
  ts_rank_info info{};
  uint64_t seed = 0, metadata_bytes = 0;
  std::vector<obj> objs;
};

std::vector<ts_pattern_desc> pattern_descs(const rank& r) {
  std::vector<ts_pattern_desc> v;
  for (const auto& o : r.objs)
    if (o.kind == TS_KIND_RAW && o.tier == TS_TIER_DEVICE) v.push_back({o.data, o.size, o.space, o.offset});
  return v;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: %s <spec> <out dir>\n", argv[0]);
    return 1;
  }
  uint64_t ckpt_id = 0, iteration = 0, pit = 0;
  bool have_echo = false;
  ts_manifest_echo echo{};
  std::vector<rank> ranks;
  std::ifstream in(argv[1]);
  for (std::string line; std::getline(in, line);) {
    std::istringstream ss(line);
    std::string k;
    ss >> k;
    if (k == "checkpoint") {
      ss >> ckpt_id >> iteration;
      pit = iteration;
    } else if (k == "pattern_iteration") {
      ss >> pit;
    } else if (k == "echo") {
      ss >> echo.tp >> echo.pp >> echo.dp >> echo.zero1 >> echo.seed >> echo.n_params >> echo.layers >>
          echo.metadata_bytes;
      have_echo = true;
    } else if (k == "rank") {
      rank r;
      ss >> r.info.rank_id >> r.info.tp_idx >> r.info.pp_idx >> r.info.dp_idx >> r.seed >> r.metadata_bytes;
      ranks.push_back(r);
    } else if (k == "raw") {
      obj o;
      ss >> o.id >> o.file >> o.precision >> o.tier >> o.size >> o.space >> o.offset;
      o.kind = TS_KIND_RAW;
      ranks.back().objs.push_back(o);
    } else if (k == "meta") {
      obj o;
      ss >> o.id >> o.file;
      o.kind = TS_KIND_STRUCTURED;
      o.tier = TS_TIER_HOST;
      o.precision = TS_PREC_OPAQUE;
      ranks.back().objs.push_back(o);
    }
  }

  // Device state at the pattern iteration (materialize_payloads, model.cpp:195-204).
  for (auto& r : ranks) {
    for (auto& o : r.objs) {
      if (o.kind == TS_KIND_RAW) {
        if (o.tier != TS_TIER_DEVICE) {
          std::fprintf(stderr, "host-tier objects are not part of this driver\n");
          return 1;
        }
        if (cudaMalloc(&o.data, o.size) != cudaSuccess) return 3;
      } else {
        o.value = ts_make_metadata_value(r.info.rank_id, r.info.tp_idx, r.info.pp_idx, r.info.dp_idx, r.seed,
                                         r.metadata_bytes, pit);
      }
    }
    const auto pd = pattern_descs(r);
    CHECK(ts_pattern_fill(pd.data(), pd.size(), r.seed, pit, nullptr));
  }
  cudaDeviceSynchronize();

  // One lazy checkpoint of every rank (engines of one process share the session).
  ts_engine_config cfg;
  ts_engine_config_default(&cfg);
  cfg.raw_chunk_bytes = 64 << 10;
  cfg.staging_capacity_bytes = 1 << 20;
  cfg.device_staging_bytes = 256 << 10;
  ts_session* sess = nullptr;
  CHECK(ts_session_create(argv[2], ckpt_id, iteration, have_echo ? &echo : nullptr, static_cast<int>(ranks.size()),
                          1, &sess));
  std::vector<ts_engine*> engines;
  std::vector<ts_ticket*> tickets;
  for (auto& r : ranks) {
    ts_engine* e = nullptr;
    CHECK(ts_engine_create(&cfg, r.info.rank_id, 0, &e));
    std::vector<ts_object_desc> d;
    for (const auto& o : r.objs)
      d.push_back({o.id, static_cast<uint8_t>(o.kind), static_cast<uint8_t>(o.tier), static_cast<uint8_t>(o.precision),
                   0, o.file, o.size, o.data, o.value});
    ts_ticket* t = nullptr;
    CHECK(ts_issue(e, sess, &r.info, d.data(), d.size(), iteration, nullptr, &t));
    // non-blocking ownership hand-over: the ticket frees the structured values
    std::vector<ts_value*> owned;
    for (auto& o : r.objs)
      if (o.value) owned.push_back(o.value), o.value = nullptr;
    CHECK(ts_ticket_adopt_values(t, owned.data(), owned.size()));
    // lazy contract: before mutating the state, the pre-update barrier
    int64_t blocked = 0;
    CHECK(ts_pre_update_barrier(e, t, nullptr, 1, &blocked));
    engines.push_back(e);
    tickets.push_back(t);
  }
  for (auto* t : tickets) CHECK(ts_ticket_wait_persisted(t, nullptr));
  CHECK(ts_session_wait_complete(sess, 60ll * 1000000000ll));

  // Restore every rank into fresh device buffers, bit-exact against the pattern.
  const std::string man = std::string(argv[2]) + "/MANIFEST.tlv";
  ts_restore* rs = nullptr;
  CHECK(ts_restore_open(man.c_str(), &rs));
  uint64_t bad_total = 0;
  for (int i = 0; i < ts_restore_n_ranks(rs); ++i) {
    ts_rank_info ri{};
    CHECK(ts_restore_rank_info(rs, i, &ri));
    rank* src = nullptr;
    for (auto& r : ranks)
      if (r.info.rank_id == ri.rank_id) src = &r;
    if (!src) return 4;
    rank dst = *src;
    std::vector<ts_object_desc> d;
    for (auto& o : dst.objs) {
      if (o.kind != TS_KIND_RAW) continue;
      if (cudaMalloc(&o.data, o.size) != cudaSuccess) return 3;
      cudaMemset(o.data, 0, o.size);
      d.push_back({o.id, static_cast<uint8_t>(o.kind), static_cast<uint8_t>(o.tier), static_cast<uint8_t>(o.precision),
                   0, o.file, o.size, o.data, nullptr});
    }
    ts_restore_stats st{};
    CHECK(ts_restore_rank(rs, i, d.data(), d.size(), 0, nullptr, &st));
    const auto pd = pattern_descs(dst);
    uint64_t bad = 0;
    CHECK(ts_pattern_verify(pd.data(), pd.size(), dst.seed, pit, nullptr, &bad));
    bad_total += bad;
    for (auto& o : dst.objs)
      if (o.data) cudaFree(o.data);
  }
  ts_restore_close(rs);
  ts_verify_report rep{};
  ts_verify_issue issues[16];
  CHECK(ts_verify(man.c_str(), &rep, issues, 16));
  for (auto* t : tickets) ts_ticket_release(t);
  for (auto* e : engines) CHECK(ts_engine_destroy(e));
  CHECK(ts_session_destroy(sess));
  for (auto& r : ranks)
    for (auto& o : r.objs) {
      if (o.data) cudaFree(o.data);
      if (o.value) ts_value_free(o.value);
    }
  std::printf("{\"ranks\": %zu, \"restore_mismatched_bytes\": %llu, \"verify_ok\": %d, \"objects_checked\": %llu}\n",
              ranks.size(), static_cast<unsigned long long>(bad_total), rep.ok,
              static_cast<unsigned long long>(rep.objects_checked));
  return bad_total == 0 && rep.ok ? 0 : 5;
}
