// Driver for the UNMODIFIED reference engine ("tierstream", /root/reference/proj).
//
// TEST INFRASTRUCTURE ONLY. Built by oracle/Makefile into oracle/_ref/ts_ref_driver
// from the reference's own sources. It is used (a) to generate the golden
// checkpoint trees under tests/golden/, (b) by `bench.py --impl reference` as the
// reference CPU arm, and (c) by tests to let the reference restore/verify files
// written by the B200 engine. Nothing in paper_2601_16956_b200/ links or calls it.
//
// The state it checkpoints is described by a "recipe":
//   checkpoint <ckpt_id> <iteration>
//   pattern_iteration <it>
//   layout <n_params> <layers> <hidden> <tp> <pp> <dp> <zero1> <seed> <metadata_bytes>
// or hand-built ranks:
//   rank <rank_id> <tp_idx> <pp_idx> <dp_idx> <seed> <metadata_bytes>
//   raw <oid> <file_id> <precision> <tier> <size> <space> <offset>
//   meta <oid> <file_id>
//   tmeta <oid> <file_id> <name> <dtype> <numel> <shard_off> <shard_len>
// Payloads are materialized with the reference's own fill_pattern
// (pattern.hpp:57-69) and make_metadata_value (model.cpp:206-231).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "tierstream/engine.hpp"
#include "tierstream/format.hpp"
#include "tierstream/model.hpp"
#include "tierstream/pattern.hpp"
#include "tierstream/provider.hpp"
#include "tierstream/tlv.hpp"

using namespace tierstream;

namespace {

struct recipe {
  uint64_t ckpt_id = 1;
  uint64_t iteration = 1;
  bool have_pattern_it = false;
  uint64_t pattern_it = 0;
  bool is_layout = false;
  shard_layout layout;
  std::vector<rank_state> ranks;  // hand-built
  struct tmeta_t {
    size_t rank_index;
    size_t obj_index;
    std::string name, dtype;
    int64_t numel, off, len;
  };
  std::vector<tmeta_t> tmetas;
  std::vector<std::pair<size_t, size_t>> metas;  // (rank_index, obj_index)
};

[[noreturn]] void die(const std::string& m) {
  std::fprintf(stderr, "ts_ref_driver: %s\n", m.c_str());
  std::exit(2);
}

recipe load_recipe(const std::string& path) {
  std::ifstream f(path);
  if (!f) die("cannot open recipe " + path);
  recipe r;
  std::string line;
  while (std::getline(f, line)) {
    auto hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    std::istringstream is(line);
    std::string kw;
    if (!(is >> kw)) continue;
    if (kw == "checkpoint") {
      is >> r.ckpt_id >> r.iteration;
    } else if (kw == "pattern_iteration") {
      is >> r.pattern_it;
      r.have_pattern_it = true;
    } else if (kw == "layout") {
      model_spec spec;
      int hidden, tp, pp, dp, zero1;
      uint64_t seed, meta;
      is >> spec.n_params >> spec.layers >> hidden >> tp >> pp >> dp >> zero1 >> seed >> meta;
      spec.hidden_dim = hidden;
      layout_options opt;
      opt.metadata_bytes = meta;
      r.layout = generate_layout(spec, tp, pp, dp, zero1 != 0, seed, opt);
      r.is_layout = true;
    } else if (kw == "rank") {
      rank_state rs;
      is >> rs.rank_id >> rs.tp_idx >> rs.pp_idx >> rs.dp_idx >> rs.seed >> rs.metadata_bytes;
      r.ranks.push_back(std::move(rs));
    } else if (kw == "raw" || kw == "meta" || kw == "tmeta") {
      if (r.ranks.empty()) die("object before rank line");
      auto& rs = r.ranks.back();
      state_object o;
      is >> o.object_id >> o.file_id;
      if (kw == "raw") {
        int prec, tr;
        is >> prec >> tr >> o.size_bytes >> o.pattern_space >> o.pattern_offset;
        o.kind = object_kind::raw_buffer;
        o.precision = static_cast<precision_tag>(prec);
        o.residency = static_cast<tier>(tr);
        o.size_known = true;
      } else {
        o.kind = object_kind::structured;
        o.residency = tier::host;
        o.precision = precision_tag::opaque;
        if (kw == "meta") {
          r.metas.push_back({r.ranks.size() - 1, rs.objects.size()});
        } else {
          recipe::tmeta_t t;
          t.rank_index = r.ranks.size() - 1;
          t.obj_index = rs.objects.size();
          is >> t.name >> t.dtype >> t.numel >> t.off >> t.len;
          r.tmetas.push_back(t);
        }
      }
      if (!is) die("bad object line: " + line);
      rs.objects.push_back(std::move(o));
    } else {
      die("unknown recipe keyword " + kw);
    }
  }
  if (!r.have_pattern_it) r.pattern_it = r.iteration;
  if (!r.is_layout) {
    for (auto& rs : r.ranks) {
      std::vector<uint32_t> fids;
      for (auto& o : rs.objects) {
        bool seen = false;
        for (auto x : fids) seen |= x == o.file_id;
        if (!seen) fids.push_back(o.file_id);
      }
      rs.file_ids = fids;
    }
  }
  return r;
}

std::vector<rank_state>& ranks_of(recipe& r) { return r.is_layout ? r.layout.ranks : r.ranks; }

void materialize(recipe& r) {
  // (harness setup, not timed: the reference's fill_pattern per object, objects
  // spread over the host threads this process may use)
  auto& ranks = ranks_of(r);
  std::vector<std::pair<rank_state*, state_object*>> todo;
  for (auto& rs : ranks)
    for (auto& o : rs.objects)
      if (o.is_raw()) todo.push_back({&rs, &o});
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t k; (k = next++) < todo.size();) {
      auto& [rs, o] = todo[k];
      o->payload.resize(o->size_bytes);
      fill_pattern(o->payload, pattern_key{rs->seed, o->pattern_space, r.pattern_it}, o->pattern_offset);
    }
  };
  const unsigned nt = std::max(1u, std::min<unsigned>(32, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned t = 1; t < nt; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  if (r.is_layout) {
    for (auto& rs : ranks)
      for (auto& o : rs.objects)
        if (!o.is_raw()) o.structured = make_metadata_value(rs, r.pattern_it);
  } else {
    for (auto [ri, oi] : r.metas) ranks[ri].objects[oi].structured = make_metadata_value(ranks[ri], r.pattern_it);
    for (auto& t : r.tmetas) {
      tlv::map m;
      m.emplace("name", tlv::value(t.name));
      m.emplace("dtype", tlv::value(t.dtype));
      m.emplace("numel", tlv::value(t.numel));
      m.emplace("shard_offset", tlv::value(t.off));
      m.emplace("shard_len", tlv::value(t.len));
      m.emplace("iteration", tlv::value(static_cast<int64_t>(r.pattern_it)));
      ranks[t.rank_index].objects[t.obj_index].structured = tlv::value(std::move(m));
    }
  }
}

struct opts_t {
  int workers = 1;
  uint64_t cache = 256_MiB;
  uint64_t raw_chunk = default_raw_chunk_bytes;
  uint64_t ser_chunk = default_serialized_chunk_bytes;
  int reps = 1;
  int warmup = 0;
  bool restore = false;       // restore after every step
  bool restore_last = false;  // restore once, after the last step
  std::string strategy = "lazy";
};

double secs(int64_t ns) { return static_cast<double>(ns) / 1e9; }

// One checkpoint of every rank in the recipe, ranks as threads of this process
// (the reference's own multi-rank model, simulator.cpp:113-175).
struct ckpt_timing {
  int64_t issue_ns = 0, snapshot_ns = 0, persist_ns = 0;
  uint64_t bytes = 0;
};

std::vector<ckpt_timing> run_checkpoint(exec_context& ctx, recipe& r, const std::string& dir,
                                        const opts_t& o, uint64_t ckpt_id) {
  engine_config cfg;
  cfg.flush_workers = o.workers;
  cfg.staging_capacity_bytes = o.cache;
  cfg.raw_chunk_bytes = o.raw_chunk;
  cfg.serialized_chunk_bytes = o.ser_chunk;
  if (o.strategy == "sync") cfg.strategy = strategy_kind::sync;
  else if (o.strategy == "two_phase") cfg.strategy = strategy_kind::two_phase;
  auto& ranks = ranks_of(r);
  std::unique_ptr<checkpoint_session> session;
  if (r.is_layout)
    session = std::make_unique<checkpoint_session>(ctx, dir, ckpt_id, r.iteration, r.layout);
  else
    session = std::make_unique<checkpoint_session>(ctx, dir, ckpt_id, r.iteration,
                                                   static_cast<int>(ranks.size()));
  std::vector<ckpt_timing> out(ranks.size());
  std::vector<scoped_task> tasks;
  for (size_t i = 0; i < ranks.size(); ++i) {
    tasks.push_back({ranks[i].rank_id, 0, [&, i] {
                       checkpoint_engine eng(ctx, cfg, ranks[i].rank_id);
                       const int64_t t0 = ctx.now_ns();
                       auto t = eng.issue_checkpoint(*session, ranks[i], r.iteration);
                       const int64_t t1 = ctx.now_ns();
                       t->wait_snapshot();
                       const int64_t t2 = ctx.now_ns();
                       t->wait_persisted();
                       const int64_t t3 = ctx.now_ns();
                       out[i] = {t1 - t0, t2 - t0, t3 - t0, t->total_bytes()};
                       eng.shutdown();
                     }});
  }
  run_tasks(ctx, std::move(tasks));
  session->wait_complete();
  return out;
}

std::string hex64(uint64_t v) {
  char b[17];
  std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(v));
  return b;
}

std::string hexbytes(const std::byte* p, size_t n) {
  std::string s;
  char b[3];
  for (size_t i = 0; i < n; ++i) {
    std::snprintf(b, sizeof b, "%02x", static_cast<unsigned>(p[i]));
    s += b;
  }
  return s;
}

int cmd_kat() {
  // Known-answer values printed from the reference itself.
  auto fnv = [](const char* s) {
    return fnv1a64(std::span<const std::byte>(reinterpret_cast<const std::byte*>(s), std::strlen(s)));
  };
  std::printf("{\n");
  std::printf("\"fnv_empty\": \"%s\",\n", hex64(fnv("")).c_str());
  std::printf("\"fnv_a\": \"%s\",\n", hex64(fnv("a")).c_str());
  std::printf("\"fnv_foobar\": \"%s\",\n", hex64(fnv("foobar")).c_str());
  std::vector<std::byte> p(24);
  const uint64_t space = (1ull << 56);
  fill_pattern(p, pattern_key{42, space, 0}, 0);
  std::printf("\"pattern_42_L0_it0_off0\": \"%s\",\n", hexbytes(p.data(), 24).c_str());
  fill_pattern(p, pattern_key{42, space, 1}, 5);
  std::printf("\"pattern_42_L0_it1_off5\": \"%s\",\n", hexbytes(p.data(), 24).c_str());
  tlv::map m;
  m.emplace("iteration", tlv::value(7));
  m.emplace("rng_seed", tlv::value(42));
  auto e = tlv::encode(tlv::value(m));
  std::printf("\"tlv_iter7_seed42\": \"%s\",\n", hexbytes(e.data(), e.size()).c_str());
  auto e0 = tlv::encode(tlv::value(tlv::map{}));
  std::printf("\"tlv_empty_map\": \"%s\",\n", hexbytes(e0.data(), e0.size()).c_str());
  tlv::list l;
  l.emplace_back(nullptr);
  l.emplace_back(1.5);
  l.emplace_back(std::string("h\xc3\xa9"));
  l.emplace_back(tlv::bytes{std::byte{1}, std::byte{2}});
  l.emplace_back(static_cast<int64_t>(-3));
  auto el = tlv::encode(tlv::value(l));
  std::printf("\"tlv_mixed_list\": \"%s\",\n", hexbytes(el.data(), el.size()).c_str());
  // plan_layout examples
  std::vector<state_object> objs(4);
  uint64_t sizes[3] = {3500000000ull, 1000000000ull, 4096};
  for (int i = 0; i < 3; ++i) {
    objs[i].object_id = static_cast<uint64_t>(i + 1);
    objs[i].file_id = 1;
    objs[i].size_bytes = sizes[i];
    objs[i].size_known = true;
  }
  objs[3].object_id = 4;
  objs[3].kind = object_kind::structured;
  objs[3].file_id = 0;
  auto plan = plan_layout(objs, 4096);
  std::printf("\"plan3_offsets\": [%llu, %llu, %llu],\n",
              (unsigned long long)plan.file(1).fixed[0].file_offset,
              (unsigned long long)plan.file(1).fixed[1].file_offset,
              (unsigned long long)plan.file(1).fixed[2].file_offset);
  std::printf("\"plan3_end_f1\": %llu,\n\"plan3_end_f0\": %llu,\n\"plan3_hash\": \"%s\",\n",
              (unsigned long long)plan.file(1).tensor_region_end,
              (unsigned long long)plan.file(0).tensor_region_end, hex64(plan.plan_hash()).c_str());
  std::vector<state_object> one(1);
  one[0].object_id = 1;
  one[0].file_id = 1;
  one[0].size_bytes = 4096;
  one[0].size_known = true;
  auto p1 = plan_layout(one, 4096);
  std::printf("\"plan1_hash\": \"%s\",\n\"plan1_end\": %llu,\n", hex64(p1.plan_hash()).c_str(),
              (unsigned long long)p1.file(1).tensor_region_end);
  layout_plan empty = plan_layout({}, 4096);
  std::printf("\"plan_empty_hash\": \"%s\",\n", hex64(empty.plan_hash()).c_str());
  rank_state rs;
  rs.rank_id = 0;
  rs.seed = 42;
  rs.metadata_bytes = 2_MiB;
  auto mv = tlv::encode(make_metadata_value(rs, 0));
  std::printf("\"metadata_2MiB_len\": %zu,\n", mv.size());
  std::printf("\"metadata_2MiB_fnv\": \"%s\"\n",
              hex64(fnv1a64(std::span<const std::byte>(mv.data(), mv.size()))).c_str());
  std::printf("}\n");
  return 0;
}

int cmd_write(recipe& r, const std::string& dir, const opts_t& o) {
  materialize(r);
  wall_context ctx;
  auto t = run_checkpoint(ctx, r, dir, o, r.ckpt_id);
  uint64_t bytes = 0;
  int64_t snap = 0, pers = 0, iss = 0;
  for (auto& x : t) {
    bytes += x.bytes;
    snap = std::max(snap, x.snapshot_ns);
    pers = std::max(pers, x.persist_ns);
    iss = std::max(iss, x.issue_ns);
  }
  std::printf("{\"bytes\": %llu, \"issue_s\": %.6f, \"snapshot_s\": %.6f, \"persist_s\": %.6f}\n",
              (unsigned long long)bytes, secs(iss), secs(snap), secs(pers));
  return 0;
}

// Reference CPU arm for bench.py: repeated lazy checkpoints of the recipe state,
// every step = one checkpoint issued, snapshot, persisted (and optionally restored).
int cmd_bench(recipe& r, const std::string& dir, const opts_t& o) {
  auto tm0 = std::chrono::steady_clock::now();
  materialize(r);
  const double t_mat =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - tm0).count();
  wall_context ctx;
  for (int s = 0; s < o.warmup + o.reps; ++s) {
    auto t = run_checkpoint(ctx, r, dir, o, r.ckpt_id);
    uint64_t bytes = 0;
    int64_t snap = 0, pers = 0, iss = 0;
    for (auto& x : t) {
      bytes += x.bytes;
      snap = std::max(snap, x.snapshot_ns);
      pers = std::max(pers, x.persist_ns);
      iss = std::max(iss, x.issue_ns);
    }
    double restore_s = -1;
    if (o.restore || (o.restore_last && s + 1 == o.warmup + o.reps)) {
      auto a = std::chrono::steady_clock::now();
      auto st = restore_checkpoint(std::filesystem::path(dir) / "MANIFEST.tlv");
      restore_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
      (void)st;
    }
    std::printf(
        "{\"step\": %d, \"warmup\": %s, \"bytes\": %llu, \"issue_s\": %.6f, \"snapshot_s\": %.6f, "
        "\"persist_s\": %.6f, \"restore_s\": %.6f, \"materialize_s\": %.3f}\n",
        s, s < o.warmup ? "true" : "false", (unsigned long long)bytes, secs(iss), secs(snap),
        secs(pers), restore_s, t_mat);
    std::fflush(stdout);
  }
  return 0;
}

// Restore with the reference reader and print per-object FNV + size, so tests can
// check that files written by the B200 engine restore under the reference.
int cmd_restore(const std::string& manifest) {
  try {
    auto ranks = restore_checkpoint(manifest);
    std::printf("{\"ok\": true, \"ranks\": [");
    for (size_t i = 0; i < ranks.size(); ++i) {
      std::printf("%s{\"rank_id\": %d, \"objects\": [", i ? ", " : "", ranks[i].rank_id);
      for (size_t j = 0; j < ranks[i].objects.size(); ++j) {
        const auto& ob = ranks[i].objects[j];
        uint64_t h;
        if (ob.is_raw()) h = fnv1a64(ob.payload);
        else {
          auto e = tlv::encode(ob.structured);
          h = fnv1a64(std::span<const std::byte>(e.data(), e.size()));
        }
        std::printf("%s[%llu, %d, %llu, \"%s\"]", j ? ", " : "", (unsigned long long)ob.object_id,
                    static_cast<int>(ob.kind), (unsigned long long)ob.size_bytes, hex64(h).c_str());
      }
      std::printf("]}");
    }
    std::printf("]}\n");
  } catch (const format_error& e) {
    std::printf("{\"ok\": false, \"kind\": %d, \"object_id\": %lld, \"what\": \"%s\"}\n",
                static_cast<int>(e.kind), e.object_id ? (long long)*e.object_id : -1LL, e.what());
  }
  return 0;
}

int cmd_verify(const std::string& manifest) {
  auto rep = verify_checkpoint(manifest);
  std::printf("{\"ok\": %s, \"files\": %zu, \"objects\": %zu, \"issues\": [", rep.ok ? "true" : "false",
              rep.files_checked, rep.objects_checked);
  for (size_t i = 0; i < rep.issues.size(); ++i)
    std::printf("%s[%d, %lld]", i ? ", " : "", static_cast<int>(rep.issues[i].kind),
                rep.issues[i].object_id ? (long long)*rep.issues[i].object_id : -1LL);
  std::printf("]}\n");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) die("usage: ts_ref_driver kat | write|bench <recipe> <dir> [opts] | restore|verify <manifest>");
  std::string cmd = argv[1];
  if (cmd == "kat") return cmd_kat();
  if ((cmd == "restore" || cmd == "verify") && argc >= 3)
    return cmd == "restore" ? cmd_restore(argv[2]) : cmd_verify(argv[2]);
  if (argc < 4) die("missing recipe/dir");
  opts_t o;
  for (int i = 4; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) die("missing value for " + a);
      return argv[++i];
    };
    if (a == "--workers") o.workers = std::stoi(next());
    else if (a == "--cache") o.cache = std::stoull(next());
    else if (a == "--raw-chunk") o.raw_chunk = std::stoull(next());
    else if (a == "--ser-chunk") o.ser_chunk = std::stoull(next());
    else if (a == "--reps") o.reps = std::stoi(next());
    else if (a == "--warmup") o.warmup = std::stoi(next());
    else if (a == "--restore") o.restore = true;
    else if (a == "--restore-last") o.restore_last = true;
    else if (a == "--strategy") o.strategy = next();
    else die("unknown option " + a);
  }
  recipe r = load_recipe(argv[2]);
  try {
    if (cmd == "write") return cmd_write(r, argv[3], o);
    if (cmd == "bench") return cmd_bench(r, argv[3], o);
  } catch (const std::exception& e) {
    die(std::string("error: ") + e.what());
  }
  die("unknown command " + cmd);
}
