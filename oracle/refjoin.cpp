// refjoin — a driver around the UNMODIFIED reference library (test
// infrastructure; built by oracle/Makefile into oracle/_ref/, never linked into
// the product).  It is the "reference arm" of bench.py and the generator of the
// golden fixtures under tests/golden/.
//
//   refjoin join  [workload opts] --algo phj|smj --pattern gftr|gfur
//                 [--reps N] [--warmup W] [--threads T] [--prealloc] [--digest] [--pdigest]
//                 [--dump DIR]   (--pdigest: canonical digest by a parallel sort)
//   refjoin prim  --n N --seed S [--dump DIR]
//   refjoin gen   [workload opts] --dump DIR
//   refjoin star  --fact N --dims D --dim-rows M --seed S --algo phj|smj --pattern gftr|gfur
//                 [--reps N] [--threads T]   (workloads::gen_star + the reference's
//                 run_join_sequence loop, sequence.cpp:9-67, keeping the last output)
//   refjoin export [workload opts] --dir DIR   (workloads::export_relation of R, S
//                 into DIR/R, DIR/S; prints the generator digests)
//   refjoin import --dir DIR                  (workloads::import_relation; prints
//                 name, rows, key_unique, column kinds and digests)
//   refjoin report --in CSV                   (benchio::read_csv + render_report)
//   (--swap builds on S, whose keys repeat, and probes with R)
//
// Workload options mirror workloads::WorkloadSpec (workloads.hpp:11-21):
//   --r N --s N --rpay K --spay K --key u32|u64 --pay u32|u64 --match F
//   --zipf F --seed S [--widths 4,8,4,8]  (C3: per-column widths; generated as
//   u64 and truncated to u32 where the width is 4)
//
// Timing follows run_join's own PhaseReport (mem_ledger.hpp:231-246): total =
// transform + find + materialise; generation is excluded.

#include <omp.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include <iostream>
#include <sstream>

#include "coljoin/bench_io.hpp"
#include "coljoin/hash_match.hpp"
#include "coljoin/join_engine.hpp"
#include "coljoin/merge_match.hpp"
#include "coljoin/oracle.hpp"
#include "coljoin/primitives.hpp"
#include "coljoin/reference.hpp"
#include "coljoin/relation_io.hpp"
#include "coljoin/rng.hpp"
#include "coljoin/sequence.hpp"
#include "coljoin/workloads.hpp"

using namespace coljoin;

namespace {

struct Args {
  std::vector<std::string> v;
  const char* get(const char* name, const char* dflt) const {
    for (size_t i = 0; i + 1 < v.size(); ++i)
      if (v[i] == name) return v[i + 1].c_str();
    return dflt;
  }
  bool has(const char* name) const {
    return std::find(v.begin(), v.end(), std::string(name)) != v.end();
  }
};

uint64_t digest_words(const std::vector<uint64_t>& w) {
  uint64_t h = 0x12345678ull;
  for (size_t i = 0; i < w.size(); ++i) h = mix64(h ^ w[i]) + i;
  return h;
}

std::vector<uint64_t> widen(const Column& c) {
  std::vector<uint64_t> w(c.size());
  for (size_t i = 0; i < c.size(); ++i) w[i] = c.at(i);
  return w;
}

uint64_t digest_col(const Column& c) { return digest_words(widen(c)); }

uint64_t digest_u32(const std::vector<uint32_t>& v) {
  std::vector<uint64_t> w(v.begin(), v.end());
  return digest_words(w);
}

// Canonical-row digest of a join output, equal to
// digest_words(oracle::canonical_rows(rel)) (oracle.cpp:77-88: rows widened to
// u64, sorted lexicographically) but sorted in parallel: T chunk sorts, then
// rounds of pairwise merges.  Identical rows are interchangeable, so any
// correct sort gives the reference's flat vector.  The reference's
// single-threaded index sort takes tens of minutes at 2^28 rows; this is test
// infrastructure for the full-size golden digests (tests/golden/make_golden.py
// --full), not a change to the reference.
template <size_t W>
uint64_t parallel_canonical_digest_w(const Relation& rel) {
  using Row = std::array<uint64_t, W>;
  const size_t n = rel.rows();
  std::vector<Row> rows(n), tmp(n);
  std::vector<const Column*> cols{&rel.key};
  for (const auto& p : rel.payloads) cols.push_back(&p);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i)
    for (size_t c = 0; c < W; ++c) rows[i][c] = cols[c]->at(i);
  const size_t T = static_cast<size_t>(std::max(1, omp_get_max_threads()));
  size_t parts = 1;
  while (parts < T) parts <<= 1;
  std::vector<size_t> b(parts + 1);
  for (size_t p = 0; p <= parts; ++p) b[p] = n * p / parts;
#pragma omp parallel for schedule(dynamic, 1)
  for (size_t p = 0; p < parts; ++p) std::sort(rows.begin() + b[p], rows.begin() + b[p + 1]);
  for (size_t width = 1; width < parts; width <<= 1) {
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t p = 0; p < parts; p += 2 * width) {
      const size_t lo = b[p], mid = b[std::min(p + width, parts)], hi = b[std::min(p + 2 * width, parts)];
      std::merge(rows.begin() + lo, rows.begin() + mid, rows.begin() + mid, rows.begin() + hi,
                 tmp.begin() + lo);
    }
    rows.swap(tmp);
  }
  uint64_t h = 0x12345678ull, i = 0;
  for (const Row& r : rows)
    for (size_t c = 0; c < W; ++c, ++i) h = mix64(h ^ r[c]) + i;
  return h;
}

uint64_t parallel_canonical_digest(const Relation& rel) {
  switch (rel.column_count()) {
    case 1: return parallel_canonical_digest_w<1>(rel);
    case 2: return parallel_canonical_digest_w<2>(rel);
    case 3: return parallel_canonical_digest_w<3>(rel);
    case 4: return parallel_canonical_digest_w<4>(rel);
    case 5: return parallel_canonical_digest_w<5>(rel);
    case 6: return parallel_canonical_digest_w<6>(rel);
    case 7: return parallel_canonical_digest_w<7>(rel);
    case 8: return parallel_canonical_digest_w<8>(rel);
    case 9: return parallel_canonical_digest_w<9>(rel);
    default: return digest_words(oracle::canonical_rows(rel));
  }
}

std::vector<unsigned> parse_widths(const char* s) {
  std::vector<unsigned> out;
  if (!s || !*s) return out;
  std::string str(s);
  size_t pos = 0;
  while (pos <= str.size()) {
    size_t comma = str.find(',', pos);
    if (comma == std::string::npos) comma = str.size();
    out.push_back(static_cast<unsigned>(std::stoul(str.substr(pos, comma - pos))));
    pos = comma + 1;
  }
  return out;
}

ValueKind kind_of(const char* s) {
  return std::strcmp(s, "u64") == 0 ? ValueKind::u64 : ValueKind::u32;
}

Column narrow_u32(const Column& c) {
  std::vector<uint32_t> v(c.size());
  for (size_t i = 0; i < c.size(); ++i) v[i] = static_cast<uint32_t>(c.at(i));
  return Column::of_u32(std::move(v));
}

std::pair<Relation, Relation> make_workload(const Args& a) {
  workloads::WorkloadSpec spec;
  spec.r_rows = std::strtoull(a.get("--r", "1024"), nullptr, 10);
  spec.s_rows = std::strtoull(a.get("--s", "2048"), nullptr, 10);
  spec.r_payloads = static_cast<unsigned>(std::atoi(a.get("--rpay", "1")));
  spec.s_payloads = static_cast<unsigned>(std::atoi(a.get("--spay", "1")));
  spec.key_kind = kind_of(a.get("--key", "u32"));
  spec.payload_kind = kind_of(a.get("--pay", "u32"));
  spec.match_ratio = std::atof(a.get("--match", "1"));
  spec.zipf_factor = std::atof(a.get("--zipf", "0"));
  spec.seed = std::strtoull(a.get("--seed", "42"), nullptr, 10);
  auto widths = parse_widths(a.get("--widths", ""));
  if (!widths.empty()) {
    spec.payload_kind = ValueKind::u64;
    spec.r_payloads = spec.s_payloads = static_cast<unsigned>(widths.size());
  }
  auto rs = workloads::gen_pk_fk(spec);
  for (size_t c = 0; c < widths.size(); ++c) {
    if (widths[c] == 4) {
      rs.first.payloads[c] = narrow_u32(rs.first.payloads[c]);
      rs.second.payloads[c] = narrow_u32(rs.second.payloads[c]);
    }
  }
  return rs;
}

void dump_col(const std::string& path, const Column& c) {
  std::ofstream f(path, std::ios::binary);
  if (c.kind() == ValueKind::u32)
    f.write(reinterpret_cast<const char*>(c.u32().data()), c.byte_size());
  else
    f.write(reinterpret_cast<const char*>(c.u64().data()), c.byte_size());
}

void dump_rel(const std::string& dir, const std::string& tag, const Relation& r) {
  dump_col(dir + "/" + tag + "_key.bin", r.key);
  for (size_t c = 0; c < r.payloads.size(); ++c)
    dump_col(dir + "/" + tag + "_p" + std::to_string(c) + ".bin", r.payloads[c]);
}

int join_one(const Args& a, const Relation& r, const Relation& s, JoinAlgo algo, JoinPattern pattern);

// --all-variants: generate once, then run PHJ/SMJ x GFTR/GFUR (one JSON line each)
int cmd_join(const Args& a) {
  auto [r, s] = make_workload(a);
  auto algo = std::strcmp(a.get("--algo", "phj"), "smj") == 0 ? JoinAlgo::SMJ : JoinAlgo::PHJ;
  auto pattern = std::strcmp(a.get("--pattern", "gftr"), "gfur") == 0 ? JoinPattern::GFUR
                                                                     : JoinPattern::GFTR;
  if (!a.has("--all-variants")) return join_one(a, r, s, algo, pattern);
  for (JoinAlgo al : {JoinAlgo::PHJ, JoinAlgo::SMJ})
    for (JoinPattern pa : {JoinPattern::GFTR, JoinPattern::GFUR}) {
      join_one(a, r, s, al, pa);
      std::fflush(stdout);
    }
  return 0;
}

int join_one(const Args& a, const Relation& r, const Relation& s, JoinAlgo algo, JoinPattern pattern) {
  JoinTask task;
  task.algorithm = algo;
  task.pattern = pattern;
  // --swap: build on S (duplicate keys, key_unique=false), probe with R
  const bool swap = a.has("--swap");
  task.build = swap ? &s : &r;
  task.probe = swap ? &r : &s;
  task.options.worker_count = static_cast<unsigned>(std::atoi(a.get("--threads", "0")));
  task.options.preallocate = a.has("--prealloc");
  task.options.total_radix_bits = std::atoi(a.get("--total-bits", "-1"));
  const int reps = std::max(1, std::atoi(a.get("--reps", "1")));
  const int warmup = std::max(0, std::atoi(a.get("--warmup", "0")));
  std::vector<uint64_t> totals;
  JoinOutput out;
  for (int i = 0; i < warmup; ++i) out = run_join(task);
  for (int i = 0; i < reps; ++i) {
    out = run_join(task);
    totals.push_back(out.report.total_ns());
  }
  uint64_t sum = 0;
  for (uint64_t t : totals) sum += t;
  const uint64_t mean = sum / totals.size();
  std::sort(totals.begin(), totals.end());
  const uint64_t med = totals[totals.size() / 2];
  const double tput = static_cast<double>(r.rows() + s.rows()) / (med * 1e-9);
  std::string dig = "null", odig = "null";
  if (a.has("--digest") || a.has("--pdigest")) {
    char buf[32];
    // --pdigest: the same digest through the parallel canonical sort
    // (--digest --pdigest checks that both agree)
    uint64_t d = 0;
    if (a.has("--digest")) d = digest_words(oracle::canonical_rows(out.relation));
    if (a.has("--pdigest")) {
      const uint64_t pd = parallel_canonical_digest(out.relation);
      if (a.has("--digest") && pd != d) throw SpecInvalid("parallel canonical digest differs");
      d = pd;
    }
    std::snprintf(buf, sizeof(buf), "\"%016llx\"", (unsigned long long)d);
    dig = buf;
    // emission-order digest over the flat columns (key, then payloads)
    std::vector<uint64_t> flat = widen(out.relation.key);
    for (const auto& p : out.relation.payloads) {
      auto w = widen(p);
      flat.insert(flat.end(), w.begin(), w.end());
    }
    std::snprintf(buf, sizeof(buf), "\"%016llx\"", (unsigned long long)digest_words(flat));
    odig = buf;
  }
  if (const char* dir = a.get("--dump", nullptr)) {
    dump_rel(dir, "R", r);
    dump_rel(dir, "S", s);
    dump_rel(dir, "T", out.relation);
  }
  const unsigned threads = task.options.worker_count ? task.options.worker_count
                                                     : static_cast<unsigned>(omp_get_max_threads());
  std::printf(
      "{\"variant\": \"%s\", \"rows_r\": %zu, \"rows_s\": %zu, \"rows_out\": %zu, "
      "\"threads\": %u, \"reps\": %d, \"total_ns_mean\": %llu, \"total_ns_median\": %llu, \"transform_ns\": %llu, "
      "\"find_ns\": %llu, \"materialize_ns\": %llu, \"tuples_per_s\": %.6e, "
      "\"clusteredness_r\": %.6f, \"clusteredness_s\": %.6f, \"digest\": %s, "
      "\"order_digest\": %s}\n",
      variant_name(task.algorithm, task.pattern), r.rows(), s.rows(), out.relation.rows(),
      threads, reps, (unsigned long long)mean, (unsigned long long)med, (unsigned long long)out.report.transform_ns,
      (unsigned long long)out.report.find_ns, (unsigned long long)out.report.materialize_ns,
      tput, out.stats.clusteredness_r, out.stats.clusteredness_s, dig.c_str(), odig.c_str());
  return 0;
}

int cmd_gen(const Args& a) {
  auto [r, s] = make_workload(a);
  const char* dir = a.get("--dump", nullptr);
  if (dir) {
    dump_rel(dir, "R", r);
    dump_rel(dir, "S", s);
  }
  std::printf("{\"r_key\": \"%016llx\", \"s_key\": \"%016llx\"",
              (unsigned long long)digest_col(r.key), (unsigned long long)digest_col(s.key));
  for (size_t c = 0; c < r.payloads.size(); ++c)
    std::printf(", \"r_p%zu\": \"%016llx\"", c, (unsigned long long)digest_col(r.payloads[c]));
  for (size_t c = 0; c < s.payloads.size(); ++c)
    std::printf(", \"s_p%zu\": \"%016llx\"", c, (unsigned long long)digest_col(s.payloads[c]));
  std::printf("}\n");
  return 0;
}

// Star schema (workloads.cpp:135-160) and the chained joins of
// run_join_sequence (sequence.cpp:9-67).  The reference's function returns the
// steps only; the loop is restated here with the reference's own run_join and
// gather_copy so that the final join's output can be digested, and the
// reference's run_join_sequence is timed as is (--reps).
int cmd_star(const Args& a) {
  workloads::StarSchemaSpec spec;
  spec.fact_rows = std::strtoull(a.get("--fact", "4096"), nullptr, 10);
  spec.dims = static_cast<unsigned>(std::atoi(a.get("--dims", "3")));
  spec.dim_rows = std::strtoull(a.get("--dim-rows", "1024"), nullptr, 10);
  spec.seed = std::strtoull(a.get("--seed", "42"), nullptr, 10);
  auto star = workloads::gen_star(spec);
  JoinTask proto;
  proto.algorithm = std::strcmp(a.get("--algo", "phj"), "smj") == 0 ? JoinAlgo::SMJ : JoinAlgo::PHJ;
  proto.pattern = std::strcmp(a.get("--pattern", "gftr"), "gfur") == 0 ? JoinPattern::GFUR
                                                                       : JoinPattern::GFTR;
  proto.options.worker_count = static_cast<unsigned>(std::atoi(a.get("--threads", "0")));
  proto.options.preallocate = a.has("--prealloc");
  const unsigned workers = proto.options.worker_count ? proto.options.worker_count
                                                      : static_cast<unsigned>(omp_get_max_threads());
  std::printf("{\"fact_ids\": \"%016llx\"", (unsigned long long)digest_col(star.fact.key));
  for (size_t d = 0; d < star.dims.size(); ++d)
    std::printf(", \"fk%zu\": \"%016llx\", \"dim%zu_key\": \"%016llx\", \"dim%zu_p0\": \"%016llx\"", d,
                (unsigned long long)digest_col(star.fact.payloads[d]), d,
                (unsigned long long)digest_col(star.dims[d].key), d,
                (unsigned long long)digest_col(star.dims[d].payloads[0]));
  // the chain, as sequence.cpp:23-66
  Relation probe;
  probe.key = star.fact.payloads[0];
  probe.payloads.push_back(star.fact.key);
  std::printf(", \"steps\": [");
  for (size_t i = 0; i < star.dims.size(); ++i) {
    JoinTask task = proto;
    task.build = &star.dims[i];
    task.probe = &probe;
    JoinOutput out = run_join(task);
    std::vector<uint64_t> flat = widen(out.relation.key);
    for (const auto& c : out.relation.payloads) {
      auto w = widen(c);
      flat.insert(flat.end(), w.begin(), w.end());
    }
    std::printf("%s{\"rows\": %zu, \"columns\": %zu, \"digest\": \"%016llx\", \"order_digest\": \"%016llx\"}",
                i ? ", " : "", out.relation.rows(), out.relation.column_count(),
                (unsigned long long)digest_words(oracle::canonical_rows(out.relation)),
                (unsigned long long)digest_words(flat));
    if (i + 1 < star.dims.size()) {
      const size_t dim_pay = star.dims[i].payloads.size();
      Column next_fk =
          primitives::gather_copy(star.fact.payloads[i + 1], out.relation.payloads[dim_pay].u32(), workers);
      probe = Relation{};
      probe.key = std::move(next_fk);
      for (size_t c = dim_pay; c < out.relation.payloads.size(); ++c)
        probe.payloads.push_back(std::move(out.relation.payloads[c]));
      for (size_t c = 0; c < dim_pay; ++c) probe.payloads.push_back(std::move(out.relation.payloads[c]));
    }
  }
  std::printf("]");
  const int reps = std::atoi(a.get("--reps", "0"));
  if (reps > 0) {
    std::vector<uint64_t> t;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      auto steps = run_join_sequence(star.fact, star.dims, proto.algorithm, proto.pattern,
                                     proto.options);
      t.push_back(static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                            std::chrono::steady_clock::now() - t0)
                                            .count()));
    }
    std::sort(t.begin(), t.end());
    std::printf(", \"sequence_ns_median\": %llu, \"threads\": %u", (unsigned long long)t[t.size() / 2],
                workers);
  }
  std::printf("}\n");
  return 0;
}

// Primitive known-answer digests on seeded inputs (for pinning the C port).
// Inputs: keys_i = CounterRng(seed).at(i) truncated/bounded as noted.
int cmd_prim(const Args& a) {
  const size_t n = std::strtoull(a.get("--n", "100000"), nullptr, 10);
  const uint64_t seed = std::strtoull(a.get("--seed", "1"), nullptr, 10);
  const unsigned workers = 4;
  CounterRng rng(seed);
  std::vector<uint32_t> k32(n), v32(n), dup32(n);
  std::vector<uint64_t> k64(n);
  for (size_t i = 0; i < n; ++i) {
    k32[i] = static_cast<uint32_t>(rng.at(i));
    v32[i] = static_cast<uint32_t>(rng.stream(1).at(i));
    dup32[i] = static_cast<uint32_t>(rng.stream(2).below(i, 97));
    k64[i] = rng.stream(3).at(i) >> (rng.stream(4).below(i, 40));
  }
  Column K32 = Column::of_u32(k32), V32 = Column::of_u32(v32), D32 = Column::of_u32(dup32);
  Column K64 = Column::of_u64(k64);
  auto pr = [](const char* name, uint64_t d, bool last = false) {
    std::printf("\"%s\": \"%016llx\"%s", name, (unsigned long long)d, last ? "" : ", ");
  };
  std::printf("{");
  {
    Column ko, vo;
    auto lay = primitives::radix_partition(K32, V32, ko, vo, 3, 11, workers);
    pr("part32_k", digest_col(ko));
    pr("part32_v", digest_col(vo));
    pr("part32_off", digest_words(lay.offsets));
  }
  {
    Column ko, vo;
    primitives::sort_pairs(K32, V32, ko, vo, workers);
    pr("sort32_k", digest_col(ko));
    pr("sort32_v", digest_col(vo));
    Column dk, dv;
    primitives::sort_pairs(D32, V32, dk, dv, workers);
    pr("sortdup_k", digest_col(dk));
    pr("sortdup_v", digest_col(dv));
  }
  {
    Column ko, vo;
    primitives::sort_pairs(K64, V32, ko, vo, workers);
    pr("sort64_k", digest_col(ko));
    pr("sort64_v", digest_col(vo));
  }
  {
    Column ko, vo;
    auto lay = hashjoin::partition_relation(K32, V32, ko, vo, 16, 8, workers);
    pr("prel32_k", digest_col(ko));
    pr("prel32_v", digest_col(vo));
    pr("prel32_off", digest_words(lay.offsets));
    Column k6, v6;
    auto lay6 = hashjoin::partition_relation(K64, V32, k6, v6, 13, 5, workers);
    pr("prel64_k", digest_col(k6));
    pr("prel64_v", digest_col(v6));
    pr("prel64_off", digest_words(lay6.offsets));
  }
  {
    std::vector<uint32_t> map(n);
    for (size_t i = 0; i < n; ++i) map[i] = static_cast<uint32_t>(rng.stream(5).below(i, n));
    pr("gather32", digest_col(primitives::gather_copy(V32, map, workers)));
    pr("gather64", digest_col(primitives::gather_copy(K64, map, workers)));
  }
  {
    // hash + merge match on a duplicate-heavy self join of dup32 (97 values)
    const size_t m = std::min<size_t>(n, 4000);
    std::vector<uint32_t> rk(dup32.begin(), dup32.begin() + m / 2);
    std::vector<uint32_t> sk(dup32.begin() + m / 2, dup32.begin() + m);
    Column RK = Column::of_u32(rk), SK = Column::of_u32(sk);
    Column rko, sko;
    auto lr = hashjoin::partition_relation_keys(RK, rko, 4, 8, workers);
    auto ls = hashjoin::partition_relation_keys(SK, sko, 4, 8, workers);
    hashjoin::PartitionedRelationView bv{&rko, &lr, nullptr}, pv{&sko, &ls, nullptr};
    auto plan = hashjoin::plan_subpartitions(bv, pv, 16);
    auto hm = hashjoin::hash_find_matches(bv, pv, plan, TupleIdSemantics::Virtual, workers);
    pr("hash_keys", digest_col(hm.keys));
    pr("hash_ids_r", digest_u32(hm.ids_r));
    pr("hash_ids_s", digest_u32(hm.ids_s));
    Column rs, ss;
    primitives::sort_keys(RK, rs, workers);
    primitives::sort_keys(SK, ss, workers);
    auto mm = mergejoin::merge_find_matches(rs, ss, false, 7, workers);
    pr("merge_keys", digest_col(mm.keys));
    pr("merge_ids_r", digest_u32(mm.ids_r));
    pr("merge_ids_s", digest_u32(mm.ids_s), true);
  }
  std::printf("}\n");
  return 0;
}

// Relation manifests and the bench CSV through the reference's own
// relation_io.cpp / bench_io.cpp: the interop checks of tests/test_formats.py.
int cmd_export(const Args& a) {
  auto [r, s] = make_workload(a);
  const std::string dir = a.get("--dir", "");
  if (dir.empty()) throw SpecInvalid("--dir is required");
  workloads::export_relation(r, std::filesystem::path(dir) / "R");
  workloads::export_relation(s, std::filesystem::path(dir) / "S");
  return cmd_gen(a);
}

int cmd_import(const Args& a) {
  const Relation r = workloads::import_relation(a.get("--dir", ""));
  std::printf("{\"name\": \"%s\", \"rows\": %zu, \"key_unique\": %d, \"columns\": [",
              r.name.c_str(), r.rows(), r.key_unique ? 1 : 0);
  auto col = [](const Column& c, bool first) {
    std::printf("%s{\"kind\": \"%s\", \"digest\": \"%016llx\"}", first ? "" : ", ",
                c.kind() == ValueKind::u64 ? "u64" : "u32",
                (unsigned long long)digest_col(c));
  };
  col(r.key, true);
  for (const auto& p : r.payloads) col(p, false);
  std::printf("]}\n");
  return 0;
}

int cmd_report(const Args& a) {
  std::ifstream in(a.get("--in", ""));
  if (!in) throw SchemaError("cannot open the CSV");
  std::cout << benchio::render_report(benchio::read_csv(in));
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: refjoin join|gen|prim [options]\n");
    return 2;
  }
  Args a;
  for (int i = 2; i < argc; ++i) a.v.emplace_back(argv[i]);
  try {
    if (std::strcmp(argv[1], "join") == 0) return cmd_join(a);
    if (std::strcmp(argv[1], "gen") == 0) return cmd_gen(a);
    if (std::strcmp(argv[1], "prim") == 0) return cmd_prim(a);
    if (std::strcmp(argv[1], "star") == 0) return cmd_star(a);
    if (std::strcmp(argv[1], "export") == 0) return cmd_export(a);
    if (std::strcmp(argv[1], "import") == 0) return cmd_import(a);
    if (std::strcmp(argv[1], "report") == 0) return cmd_report(a);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "refjoin: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown subcommand %s\n", argv[1]);
  return 2;
}
