// cj_bench — the B200 counterpart of the reference's bench harness
// (reference: tools/bench_main.cpp:140-467, the `join`, `gather`, `sequence`,
// `report`, `gen` subcommands), writing the reference's CSV wire format
// (coljoin/bench_io.hpp) so rows measured here drop into its report tooling.
//
//   cj_bench join     [common] [--in-r DIR --in-s DIR] [--warmup W] [--stats]
//   cj_bench gather   [common] --items N --mode clustered|unclustered
//   cj_bench sequence [common] --joins N --fact-rows F --dim-rows D
//   cj_bench report   CSV|- [--out FILE]
//   cj_bench gen      [common] --shape pkfk|star --out-dir DIR [--star-joins N]
//   cj_bench manifest DIR           (rows, kinds and column digests of a manifest)
//   common: --r-rows --s-rows --payloads --match --zipf --key-bytes --payload-bytes
//           --workers --seed --reps --radix-bits --sub-limit --algo phj|smj|nphj
//           --pattern gftr|gfur --out CSV --device D
//
// Measurements follow the paper's scope: inputs resident in
// HBM (generated there bit-identically to workloads::gen_pk_fk, or imported
// from manifests and uploaded once), phase times from the device-timed
// PhaseReport, outputs left in HBM.  `workers` is reported as given (0 = the
// device's default, as the reference's hw default); the peak_*_b columns are
// the device bytes the call held at its high-water mark in each phase.
// Exit codes as the reference's CLI: 1 on a coljoin error, 2 on usage.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "cj_api.h"
#include "coljoin/bench_io.hpp"
#include "coljoin/errors.hpp"
#include "coljoin/primitives.hpp"
#include "coljoin/relation_io.hpp"
#include "coljoin/rng.hpp"

using namespace coljoin;
namespace bio = coljoin::benchio;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Opts {
  std::map<std::string, std::string> kv;
  std::vector<std::string> pos;
  std::vector<std::string> flags;
  std::string get(const std::string& k, const std::string& d) const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  uint64_t u(const std::string& k, uint64_t d) const {
    auto it = kv.find(k);
    if (it == kv.end()) return d;
    try {
      return std::stoull(it->second);
    } catch (const std::exception&) {
      throw UsageError(k + " expects an integer");
    }
  }
  double f(const std::string& k, double d) const {
    auto it = kv.find(k);
    if (it == kv.end()) return d;
    try {
      return std::stod(it->second);
    } catch (const std::exception&) {
      throw UsageError(k + " expects a number");
    }
  }
  bool flag(const std::string& k) const {
    for (const auto& x : flags)
      if (x == k) return true;
    return false;
  }
};

const char* kFlags[] = {"--stats", "--prealloc"};

Opts parse(int argc, char** argv) {
  Opts o;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--", 0) != 0) {
      o.pos.push_back(a);
      continue;
    }
    bool is_flag = false;
    for (const char* f : kFlags) is_flag |= a == f;
    if (is_flag) {
      o.flags.push_back(a);
    } else {
      if (i + 1 >= argc) throw UsageError(a + " needs a value");
      o.kv[a] = argv[++i];
    }
  }
  return o;
}

// ---- device plumbing ------------------------------------------------------
struct Ctx {
  cj_ctx* c = nullptr;
  explicit Ctx(int dev) { check(cj_ctx_create(dev, nullptr, &c), "context"); }
  ~Ctx() {
    if (c) cj_ctx_destroy(c);
  }
  void check(int st, const char* what) const;
};

[[noreturn]] void raise(int st, const std::string& msg) {
  switch (st) {
    case CJ_ERR_SPEC_INVALID: throw SpecInvalid(msg);
    case CJ_ERR_SCHEMA: throw SchemaError(msg);
    case CJ_ERR_KIND: throw KindError(msg);
    default: throw Error(msg + " (status " + std::to_string(st) + ")");
  }
}

void Ctx::check(int st, const char* what) const {
  if (st != CJ_OK) raise(st, std::string(what) + ": " + (c ? cj_last_error(c) : "no context"));
}

struct DevBuf {
  const Ctx* ctx = nullptr;
  void* p = nullptr;
  DevBuf() = default;
  DevBuf(const Ctx& c, uint64_t bytes) : ctx(&c) { c.check(cj_alloc(c.c, bytes + 64, &p), "alloc"); }
  DevBuf(DevBuf&& o) noexcept : ctx(o.ctx), p(o.p) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(ctx, o.ctx);
    std::swap(p, o.p);
    return *this;
  }
  ~DevBuf() {
    if (p) cj_free(ctx->c, p);
  }
};

// A device-resident relation (columns owned by DevBufs).
struct DevRel {
  std::string name;
  bool key_unique = false;
  uint64_t rows = 0;
  uint32_t key_bytes = 4;
  DevBuf key;
  std::vector<DevBuf> pays;
  std::vector<uint32_t> pay_bytes;

  cj_relation view() const {
    cj_relation r{};
    r.key = key.p;
    r.key_bytes = key_bytes;
    r.rows = rows;
    r.npay = static_cast<uint32_t>(pays.size());
    for (size_t c = 0; c < pays.size(); ++c) {
      r.pay[c] = pays[c].p;
      r.pay_bytes[c] = pay_bytes[c];
    }
    r.key_unique = key_unique ? 1 : 0;
    return r;
  }
  Relation download(const Ctx& c) const {
    auto col = [&](const DevBuf& b, uint32_t w) {
      Column out(w == 8 ? ValueKind::u64 : ValueKind::u32, rows);
      if (rows) c.check(cj_copy(c.c, out.raw(), b.p, out.byte_size(), 2), "download");
      return out;
    };
    Relation r;
    r.name = name;
    r.key_unique = key_unique;
    r.key = col(key, key_bytes);
    for (size_t i = 0; i < pays.size(); ++i) r.payloads.push_back(col(pays[i], pay_bytes[i]));
    return r;
  }
};

DevRel upload(const Ctx& c, const Relation& h) {
  DevRel d;
  d.name = h.name;
  d.key_unique = h.key_unique;
  d.rows = h.rows();
  d.key_bytes = static_cast<uint32_t>(value_bytes(h.key.kind()));
  auto put = [&](const Column& col) {
    DevBuf b(c, col.byte_size());
    if (col.byte_size()) c.check(cj_copy(c.c, b.p, col.raw(), col.byte_size(), 1), "upload");
    return b;
  };
  d.key = put(h.key);
  for (const auto& p : h.payloads) {
    d.pays.push_back(put(p));
    d.pay_bytes.push_back(static_cast<uint32_t>(value_bytes(p.kind())));
  }
  return d;
}

uint32_t width(const Opts& o, const char* k) {
  const uint64_t w = o.u(k, 4);
  if (w != 4 && w != 8) throw SpecInvalid("value width must be 4 or 8 bytes");
  return static_cast<uint32_t>(w);
}

std::pair<DevRel, DevRel> gen_pk_fk(const Ctx& c, const Opts& o) {
  const uint64_t nr = o.u("--r-rows", 1 << 20), ns = o.u("--s-rows", 1 << 21);
  const uint32_t np = static_cast<uint32_t>(o.u("--payloads", 1));
  const uint32_t kb = width(o, "--key-bytes"), pb = width(o, "--payload-bytes");
  DevRel r, s;
  r.name = "R";
  s.name = "S";
  r.key_unique = true;
  r.rows = nr;
  s.rows = ns;
  r.key_bytes = s.key_bytes = kb;
  r.key = DevBuf(c, nr * kb);
  s.key = DevBuf(c, ns * kb);
  std::vector<void*> rp, sp;
  for (uint32_t i = 0; i < np; ++i) {
    r.pays.emplace_back(c, nr * pb);
    s.pays.emplace_back(c, ns * pb);
    r.pay_bytes.push_back(pb);
    s.pay_bytes.push_back(pb);
    rp.push_back(r.pays.back().p);
    sp.push_back(s.pays.back().p);
  }
  c.check(cj_gen_pk_fk(c.c, nr, ns, np, np, kb, pb, o.f("--match", 1.0), o.f("--zipf", 0.0),
                       o.u("--seed", 42), r.key.p, rp.data(), s.key.p, sp.data()),
          "gen_pk_fk");
  return {std::move(r), std::move(s)};
}

cj_join_options join_options(const Opts& o) {
  cj_join_options opt;
  cj_default_options(&opt);
  const std::string a = o.get("--algo", "phj"), p = o.get("--pattern", "gftr");
  if (a == "phj") opt.algo = CJ_PHJ;
  else if (a == "smj") opt.algo = CJ_SMJ;
  else if (a == "nphj") opt.algo = CJ_NPHJ;
  else throw SpecInvalid("--algo must be smj, phj or nphj");
  if (p == "gftr") opt.pattern = CJ_GFTR;
  else if (p == "gfur") opt.pattern = CJ_GFUR;
  else throw SpecInvalid("--pattern must be gfur or gftr");
  opt.total_radix_bits = static_cast<int>(std::stoll(o.get("--radix-bits", "-1")));
  opt.sub_partition_limit = static_cast<uint32_t>(o.u("--sub-limit", 4096));
  if (o.flag("--stats")) opt.want_ids = opt.want_stats = 1;
  return opt;
}

class Sink {
 public:
  explicit Sink(const std::string& path) {
    if (!path.empty()) {
      file_.open(path);
      if (!file_) throw SpecInvalid("cannot open output file " + path);
    }
    out() << bio::csv_header() << "\n";
  }
  std::ostream& out() { return file_.is_open() ? file_ : std::cout; }
  void add(const bio::BenchRow& r) {
    bio::write_csv_row(out(), r);
    out().flush();
  }

 private:
  std::ofstream file_;
};

bio::BenchRow row_for(const Opts& o, const std::string& experiment) {
  bio::BenchRow r;
  r.experiment = experiment;
  r.algo = o.get("--algo", "phj");
  r.pattern = o.get("--pattern", "gftr");
  r.r_rows = o.u("--r-rows", 1 << 20);
  r.s_rows = o.u("--s-rows", 1 << 21);
  r.r_payloads = r.s_payloads = static_cast<unsigned>(o.u("--payloads", 1));
  r.key_bytes = width(o, "--key-bytes");
  r.payload_bytes = width(o, "--payload-bytes");
  r.match_ratio = o.f("--match", 1.0);
  r.zipf = o.f("--zipf", 0.0);
  r.workers = static_cast<unsigned>(o.u("--workers", 0));
  r.seed = o.u("--seed", 42);
  return r;
}

// ---- subcommands ------------------------------------------------------------
int cmd_join(const Opts& o) {
  Ctx c(static_cast<int>(o.u("--device", 0)));
  DevRel r, s;
  const std::string in_r = o.get("--in-r", ""), in_s = o.get("--in-s", "");
  if (!in_r.empty() || !in_s.empty()) {
    if (in_r.empty() || in_s.empty()) throw SpecInvalid("--in-r and --in-s must both be given");
    r = upload(c, workloads::import_relation(in_r));
    s = upload(c, workloads::import_relation(in_s));
  } else {
    std::tie(r, s) = gen_pk_fk(c, o);
  }
  const cj_join_options opt = join_options(o);
  const cj_relation rv = r.view(), sv = s.view();
  Sink sink(o.get("--out", ""));
  const uint64_t reps = o.u("--reps", 7), warm = o.u("--warmup", 1);
  for (uint64_t i = 0; i < warm + reps; ++i) {
    cj_join_result res{};
    c.check(cj_run_join(c.c, &rv, &sv, &opt, &res), "run_join");
    if (i >= warm) {
      auto row = row_for(o, "join");
      row.r_rows = r.rows;
      row.s_rows = s.rows;
      row.r_payloads = static_cast<unsigned>(r.pays.size());
      row.s_payloads = static_cast<unsigned>(s.pays.size());
      row.rep = static_cast<unsigned>(i - warm);
      row.transform_ns = res.transform_ns;
      row.find_ns = res.find_ns;
      row.materialize_ns = res.materialize_ns;
      row.total_ns = res.transform_ns + res.find_ns + res.materialize_ns;
      row.peak_transform_b = res.peak_transform_b;
      row.peak_find_b = res.peak_find_b;
      row.peak_materialize_b = res.peak_materialize_b;
      if (opt.want_stats) {
        row.clusteredness_r = res.clusteredness_r;
        row.clusteredness_s = res.clusteredness_s;
      }
      bio::finalize_throughput(row);
      sink.add(row);
    }
    c.check(cj_result_free(c.c, &res), "result_free");
  }
  return 0;
}

int cmd_gather(const Opts& o) {
  const std::string mode = o.get("--mode", "unclustered");
  if (mode != "clustered" && mode != "unclustered")
    throw SpecInvalid("--mode must be clustered or unclustered");
  const uint64_t items = o.u("--items", 1 << 24), seed = o.u("--seed", 42);
  const uint32_t w = width(o, "--payload-bytes");
  Ctx c(static_cast<int>(o.u("--device", 0)));
  // input column: the counter stream at seed; map: iota, or its Fisher-Yates
  // shuffle from the stream at seed + 1 (bench_main.cpp:191-207)
  Column in(w == 8 ? ValueKind::u64 : ValueKind::u32, items);
  CounterRng rng(seed);
  for (uint64_t i = 0; i < items; ++i) {
    if (w == 8) in.u64()[i] = rng.at(i);
    else in.u32()[i] = static_cast<uint32_t>(rng.at(i));
  }
  std::vector<uint32_t> map(items);
  std::iota(map.begin(), map.end(), 0u);
  if (mode == "unclustered") {
    CounterRng mr(seed + 1);
    for (uint64_t i = items; i > 1; --i) std::swap(map[i - 1], map[mr.below(i, i)]);
  }
  DevBuf din(c, items * w), dmap(c, items * 4), dout(c, items * w);
  c.check(cj_copy(c.c, din.p, in.raw(), items * w, 1), "upload");
  c.check(cj_copy(c.c, dmap.p, map.data(), items * 4, 1), "upload");
  const double clus = primitives::gather_clusteredness(map);
  Sink sink(o.get("--out", ""));
  const uint64_t reps = o.u("--reps", 7);
  const void* ins[1] = {din.p};
  void* outs[1] = {dout.p};
  for (uint64_t rep = 0; rep < reps + 1; ++rep) {
    c.check(cj_mark(c.c, 0), "mark");
    c.check(cj_gather(c.c, ins, items, static_cast<const uint32_t*>(dmap.p), items, outs, &w, 1),
            "gather");
    c.check(cj_mark(c.c, 1), "mark");
    c.check(cj_sync(c.c), "sync");
    float ms = 0;
    c.check(cj_elapsed_ms(c.c, 0, 1, &ms), "elapsed");
    if (rep == 0) continue;  // warm-up
    auto row = row_for(o, "gather-" + mode);
    row.algo = row.pattern = "-";
    row.r_rows = items;
    row.s_rows = 0;
    row.r_payloads = row.s_payloads = 0;
    row.rep = static_cast<unsigned>(rep - 1);
    row.materialize_ns = static_cast<uint64_t>(ms * 1e6);
    row.total_ns = row.materialize_ns;
    row.clusteredness_r = row.clusteredness_s = clus;
    bio::finalize_throughput(row);
    sink.add(row);
  }
  return 0;
}

int cmd_sequence(const Opts& o) {
  const uint32_t joins = static_cast<uint32_t>(o.u("--joins", 4));
  const uint64_t nf = o.u("--fact-rows", 1 << 20), nd = o.u("--dim-rows", 1 << 18);
  const uint32_t kb = width(o, "--key-bytes"), pb = width(o, "--payload-bytes");
  if (joins == 0 || joins > CJ_MAX_COLS) throw SpecInvalid("--joins must be in [1, 16]");
  Ctx c(static_cast<int>(o.u("--device", 0)));
  DevBuf ids(c, nf * 4);
  std::vector<DevBuf> fks, dk, dp;
  std::vector<void*> fkp, dkp, dpp;
  for (uint32_t d = 0; d < joins; ++d) {
    fks.emplace_back(c, nf * kb);
    dk.emplace_back(c, nd * kb);
    dp.emplace_back(c, nd * pb);
    fkp.push_back(fks.back().p);
    dkp.push_back(dk.back().p);
    dpp.push_back(dp.back().p);
  }
  c.check(cj_gen_star(c.c, nf, joins, nd, o.u("--seed", 42), kb, pb, ids.p, fkp.data(),
                      dkp.data(), dpp.data()),
          "gen_star");
  cj_relation fact{};
  fact.key = ids.p;
  fact.key_bytes = 4;
  fact.rows = nf;
  fact.key_unique = 1;
  fact.npay = joins;
  for (uint32_t d = 0; d < joins; ++d) {
    fact.pay[d] = fkp[d];
    fact.pay_bytes[d] = kb;
  }
  std::vector<cj_relation> dims(joins);
  for (uint32_t d = 0; d < joins; ++d) {
    dims[d] = cj_relation{};
    dims[d].key = dkp[d];
    dims[d].key_bytes = kb;
    dims[d].rows = nd;
    dims[d].npay = 1;
    dims[d].pay[0] = dpp[d];
    dims[d].pay_bytes[0] = pb;
    dims[d].key_unique = 1;
  }
  const cj_join_options opt = join_options(o);
  Sink sink(o.get("--out", ""));
  std::vector<cj_sequence_step> steps(joins);
  const uint64_t reps = o.u("--reps", 7);
  for (uint64_t rep = 0; rep < reps + 1; ++rep) {
    c.check(cj_run_join_sequence(c.c, &fact, dims.data(), joins, &opt, steps.data(), nullptr),
            "run_join_sequence");
    if (rep == 0) continue;  // warm-up
    for (uint32_t i = 0; i < joins; ++i) {
      auto row = row_for(o, "sequence-" + std::to_string(i + 1));
      row.r_rows = nd;
      row.s_rows = nf;
      row.r_payloads = 1;
      row.s_payloads = i + 1;
      row.rep = static_cast<unsigned>(rep - 1);
      row.transform_ns = steps[i].transform_ns;
      row.find_ns = steps[i].find_ns;
      row.materialize_ns = steps[i].materialize_ns;
      row.total_ns = row.transform_ns + row.find_ns + row.materialize_ns;
      bio::finalize_throughput(row);
      sink.add(row);
    }
  }
  return 0;
}

int cmd_report(const Opts& o) {
  if (o.pos.empty()) throw UsageError("report needs a CSV path or -");
  std::vector<bio::BenchRow> rows;
  if (o.pos[0] == "-") {
    rows = bio::read_csv(std::cin);
  } else {
    std::ifstream in(o.pos[0]);
    if (!in) throw SchemaError("cannot open " + o.pos[0]);
    rows = bio::read_csv(in);
  }
  const std::string md = bio::render_report(rows);
  const std::string out = o.get("--out", "");
  if (out.empty()) std::cout << md;
  else std::ofstream(out) << md;
  return 0;
}

int cmd_gen(const Opts& o) {
  const std::string shape = o.get("--shape", "pkfk"), dir = o.get("--out-dir", "");
  if (dir.empty()) throw SpecInvalid("--out-dir is required");
  Ctx c(static_cast<int>(o.u("--device", 0)));
  const std::filesystem::path root(dir);
  if (shape == "pkfk") {
    auto [r, s] = gen_pk_fk(c, o);
    workloads::export_relation(r.download(c), root / "R");
    workloads::export_relation(s.download(c), root / "S");
  } else if (shape == "star") {
    // workloads::gen_star (workloads.cpp:135-160): --r-rows fact rows,
    // --s-rows rows per dimension, u32 columns
    const uint32_t joins = static_cast<uint32_t>(o.u("--star-joins", 4));
    const uint64_t nf = o.u("--r-rows", 1 << 20), nd = o.u("--s-rows", 1 << 21);
    DevRel fact;
    fact.name = "fact";
    fact.key_unique = true;
    fact.rows = nf;
    fact.key = DevBuf(c, nf * 4);
    std::vector<DevRel> dims(joins);
    std::vector<void*> fkp, dkp, dpp;
    for (uint32_t d = 0; d < joins; ++d) {
      fact.pays.emplace_back(c, nf * 4);
      fact.pay_bytes.push_back(4);
      fkp.push_back(fact.pays.back().p);
      dims[d].name = "dim" + std::to_string(d + 1);  // workloads.cpp:155
      dims[d].key_unique = true;
      dims[d].rows = nd;
      dims[d].key = DevBuf(c, nd * 4);
      dims[d].pays.emplace_back(c, nd * 4);
      dims[d].pay_bytes.push_back(4);
      dkp.push_back(dims[d].key.p);
      dpp.push_back(dims[d].pays.back().p);
    }
    c.check(cj_gen_star(c.c, nf, joins, nd, o.u("--seed", 42), 4, 4, fact.key.p, fkp.data(),
                        dkp.data(), dpp.data()),
            "gen_star");
    workloads::export_relation(fact.download(c), root / "fact");
    for (auto& d : dims) workloads::export_relation(d.download(c), root / d.name);
  } else {
    throw UnknownShape("--shape must be pkfk or star (TPC shapes are out of scope)");
  }
  std::cout << "wrote " << dir << "\n";
  return 0;
}

uint64_t digest(const Column& c) {  // oracle.cpp digest over u64-widened values
  uint64_t h = 0x12345678ull;
  for (size_t i = 0; i < c.size(); ++i) h = mix64(h ^ c.at(i)) + i;
  return h;
}

int cmd_manifest(const Opts& o) {
  if (o.pos.empty()) throw UsageError("manifest needs a directory");
  const Relation r = workloads::import_relation(o.pos[0]);
  std::printf("{\"name\": \"%s\", \"rows\": %zu, \"key_unique\": %d, \"columns\": [",
              r.name.c_str(), r.rows(), r.key_unique ? 1 : 0);
  auto col = [](const Column& c, bool first) {
    std::printf("%s{\"kind\": \"%s\", \"digest\": \"%016llx\"}", first ? "" : ", ",
                c.kind() == ValueKind::u64 ? "u64" : "u32",
                static_cast<unsigned long long>(digest(c)));
  };
  col(r.key, true);
  for (const auto& p : r.payloads) col(p, false);
  std::printf("]}\n");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const char* usage = "usage: cj_bench join|gather|sequence|report|gen|manifest [options]\n";
  if (argc < 2) {
    std::fputs(usage, stderr);
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    const Opts o = parse(argc, argv);
    if (cmd == "join") return cmd_join(o);
    if (cmd == "gather") return cmd_gather(o);
    if (cmd == "sequence") return cmd_sequence(o);
    if (cmd == "report") return cmd_report(o);
    if (cmd == "gen") return cmd_gen(o);
    if (cmd == "manifest") return cmd_manifest(o);
    std::fputs(usage, stderr);
    return 2;
  } catch (const UsageError& e) {
    std::fprintf(stderr, "usage error: %s\n%s", e.what(), usage);
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
