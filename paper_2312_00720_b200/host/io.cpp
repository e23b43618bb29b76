// Host-side data formats either side of the join path:
//  - relation manifests (coljoin/relation_io.hpp; reference format:
//    src/relation_io.cpp:48-103), and
//  - the bench CSV wire format + markdown report (coljoin/bench_io.hpp;
//    reference: src/bench_io.cpp:16-184).
// Both are byte-compatible with the reference so its tools and ours read each
// other's files.  The CSV schema is one table of field descriptors: the
// header, the writer and the parser all walk it, so the column order is
// stated once.
#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <fstream>
#include <functional>
#include <istream>
#include <map>
#include <ostream>
#include <sstream>

#include "coljoin/bench_io.hpp"
#include "coljoin/relation_io.hpp"

namespace coljoin {

// ------------------------------------------------------------ manifests ---
namespace workloads {
namespace {

const char* kind_token(ValueKind k) { return k == ValueKind::u64 ? "u64" : "u32"; }

ValueKind kind_from_token(const std::string& t) {
  if (t == "u32") return ValueKind::u32;
  if (t == "u64") return ValueKind::u64;
  throw SchemaError("unknown column kind in manifest: " + t);
}

void dump_column(const Column& c, const std::filesystem::path& file) {
  std::ofstream f(file, std::ios::binary | std::ios::trunc);
  if (!f) throw SchemaError("cannot write " + file.string());
  f.write(static_cast<const char*>(c.raw()), static_cast<std::streamsize>(c.byte_size()));
  if (!f) throw SchemaError("short write to " + file.string());
}

Column load_column(ValueKind kind, uint64_t rows, const std::filesystem::path& file) {
  std::ifstream f(file, std::ios::binary);
  if (!f) throw SchemaError("cannot read " + file.string());
  Column c(kind, rows);
  const auto want = static_cast<std::streamsize>(c.byte_size());
  f.read(static_cast<char*>(c.raw()), want);
  if (f.gcount() != want)
    throw SchemaError("column file shorter than the manifest row count: " + file.string());
  return c;
}

}  // namespace

void export_relation(const Relation& rel, const std::filesystem::path& dir) {
  std::filesystem::create_directories(dir);
  std::ostringstream mf;
  mf << "name " << (rel.name.empty() ? std::string("relation") : rel.name) << "\n"
     << "rows " << rel.rows() << "\n"
     << "key_unique " << (rel.key_unique ? 1 : 0) << "\n";
  auto column = [&](const Column& c, const std::string& label, const std::string& file) {
    mf << "column " << label << " " << kind_token(c.kind()) << " " << file << "\n";
    dump_column(c, dir / file);
  };
  column(rel.key, "key", "key.bin");
  for (size_t i = 0; i < rel.payloads.size(); ++i)
    column(rel.payloads[i], "payload" + std::to_string(i), "payload" + std::to_string(i) + ".bin");
  std::ofstream out(dir / "manifest.txt", std::ios::trunc);
  if (!out) throw SchemaError("cannot write manifest in " + dir.string());
  out << mf.str();
}

Relation import_relation(const std::filesystem::path& dir) {
  std::ifstream mf(dir / "manifest.txt");
  if (!mf) throw SchemaError("no manifest.txt in " + dir.string());
  Relation rel;
  uint64_t rows = 0;
  bool keyed = false;
  for (std::string line; std::getline(mf, line);) {
    if (line.empty() || line.front() == '#') continue;
    std::istringstream in(line);
    std::string field;
    in >> field;
    if (field == "name") {
      in >> rel.name;
    } else if (field == "rows") {
      in >> rows;
    } else if (field == "key_unique") {
      int flag = 0;
      in >> flag;
      rel.key_unique = flag != 0;
    } else if (field == "column") {
      std::string label, kind, file;
      in >> label >> kind >> file;
      if (label.empty() || kind.empty() || file.empty())
        throw SchemaError("malformed column line: " + line);
      Column c = load_column(kind_from_token(kind), rows, dir / file);
      if (label == "key") {
        rel.key = std::move(c);
        keyed = true;
      } else {
        rel.payloads.push_back(std::move(c));
      }
    } else {
      throw SchemaError("unknown manifest field: " + field);
    }
  }
  if (!keyed) throw SchemaError("manifest lists no key column");
  return rel;
}

}  // namespace workloads

// ------------------------------------------------------------ bench CSV ---
namespace benchio {
namespace {

std::string g17(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

uint64_t parse_uint(const std::string& s) {
  try {
    size_t used = 0;
    const uint64_t v = std::stoull(s, &used);
    (void)used;
    return v;
  } catch (const std::exception&) {
    throw SchemaError("expected an integer CSV field, got: " + s);
  }
}

double parse_real(const std::string& s) {
  try {
    return std::stod(s);
  } catch (const std::exception&) {
    throw SchemaError("expected a numeric CSV field, got: " + s);
  }
}

struct Field {
  const char* name;
  std::function<std::string(const BenchRow&)> put;
  std::function<void(BenchRow&, const std::string&)> get;
};

template <class T>
Field text(const char* n, T BenchRow::*m) {
  return {n, [m](const BenchRow& r) { return r.*m; },
          [m](BenchRow& r, const std::string& s) { r.*m = s; }};
}
template <class T>
Field uint_field(const char* n, T BenchRow::*m) {
  return {n, [m](const BenchRow& r) { return std::to_string(r.*m); },
          [m](BenchRow& r, const std::string& s) { r.*m = static_cast<T>(parse_uint(s)); }};
}
Field real(const char* n, double BenchRow::*m) {
  return {n, [m](const BenchRow& r) { return g17(r.*m); },
          [m](BenchRow& r, const std::string& s) { r.*m = parse_real(s); }};
}

// the wire contract, in order (bench_io.hpp)
const std::vector<Field>& schema() {
  static const std::vector<Field> f = {
      text("experiment", &BenchRow::experiment),
      text("algo", &BenchRow::algo),
      text("pattern", &BenchRow::pattern),
      uint_field("r_rows", &BenchRow::r_rows),
      uint_field("s_rows", &BenchRow::s_rows),
      uint_field("r_payloads", &BenchRow::r_payloads),
      uint_field("s_payloads", &BenchRow::s_payloads),
      uint_field("key_bytes", &BenchRow::key_bytes),
      uint_field("payload_bytes", &BenchRow::payload_bytes),
      real("match_ratio", &BenchRow::match_ratio),
      real("zipf", &BenchRow::zipf),
      uint_field("workers", &BenchRow::workers),
      uint_field("seed", &BenchRow::seed),
      uint_field("rep", &BenchRow::rep),
      uint_field("transform_ns", &BenchRow::transform_ns),
      uint_field("find_ns", &BenchRow::find_ns),
      uint_field("materialize_ns", &BenchRow::materialize_ns),
      uint_field("total_ns", &BenchRow::total_ns),
      real("throughput_tps", &BenchRow::throughput_tps),
      uint_field("peak_transform_b", &BenchRow::peak_transform_b),
      uint_field("peak_find_b", &BenchRow::peak_find_b),
      uint_field("peak_materialize_b", &BenchRow::peak_materialize_b),
      real("clusteredness_s", &BenchRow::clusteredness_s),
      real("clusteredness_r", &BenchRow::clusteredness_r),
  };
  return f;
}

std::vector<std::string> cells(const std::string& line) {
  std::vector<std::string> out(1);
  for (char ch : line) {
    if (ch == ',') out.emplace_back();
    else out.back().push_back(ch);
  }
  return out;
}

// a repetition group: every input field but rep and the measurements
std::string group_of(const BenchRow& r) {
  std::ostringstream k;
  k << r.experiment << '|' << r.algo << '|' << r.pattern << '|' << r.r_rows << '|' << r.s_rows
    << '|' << r.r_payloads << '|' << r.s_payloads << '|' << r.key_bytes << '|'
    << r.payload_bytes << '|' << r.match_ratio << '|' << r.zipf << '|' << r.workers << '|'
    << r.seed;
  return k.str();
}

}  // namespace

std::string csv_header() {
  std::string h;
  for (const auto& f : schema()) {
    if (!h.empty()) h += ',';
    h += f.name;
  }
  return h;
}

void write_csv_row(std::ostream& out, const BenchRow& row) {
  const auto& s = schema();
  for (size_t i = 0; i < s.size(); ++i) out << (i ? "," : "") << s[i].put(row);
  out << '\n';
}

std::vector<BenchRow> read_csv(std::istream& in) {
  const auto& s = schema();
  const std::string header = csv_header();
  std::vector<BenchRow> rows;
  bool header_seen = false;
  for (std::string line; std::getline(in, line);) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    if (!header_seen) {
      if (line != header) throw SchemaError("CSV header does not match the schema");
      header_seen = true;
      continue;
    }
    const auto c = cells(line);
    if (c.size() != s.size())
      throw SchemaError("CSV row has " + std::to_string(c.size()) + " fields, expected " +
                        std::to_string(s.size()));
    BenchRow r;
    for (size_t i = 0; i < s.size(); ++i) s[i].get(r, c[i]);
    rows.push_back(std::move(r));
  }
  return rows;
}

void finalize_throughput(BenchRow& row) {
  row.throughput_tps = row.total_ns == 0
                           ? 0.0
                           : static_cast<double>(row.r_rows + row.s_rows) /
                                 (static_cast<double>(row.total_ns) * 1e-9);
}

std::string render_report(const std::vector<BenchRow>& rows) {
  // groups in first-seen order
  std::vector<std::string> order;
  std::map<std::string, std::vector<const BenchRow*>> groups;
  for (const auto& r : rows) {
    auto& g = groups[group_of(r)];
    if (g.empty()) order.push_back(group_of(r));
    g.push_back(&r);
  }
  std::ostringstream md;
  const std::string* experiment = nullptr;
  for (const auto& key : order) {
    auto g = groups[key];
    std::sort(g.begin(), g.end(),
              [](const BenchRow* a, const BenchRow* b) { return a->total_ns < b->total_ns; });
    const BenchRow& m = *g[g.size() / 2];
    if (!experiment || *experiment != m.experiment) {
      experiment = &m.experiment;
      md << "## " << m.experiment << "\n\n"
         << "| algo | pattern | r_rows | s_rows | payloads | match | zipf | workers "
            "| total_ms | transform% | find% | materialize% | tuples/s | reps |\n"
         << "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|\n";
    }
    const double tot = static_cast<double>(m.total_ns);
    auto share = [tot](uint64_t part) { return tot == 0.0 ? 0.0 : 100.0 * part / tot; };
    char line[320];
    std::snprintf(line, sizeof line,
                  "| %s | %s | %" PRIu64 " | %" PRIu64 " | %u+%u | %.2f | %.2f | %u | %.3f | "
                  "%.1f | %.1f | %.1f | %.3g | %zu |\n",
                  m.algo.c_str(), m.pattern.c_str(), m.r_rows, m.s_rows, m.r_payloads,
                  m.s_payloads, m.match_ratio, m.zipf, m.workers, tot * 1e-6,
                  share(m.transform_ns), share(m.find_ns), share(m.materialize_ns),
                  m.throughput_tps, g.size());
    md << line;
  }
  return md.str();
}

}  // namespace benchio
}  // namespace coljoin
