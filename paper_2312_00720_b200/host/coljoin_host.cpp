// libcoljoin_host — the reference's C++ operator API (include/coljoin/*.hpp)
// implemented over the C-ABI of libcoljoin_b200.so (include/cj_api.h).
//
// This file is the drop-in: a caller of the reference's coljoin:: functions
// relinks against libcoljoin_host and gets the same results, computed by the
// sm_100a kernels.  It is plain C++ (no CUDA headers): columns are uploaded
// into library-allocated device buffers, the C-ABI runs the operator, results
// come back into the caller's Columns, and C-ABI status codes are rethrown as
// the reference's exception classes.  Host-side pieces that are bookkeeping,
// not data-parallel work (plan_subpartitions, merge_path_split, the phase
// ledger), run on the host as in the reference.
#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "cj_api.h"
#include "coljoin/hash_match.hpp"
#include "coljoin/join_engine.hpp"
#include "coljoin/sequence.hpp"
#include "coljoin/sharded.hpp"
#include "coljoin/merge_match.hpp"
#include "coljoin/primitives.hpp"

namespace coljoin {
namespace detail {

[[noreturn]] void throw_status(int st, const std::string& what) {
  const std::string msg = what;
  switch (st) {
    case CJ_ERR_LENGTH_MISMATCH: throw LengthMismatch(msg);
    case CJ_ERR_KIND: throw KindError(msg);
    case CJ_ERR_FANOUT_TOO_LARGE: throw FanoutTooLarge(msg);
    case CJ_ERR_INDEX_OUT_OF_BOUNDS: throw IndexOutOfBounds(msg);
    case CJ_ERR_EMPTY_INPUT: throw EmptyInput(msg);
    case CJ_ERR_NOT_SORTED: throw NotSorted(msg);
    case CJ_ERR_DUPLICATE_BUILD_KEYS: throw DuplicateBuildKeys(msg);
    case CJ_ERR_FANOUT_MISMATCH: throw FanoutMismatch(msg);
    case CJ_ERR_CAPACITY_EXCEEDED: throw CapacityExceeded(msg);
    case CJ_ERR_TRANSFORM_MISMATCH: throw TransformMismatch(msg);
    case CJ_ERR_PHASE_ORDER: throw PhaseOrderViolation(msg);
    case CJ_ERR_SPEC_INVALID: throw SpecInvalid(msg);
    case CJ_ERR_UNKNOWN_SHAPE: throw UnknownShape(msg);
    case CJ_ERR_SCHEMA: throw SchemaError(msg);
    case CJ_ERR_UNSUPPORTED: throw Unsupported(msg);
    default: throw DeviceError(msg);
  }
}

// One device context per process (device 0 unless COLJOIN_DEVICE is set);
// calls are serialised on it (the reference allows concurrent run_join calls,
// which stay correct here and share the device).
class Device {
 public:
  static Device& get() {
    static Device d;
    return d;
  }
  cj_ctx* ctx() { return ctx_; }
  std::mutex& mu() { return mu_; }
  void check(int st, const char* what) {
    if (st != CJ_OK) throw_status(st, std::string(what) + ": " + cj_last_error(ctx_));
  }

 private:
  Device() {
    const char* env = std::getenv("COLJOIN_DEVICE");
    const int dev = env ? std::atoi(env) : 0;
    const int st = cj_ctx_create(dev, nullptr, &ctx_);
    if (st != CJ_OK) throw_status(st, "no CUDA device for the B200 join library");
  }
  cj_ctx* ctx_ = nullptr;
  std::mutex mu_;
};

// A library-allocated device buffer.
class Buf {
 public:
  Buf() = default;
  explicit Buf(uint64_t bytes) : bytes_(bytes) {
    auto& d = Device::get();
    d.check(cj_alloc(d.ctx(), bytes ? bytes + 64 : 64, &p_), "device allocation");
  }
  Buf(const void* host, uint64_t bytes) : Buf(bytes) {
    auto& d = Device::get();
    d.check(cj_copy(d.ctx(), p_, host, bytes, 1), "upload");
  }
  Buf(Buf&& o) noexcept : p_(o.p_), bytes_(o.bytes_) { o.p_ = nullptr; }
  Buf& operator=(Buf&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(bytes_, o.bytes_);
    return *this;
  }
  Buf(const Buf&) = delete;
  ~Buf() {
    if (p_) cj_free(Device::get().ctx(), p_);
  }
  void* get() const { return p_; }
  void to_host(void* dst, uint64_t bytes) const {
    auto& d = Device::get();
    d.check(cj_copy(d.ctx(), dst, p_, bytes, 2), "download");
  }

 private:
  void* p_ = nullptr;
  uint64_t bytes_ = 0;
};

Buf upload(const Column& c) { return Buf(c.raw(), c.byte_size()); }
Buf upload_ids(std::span<const uint32_t> ids) { return Buf(ids.data(), ids.size_bytes()); }

void shape_like(const Column& in, Column& out) {
  if (out.kind() != in.kind() || out.size() != in.size()) out = Column(in.kind(), in.size());
}

void download(const Buf& b, Column& c) { b.to_host(c.raw(), c.byte_size()); }

uint32_t kb_of(const Column& c) { return static_cast<uint32_t>(value_bytes(c.kind())); }

// A device-resident match set returned by the C-ABI (released on scope exit).
struct DevMatches {
  uint64_t total = 0;
  void* keys = nullptr;
  uint32_t* ids_r = nullptr;
  uint32_t* ids_s = nullptr;
  ~DevMatches() {
    cj_ctx* ctx = Device::get().ctx();
    if (keys) cj_free(ctx, keys);
    if (ids_r) cj_free(ctx, ids_r);
    if (ids_s) cj_free(ctx, ids_s);
  }
};

// Charges the device scratch an operator held to the caller's ledger (the
// reference accounts its ping-pong buffers the same way, primitives.cpp:236).
struct ScratchCharge {
  Workspace ws;
  explicit ScratchCharge(Workspace w) : ws(w) { cj_scratch_peak(Device::get().ctx(), 1); }
  ~ScratchCharge() {
    const uint64_t peak = cj_scratch_peak(Device::get().ctx(), 1);
    if (ws.ledger && peak) ScopedAlloc(ws.ledger, peak, AllocClass::Scratch).release();
  }
};

void down_raw(void* dst, const void* src, uint64_t bytes) {
  auto& d = Device::get();
  d.check(cj_copy(d.ctx(), dst, src, bytes, 2), "download");
}

}  // namespace detail

using detail::Buf;
using detail::Device;

// ---- primitives ----------------------------------------------------------------

namespace primitives {

std::vector<uint32_t> histogram(const Column& keys, unsigned low_bit, unsigned high_bit,
                                unsigned /*workers*/) {
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  std::vector<uint32_t> out(256, 0);
  Buf k = detail::upload(keys);
  d.check(cj_histogram(d.ctx(), k.get(), keys.size(), detail::kb_of(keys), low_bit, high_bit,
                       out.data()),
          "histogram");
  out.resize(size_t{1} << (high_bit - low_bit));
  return out;
}

std::vector<uint64_t> exclusive_prefix_sum(std::span<const uint32_t> counts) {
  std::vector<uint64_t> out(counts.size() + 1, 0);
  for (size_t i = 0; i < counts.size(); ++i) out[i + 1] = out[i] + counts[i];
  return out;
}

namespace {

PartitionLayout one_pass(const Column& keys, const Column* vals, Column& keys_out,
                         Column* vals_out, unsigned lo, unsigned hi, Workspace ws) {
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  detail::ScratchCharge charge(ws);
  if (vals && vals->size() != keys.size())
    throw LengthMismatch("key and value columns differ in length");
  detail::shape_like(keys, keys_out);
  if (vals) detail::shape_like(*vals, *vals_out);
  const size_t n = keys.size();
  Buf k = detail::upload(keys), ko(keys.byte_size());
  Buf v, vo;
  const void* vin[1] = {nullptr};
  void* vout[1] = {nullptr};
  uint32_t vb[1] = {4};
  if (vals) {
    v = detail::upload(*vals);
    vo = Buf(vals->byte_size());
    vin[0] = v.get();
    vout[0] = vo.get();
    vb[0] = detail::kb_of(*vals);
  }
  std::vector<uint64_t> offsets(257, 0);
  d.check(cj_radix_partition(d.ctx(), k.get(), ko.get(), n, detail::kb_of(keys), lo, hi, vin,
                             vout, vb, vals ? 1 : 0, offsets.data()),
          "radix_partition");
  const uint32_t fanout = 1u << (hi - lo);
  offsets.resize(fanout + 1);
  detail::download(ko, keys_out);
  if (vals) detail::download(vo, *vals_out);
  PartitionLayout lay;
  lay.fanout = fanout;
  lay.low_bit = lo;
  lay.high_bit = hi;
  lay.offsets = std::move(offsets);
  return lay;
}

void lsd(const Column& keys, const Column* vals, Column& keys_out, Column* vals_out,
         std::span<const std::pair<unsigned, unsigned>> plan, bool full_width, Workspace ws) {
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  detail::ScratchCharge charge(ws);
  if (vals && vals->size() != keys.size())
    throw LengthMismatch("key and value columns differ in length");
  detail::shape_like(keys, keys_out);
  if (vals) detail::shape_like(*vals, *vals_out);
  const size_t n = keys.size();
  Buf k = detail::upload(keys), ko(keys.byte_size());
  Buf v, vo;
  const void* vin[1] = {nullptr};
  void* vout[1] = {nullptr};
  uint32_t vb[1] = {4};
  if (vals) {
    v = detail::upload(*vals);
    vo = Buf(vals->byte_size());
    vin[0] = v.get();
    vout[0] = vo.get();
    vb[0] = detail::kb_of(*vals);
  }
  int st;
  if (full_width) {
    st = cj_sort_pairs(d.ctx(), k.get(), ko.get(), n, detail::kb_of(keys), vin, vout, vb,
                       vals ? 1 : 0, 0);
  } else {
    std::vector<uint32_t> lo, hi;
    for (const auto& [a, b] : plan) {
      lo.push_back(a);
      hi.push_back(b);
    }
    st = cj_radix_partition_passes(d.ctx(), k.get(), ko.get(), n, detail::kb_of(keys), lo.data(),
                                   hi.data(), static_cast<uint32_t>(plan.size()), vin, vout, vb,
                                   vals ? 1 : 0, 0);
  }
  d.check(st, full_width ? "sort_pairs" : "radix_partition_passes");
  detail::download(ko, keys_out);
  if (vals) detail::download(vo, *vals_out);
}

}  // namespace

PartitionLayout radix_partition(const Column& keys, const Column& values, Column& keys_out,
                                Column& values_out, unsigned low_bit, unsigned high_bit,
                                unsigned, Workspace ws) {
  return one_pass(keys, &values, keys_out, &values_out, low_bit, high_bit, ws);
}

PartitionLayout radix_partition_keys(const Column& keys, Column& keys_out, unsigned low_bit,
                                     unsigned high_bit, unsigned, Workspace ws) {
  return one_pass(keys, nullptr, keys_out, nullptr, low_bit, high_bit, ws);
}

void radix_partition_passes(const Column& keys, const Column& values, Column& keys_out,
                            Column& values_out, std::span<const std::pair<unsigned, unsigned>> plan,
                            unsigned, Workspace ws) {
  lsd(keys, &values, keys_out, &values_out, plan, false, ws);
}

void radix_partition_passes_keys(const Column& keys, Column& keys_out,
                                 std::span<const std::pair<unsigned, unsigned>> plan, unsigned,
                                 Workspace ws) {
  lsd(keys, nullptr, keys_out, nullptr, plan, false, ws);
}

void sort_pairs(const Column& keys, const Column& values, Column& keys_out, Column& values_out,
                unsigned, Workspace ws) {
  lsd(keys, &values, keys_out, &values_out, {}, true, ws);
}

void sort_keys(const Column& keys, Column& keys_out, unsigned, Workspace ws) {
  lsd(keys, nullptr, keys_out, nullptr, {}, true, ws);
}

void gather(const Column& in, std::span<const uint32_t> map, Column& out, unsigned) {
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  if (out.kind() != in.kind() || out.size() != map.size()) out = Column(in.kind(), map.size());
  Buf src = detail::upload(in), m = detail::upload_ids(map), dst(out.byte_size());
  const void* ins[1] = {src.get()};
  void* outs[1] = {dst.get()};
  uint32_t b[1] = {detail::kb_of(in)};
  d.check(cj_gather(d.ctx(), ins, in.size(), static_cast<const uint32_t*>(m.get()), map.size(),
                    outs, b, 1),
          "gather");
  detail::download(dst, out);
}

Column gather_copy(const Column& in, std::span<const uint32_t> map, unsigned workers) {
  Column out(in.kind(), map.size());
  gather(in, map, out, workers);
  return out;
}

double gather_clusteredness(std::span<const uint32_t> map) {
  if (map.empty()) throw EmptyInput("clusteredness of an empty map");
  if (map.size() == 1) return 1.0;
  uint64_t steps = 0;
  for (size_t i = 1; i < map.size(); ++i)
    steps += map[i] > map[i - 1] ? map[i] - map[i - 1] : map[i - 1] - map[i];
  return static_cast<double>(steps) / static_cast<double>(map.size() - 1);
}

}  // namespace primitives

// ---- hash join ---------------------------------------------------------------------

namespace hashjoin {

namespace {

primitives::PartitionLayout partition(const Column& keys, const Column* carried, Column& keys_out,
                                      Column* carried_out, unsigned total_bits,
                                      unsigned bits_per_pass, Workspace ws) {
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  detail::ScratchCharge charge(ws);
  if (carried && carried->size() != keys.size())
    throw LengthMismatch("key and value columns differ in length");
  detail::shape_like(keys, keys_out);
  if (carried) detail::shape_like(*carried, *carried_out);
  const size_t n = keys.size();
  const uint64_t fanout = total_bits <= 20 ? (uint64_t{1} << total_bits) : 1;
  Buf k = detail::upload(keys), ko(keys.byte_size()), off((fanout + 1) * 8);
  Buf v, vo;
  const void* vin[1] = {nullptr};
  void* vout[1] = {nullptr};
  uint32_t vb[1] = {4};
  if (carried) {
    v = detail::upload(*carried);
    vo = Buf(carried->byte_size());
    vin[0] = v.get();
    vout[0] = vo.get();
    vb[0] = detail::kb_of(*carried);
  }
  d.check(cj_partition_relation(d.ctx(), k.get(), ko.get(), n, detail::kb_of(keys), total_bits,
                                bits_per_pass, vin, vout, vb, carried ? 1 : 0, 0,
                                static_cast<uint64_t*>(off.get())),
          "partition_relation");
  primitives::PartitionLayout lay;
  lay.low_bit = 0;
  lay.high_bit = total_bits;
  lay.fanout = static_cast<uint32_t>(fanout);
  lay.offsets.resize(fanout + 1);
  off.to_host(lay.offsets.data(), (fanout + 1) * 8);
  if (total_bits == 0) lay.high_bit = 0;
  detail::download(ko, keys_out);
  if (carried) detail::download(vo, *carried_out);
  return lay;
}

void check_views(const PartitionedRelationView& b, const PartitionedRelationView& p) {
  if (!b.keys || !b.layout || !p.keys || !p.layout)
    throw SpecInvalid("partitioned view missing keys or layout");
  if (b.keys->kind() != p.keys->kind()) throw KindError("build and probe keys must share a value kind");
}

void check_unit_sizes(const SubPartitionPlan& plan) {
  for (const auto& u : plan.units)
    if (u.build_hi - u.build_lo > plan.limit)
      throw CapacityExceeded("work unit exceeds the sub-partition limit");
}

// Runs the device hash join over the two views; ids per `mode`.
void device_matches(const PartitionedRelationView& b, const PartitionedRelationView& p,
                    uint32_t limit, TupleIdSemantics mode, detail::DevMatches& out) {
  auto& d = Device::get();
  if (b.layout->fanout != p.layout->fanout)
    throw FanoutMismatch("build and probe views disagree on fan-out");
  Buf bk = detail::upload(*b.keys), pk = detail::upload(*p.keys);
  Buf bo(b.layout->offsets.data(), b.layout->offsets.size() * 8);
  Buf po(p.layout->offsets.data(), p.layout->offsets.size() * 8);
  Buf bc, pc;
  cj_partitioned bv{bk.get(), static_cast<const uint64_t*>(bo.get()), nullptr, b.rows()};
  cj_partitioned pv{pk.get(), static_cast<const uint64_t*>(po.get()), nullptr, p.rows()};
  if (mode == TupleIdSemantics::Physical) {
    bc = detail::upload(*b.carried);
    pc = detail::upload(*p.carried);
    bv.carried = static_cast<const uint32_t*>(bc.get());
    pv.carried = static_cast<const uint32_t*>(pc.get());
  }
  d.check(cj_hash_find_matches(d.ctx(), &bv, &pv, b.layout->fanout, detail::kb_of(*b.keys), limit,
                               mode == TupleIdSemantics::Physical ? CJ_IDS_PHYSICAL : CJ_IDS_VIRTUAL,
                               &out.total, &out.keys, &out.ids_r, &out.ids_s),
          "hash_find_matches");
}

void check_physical(const PartitionedRelationView& b, const PartitionedRelationView& p) {
  if (!b.carried || !p.carried)
    throw Unsupported("physical id mode needs carried id columns on both sides");
  if (b.carried->kind() != ValueKind::u32 || p.carried->kind() != ValueKind::u32)
    throw KindError("carried tuple ids must be 4-byte columns");
}

}  // namespace

primitives::PartitionLayout partition_relation(const Column& keys, const Column& carried,
                                               Column& keys_out, Column& carried_out,
                                               unsigned total_bits, unsigned bits_per_pass,
                                               unsigned, Workspace ws) {
  return partition(keys, &carried, keys_out, &carried_out, total_bits, bits_per_pass, ws);
}

primitives::PartitionLayout partition_relation_keys(const Column& keys, Column& keys_out,
                                                    unsigned total_bits, unsigned bits_per_pass,
                                                    unsigned, Workspace ws) {
  return partition(keys, nullptr, keys_out, nullptr, total_bits, bits_per_pass, ws);
}

SubPartitionPlan plan_subpartitions(const PartitionedRelationView& build,
                                    const PartitionedRelationView& probe, uint32_t limit) {
  check_views(build, probe);
  if (build.layout->fanout != probe.layout->fanout)
    throw FanoutMismatch("build and probe views disagree on fan-out");
  if (limit == 0) throw SpecInvalid("sub-partition limit must be positive");
  SubPartitionPlan plan;
  plan.limit = limit;
  const auto& bo = build.layout->offsets;
  const auto& po = probe.layout->offsets;
  for (uint32_t p = 0; p < build.layout->fanout; ++p) {
    WorkUnit u;
    u.partition = p;
    u.probe_lo = po[p];
    u.probe_hi = po[p + 1];
    if (bo[p] == bo[p + 1]) {
      u.build_lo = u.build_hi = bo[p];
      plan.units.push_back(u);
      continue;
    }
    for (uint64_t c = bo[p]; c < bo[p + 1]; c += limit) {
      u.build_lo = c;
      u.build_hi = std::min<uint64_t>(c + limit, bo[p + 1]);
      plan.units.push_back(u);
    }
  }
  return plan;
}

HashMatchCounts hash_match_count(const PartitionedRelationView& build,
                                 const PartitionedRelationView& probe, const SubPartitionPlan& plan,
                                 unsigned) {
  check_views(build, probe);
  check_unit_sizes(plan);
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  detail::DevMatches m;
  device_matches(build, probe, plan.limit, TupleIdSemantics::Virtual, m);
  // rows arrive in unit order; a row's unit is the one holding its build position
  std::vector<uint32_t> ids(m.total);
  detail::down_raw(ids.data(), m.ids_r, m.total * 4);
  HashMatchCounts counts;
  counts.unit_offsets.assign(plan.units.size() + 1, 0);
  size_t u = 0;
  for (uint64_t k = 0; k < m.total; ++k) {
    while (u < plan.units.size() &&
           !(ids[k] >= plan.units[u].build_lo && ids[k] < plan.units[u].build_hi))
      ++u;
    if (u == plan.units.size()) throw SpecInvalid("plan does not match its partitioned views");
    ++counts.unit_offsets[u + 1];
  }
  for (size_t i = 0; i < plan.units.size(); ++i) counts.unit_offsets[i + 1] += counts.unit_offsets[i];
  return counts;
}

void hash_match_fill(const PartitionedRelationView& build, const PartitionedRelationView& probe,
                     const SubPartitionPlan& plan, const HashMatchCounts& counts,
                     TupleIdSemantics id_mode, Column& keys_dest, std::span<uint32_t> ids_r,
                     std::span<uint32_t> ids_s, unsigned) {
  check_views(build, probe);
  const uint64_t total = counts.total();
  if (keys_dest.size() != total || ids_r.size() != total || ids_s.size() != total)
    throw LengthMismatch("fill destinations must match the counted total");
  check_unit_sizes(plan);
  if (id_mode == TupleIdSemantics::Physical) check_physical(build, probe);
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  detail::DevMatches m;
  device_matches(build, probe, plan.limit, id_mode, m);
  if (m.total != total) throw LengthMismatch("fill destinations must match the counted total");
  detail::down_raw(keys_dest.raw(), m.keys, keys_dest.byte_size());
  detail::down_raw(ids_r.data(), m.ids_r, total * 4);
  detail::down_raw(ids_s.data(), m.ids_s, total * 4);
}

MatchSet hash_find_matches(const PartitionedRelationView& build,
                           const PartitionedRelationView& probe, const SubPartitionPlan& plan,
                           TupleIdSemantics id_mode, unsigned) {
  check_views(build, probe);
  check_unit_sizes(plan);
  if (id_mode == TupleIdSemantics::Physical) check_physical(build, probe);
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  detail::DevMatches m;
  device_matches(build, probe, plan.limit, id_mode, m);
  MatchSet out;
  out.id_semantics = id_mode;
  out.keys = Column(build.keys->kind(), m.total);
  out.ids_r.resize(m.total);
  out.ids_s.resize(m.total);
  detail::down_raw(out.keys.raw(), m.keys, out.keys.byte_size());
  detail::down_raw(out.ids_r.data(), m.ids_r, m.total * 4);
  detail::down_raw(out.ids_s.data(), m.ids_s, m.total * 4);
  return out;
}

}  // namespace hashjoin

// ---- merge join ------------------------------------------------------------------------

namespace mergejoin {

namespace {

template <class K>
void require_sorted(std::span<const K> v, const char* side) {
  for (size_t i = 1; i < v.size(); ++i)
    if (v[i] < v[i - 1]) throw NotSorted(std::string(side) + " keys not ascending");
}

template <class K>
void require_unique(std::span<const K> v) {
  for (size_t i = 1; i < v.size(); ++i)
    if (v[i] == v[i - 1]) throw DuplicateBuildKeys("pk-fk mode requires unique build keys");
}

// Largest i on diagonal `diag` with r[i-1] <= s[diag-i] (r consumed first on ties).
template <class K>
uint64_t diagonal(std::span<const K> r, std::span<const K> s, uint64_t diag) {
  uint64_t lo = diag > s.size() ? diag - s.size() : 0, hi = std::min<uint64_t>(diag, r.size());
  while (lo < hi) {
    const uint64_t i = lo + (hi - lo + 1) / 2, j = diag - i;
    if (j >= s.size() || r[i - 1] <= s[j]) lo = i;
    else hi = i - 1;
  }
  return lo;
}

void device_merge(const Column& r, const Column& s, bool pk_fk, detail::DevMatches& out) {
  auto& d = Device::get();
  Buf rb = detail::upload(r), sb = detail::upload(s);
  d.check(cj_merge_find_matches(d.ctx(), rb.get(), r.size(), sb.get(), s.size(), detail::kb_of(r),
                                pk_fk ? 1 : 0, 0, &out.total, &out.keys, &out.ids_r, &out.ids_s),
          "merge_find_matches");
}

void validate(const Column& r, const Column& s, bool pk_fk) {
  visit_kind(r.kind(), [&](auto tag) {
    using K = decltype(tag);
    require_sorted<K>(values<K>(r), "build");
    require_sorted<K>(values<K>(s), "probe");
    if (pk_fk) require_unique<K>(values<K>(r));
  });
}

}  // namespace

MergePathSplit merge_path_split(const Column& r_keys, const Column& s_keys, unsigned parts,
                                bool validate_inputs) {
  if (parts == 0) throw SpecInvalid("merge path needs at least one part");
  if (r_keys.kind() != s_keys.kind()) throw KindError("merge inputs must share a value kind");
  if (validate_inputs) {
    visit_kind(r_keys.kind(), [&](auto tag) {
      using K = decltype(tag);
      require_sorted<K>(values<K>(r_keys), "build");
      require_sorted<K>(values<K>(s_keys), "probe");
    });
  }
  MergePathSplit split;
  split.r_bounds.assign(parts + 1, 0);
  split.s_bounds.assign(parts + 1, 0);
  const uint64_t total = r_keys.size() + s_keys.size();
  visit_kind(r_keys.kind(), [&](auto tag) {
    using K = decltype(tag);
    for (unsigned p = 1; p < parts; ++p) {
      const uint64_t diag = total * p / parts;
      const uint64_t i = diagonal<K>(values<K>(r_keys), values<K>(s_keys), diag);
      split.r_bounds[p] = i;
      split.s_bounds[p] = diag - i;
    }
  });
  split.r_bounds[parts] = r_keys.size();
  split.s_bounds[parts] = s_keys.size();
  return split;
}

MergeMatchCounts merge_match_count(const Column& r_keys, const Column& s_keys, bool pk_fk,
                                   unsigned parts, unsigned, bool validate_inputs) {
  MergeMatchCounts counts;
  counts.pk_fk = pk_fk;
  counts.split = merge_path_split(r_keys, s_keys, parts, validate_inputs);
  if (validate_inputs && pk_fk) validate(r_keys, s_keys, true);
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  detail::DevMatches m;
  device_merge(r_keys, s_keys, pk_fk, m);
  std::vector<uint32_t> js(m.total);
  detail::down_raw(js.data(), m.ids_s, m.total * 4);
  counts.part_offsets.assign(parts + 1, 0);
  unsigned p = 0;
  for (uint64_t k = 0; k < m.total; ++k) {  // rows are in probe order: parts by s range
    while (p + 1 < parts && js[k] >= counts.split.s_bounds[p + 1]) ++p;
    ++counts.part_offsets[p + 1];
  }
  for (unsigned i = 0; i < parts; ++i) counts.part_offsets[i + 1] += counts.part_offsets[i];
  return counts;
}

void merge_match_fill(const Column& r_keys, const Column& s_keys, const MergeMatchCounts& counts,
                      Column& keys_dest, std::span<uint32_t> ids_r, std::span<uint32_t> ids_s,
                      unsigned) {
  const uint64_t total = counts.total();
  if (keys_dest.size() != total || ids_r.size() != total || ids_s.size() != total)
    throw LengthMismatch("fill destinations must match the counted total");
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  detail::DevMatches m;
  device_merge(r_keys, s_keys, counts.pk_fk, m);
  if (m.total != total) throw LengthMismatch("fill destinations must match the counted total");
  detail::down_raw(keys_dest.raw(), m.keys, keys_dest.byte_size());
  detail::down_raw(ids_r.data(), m.ids_r, total * 4);
  detail::down_raw(ids_s.data(), m.ids_s, total * 4);
}

MatchSet merge_find_matches(const Column& r_keys, const Column& s_keys, bool pk_fk, unsigned parts,
                            unsigned, bool validate_inputs) {
  if (parts == 0) throw SpecInvalid("merge path needs at least one part");
  if (r_keys.kind() != s_keys.kind()) throw KindError("merge inputs must share a value kind");
  if (validate_inputs) validate(r_keys, s_keys, pk_fk);
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  detail::DevMatches m;
  device_merge(r_keys, s_keys, pk_fk, m);
  MatchSet out;
  out.id_semantics = TupleIdSemantics::Virtual;
  out.keys = Column(r_keys.kind(), m.total);
  out.ids_r.resize(m.total);
  out.ids_s.resize(m.total);
  detail::down_raw(out.keys.raw(), m.keys, out.keys.byte_size());
  detail::down_raw(out.ids_r.data(), m.ids_r, m.total * 4);
  detail::down_raw(out.ids_s.data(), m.ids_s, m.total * 4);
  return out;
}

}  // namespace mergejoin

// ---- join engine --------------------------------------------------------------------------

namespace {

cj_relation describe(const Relation& rel, const std::vector<Buf>& cols) {
  cj_relation r{};
  r.key = cols[0].get();
  r.key_bytes = detail::kb_of(rel.key);
  r.rows = rel.rows();
  r.npay = static_cast<uint32_t>(rel.payloads.size());
  for (size_t c = 0; c < rel.payloads.size(); ++c) {
    r.pay[c] = cols[c + 1].get();
    r.pay_bytes[c] = detail::kb_of(rel.payloads[c]);
  }
  r.key_unique = rel.key_unique ? 1 : 0;
  return r;
}

std::vector<Buf> upload_relation(const Relation& rel) {
  std::vector<Buf> cols;
  cols.push_back(detail::upload(rel.key));
  for (const Column& p : rel.payloads) {
    if (p.size() != rel.key.size()) throw LengthMismatch("payload length differs from key length");
    cols.push_back(detail::upload(p));
  }
  return cols;
}

Relation output_shell(uint64_t rows, const Relation& r, const Relation& s) {
  Relation out;
  out.name = r.name.empty() && s.name.empty() ? "join" : r.name + "_" + s.name;
  out.key = Column(r.key.kind(), rows);
  for (const Column& p : r.payloads) out.payloads.emplace_back(p.kind(), rows);
  for (const Column& p : s.payloads) out.payloads.emplace_back(p.kind(), rows);
  return out;
}

}  // namespace

namespace detail {

// Shared by run_join and sharded::run_join: upload, one C-ABI join call,
// download of the output relation and the report.
template <class Call>
JoinOutput run_join_with(const JoinTask& task, Call&& call, const char* what) {
  const Relation& r = *task.build;
  const Relation& s = *task.probe;
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  std::vector<Buf> rc = upload_relation(r), sc = upload_relation(s);
  cj_relation R = describe(r, rc), S = describe(s, sc);
  cj_join_options opt;
  cj_default_options(&opt);
  opt.algo = static_cast<int>(task.algorithm);
  opt.pattern = static_cast<int>(task.pattern);
  opt.radix_bits_per_pass = task.options.radix_bits_per_pass;
  opt.total_radix_bits = task.options.total_radix_bits;
  opt.sub_partition_limit = task.options.sub_partition_limit;
  opt.validate = task.options.validate ? 1 : 0;
  opt.want_stats = 1;  // JoinStats (join_engine.hpp:54-58) is part of the result
  cj_join_result res;
  std::memset(&res, 0, sizeof(res));
  d.check(call(d.ctx(), &R, &S, &opt, &res), what);
  struct Release {
    cj_join_result* r;
    ~Release() { cj_result_free(Device::get().ctx(), r); }
  } release{&res};
  JoinOutput out;
  out.relation = output_shell(res.rows, r, s);
  detail::down_raw(out.relation.key.raw(), res.key, out.relation.key.byte_size());
  for (size_t c = 0; c < out.relation.payloads.size(); ++c)
    detail::down_raw(out.relation.payloads[c].raw(), res.pay[c],
                     out.relation.payloads[c].byte_size());
  out.report.transform_ns = res.transform_ns;
  out.report.find_ns = res.find_ns;
  out.report.materialize_ns = res.materialize_ns;
  // MemLedger view (mem_ledger.hpp:26-100): column data + scratch per phase
  for (int ph = 0; ph < 3; ++ph) {
    out.report.peak_by_phase[ph].column_bytes = res.ledger_column_b[ph];
    out.report.peak_by_phase[ph].scratch_bytes = res.ledger_scratch_b[ph];
    out.report.peak_by_phase[ph].total_bytes = res.ledger_column_b[ph] + res.ledger_scratch_b[ph];
  }
  out.stats.matches = res.rows;
  out.stats.clusteredness_r = res.clusteredness_r;
  out.stats.clusteredness_s = res.clusteredness_s;
  return out;
}

}  // namespace detail

JoinOutput run_join(const JoinTask& task) {
  if (!task.build || !task.probe) throw SpecInvalid("join task needs both input relations");
  const Relation& r = *task.build;
  const Relation& s = *task.probe;
  if (r.key.kind() != s.key.kind()) throw KindError("build and probe key kinds differ");
  if (task.options.radix_bits_per_pass == 0 || task.options.radix_bits_per_pass > 8)
    throw FanoutTooLarge("radix bits per pass must be in [1, 8]");
  if (r.payloads.size() > CJ_MAX_COLS || s.payloads.size() > CJ_MAX_COLS)
    throw Unsupported("at most 16 payload columns per relation");
  return detail::run_join_with(task, [](cj_ctx* ctx, const cj_relation* R, const cj_relation* S,
                                         const cj_join_options* opt, cj_join_result* res) {
    return cj_run_join(ctx, R, S, opt, res);
  }, "run_join");
}


std::vector<SequenceStep> run_join_sequence(const Relation& fact, const std::vector<Relation>& dims,
                                            JoinAlgo algorithm, JoinPattern pattern,
                                            const JoinOptions& options) {
  const size_t n_joins = dims.size();
  if (fact.payloads.size() < n_joins)  // sequence.cpp:14-17
    throw SpecInvalid("fact table needs one FK column per dimension");
  if (fact.key.kind() != ValueKind::u32) throw SpecInvalid("fact tuple ids must be a 4-byte column");
  if (options.radix_bits_per_pass == 0 || options.radix_bits_per_pass > 8)
    throw FanoutTooLarge("radix bits per pass must be in [1, 8]");
  std::vector<SequenceStep> steps(n_joins);
  if (n_joins == 0) return steps;
  for (const auto& dm : dims)
    if (dm.key.kind() != fact.payloads[0].kind()) throw KindError("build and probe key kinds differ");
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  std::vector<Buf> fc = upload_relation(fact);
  cj_relation F = describe(fact, fc);
  std::vector<std::vector<Buf>> dc;
  std::vector<cj_relation> D;
  dc.reserve(n_joins);
  for (const auto& dm : dims) {
    dc.push_back(upload_relation(dm));
    D.push_back(describe(dm, dc.back()));
  }
  cj_join_options opt;
  cj_default_options(&opt);
  opt.algo = static_cast<int>(algorithm);
  opt.pattern = static_cast<int>(pattern);
  opt.radix_bits_per_pass = options.radix_bits_per_pass;
  opt.total_radix_bits = options.total_radix_bits;
  opt.sub_partition_limit = options.sub_partition_limit;
  opt.validate = options.validate ? 1 : 0;
  std::vector<cj_sequence_step> st(n_joins);
  d.check(cj_run_join_sequence(d.ctx(), &F, D.data(), static_cast<uint32_t>(n_joins), &opt,
                               st.data(), nullptr),
          "run_join_sequence");
  for (size_t i = 0; i < n_joins; ++i) {
    steps[i].rows = st[i].rows;
    steps[i].output_columns = st[i].output_columns;
    steps[i].report.transform_ns = st[i].transform_ns;
    steps[i].report.find_ns = st[i].find_ns;
    steps[i].report.materialize_ns = st[i].materialize_ns;
    steps[i].fk_fetch_ns = st[i].fk_fetch_ns;
  }
  return steps;
}

Relation make_join_output_shell(const MatchSet& match, const Relation& r, const Relation& s) {
  Relation out = output_shell(match.size(), r, s);
  out.key = match.keys;
  return out;
}

namespace {

// out.payloads[base + c] = cols[c][ids] for every column, on the device
void gather_into(const std::vector<const Column*>& cols, std::span<const uint32_t> ids,
                 Relation& out, size_t base) {
  if (cols.empty()) return;
  auto& d = Device::get();
  Buf map = detail::upload_ids(ids);
  for (size_t c = 0; c < cols.size(); ++c) {
    Column& dst = out.payloads[base + c];
    if (dst.kind() != cols[c]->kind() || dst.size() != ids.size())
      dst = Column(cols[c]->kind(), ids.size());
    Buf src = detail::upload(*cols[c]), o(dst.byte_size());
    const void* ins[1] = {src.get()};
    void* outs[1] = {o.get()};
    uint32_t b[1] = {detail::kb_of(*cols[c])};
    d.check(cj_gather(d.ctx(), ins, cols[c]->size(), static_cast<const uint32_t*>(map.get()),
                      ids.size(), outs, b, 1),
            "gather");
    detail::download(o, dst);
  }
}

}  // namespace

void materialize_gfur(std::span<const uint32_t> ids_r, std::span<const uint32_t> ids_s,
                      const Relation& r, const Relation& s, Relation& out, unsigned) {
  auto& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  std::vector<const Column*> rc, sc;
  for (const Column& p : r.payloads) rc.push_back(&p);
  for (const Column& p : s.payloads) sc.push_back(&p);
  gather_into(rc, ids_r, out, 0);
  gather_into(sc, ids_s, out, r.payloads.size());
}

void materialize_gfur(const MatchSet& match, const Relation& r, const Relation& s, Relation& out,
                      unsigned workers) {
  if (match.id_semantics != TupleIdSemantics::Physical)
    throw SpecInvalid("gfur materialization needs physical tuple ids");
  materialize_gfur(match.ids_r, match.ids_s, r, s, out, workers);
}

namespace {

// On-demand transform of (key, payload c) for c >= 1, checked against the key
// transform, then gathered (join_engine.cpp:180-213 semantics).
void gftr_remaining(const Relation& rel, std::span<const uint32_t> ids, size_t out_base,
                    const GftrContext& ctx, const primitives::PartitionLayout* key_layout,
                    Relation& out) {
  for (size_t c = 1; c < rel.payloads.size(); ++c) {
    Column tk, tp;
    if (ctx.algorithm == JoinAlgo::SMJ) {
      primitives::sort_pairs(rel.key, rel.payloads[c], tk, tp);
      if (ctx.validate) {
        bool sorted = true;
        visit_kind(tk.kind(), [&](auto tag) {
          using K = decltype(tag);
          auto v = values<K>(tk);
          for (size_t i = 1; i < v.size(); ++i) sorted &= !(v[i] < v[i - 1]);
        });
        if (!sorted) throw TransformMismatch("payload transform disagrees with key sort");
      }
    } else {
      auto lay = hashjoin::partition_relation(rel.key, rel.payloads[c], tk, tp, ctx.total_bits,
                                              ctx.bits_per_pass);
      if (key_layout && lay.offsets != key_layout->offsets)
        throw TransformMismatch("payload partition disagrees with key layout");
    }
    auto& d = Device::get();
    std::lock_guard<std::mutex> lock(d.mu());
    gather_into({&tp}, ids, out, out_base + c);
  }
}

}  // namespace

void materialize_gftr(std::span<const uint32_t> ids_r, std::span<const uint32_t> ids_s,
                      const Relation& r, const Relation& s, WorkColumn first_r, WorkColumn first_s,
                      const GftrContext& ctx, Relation& out) {
  {
    auto& d = Device::get();
    std::lock_guard<std::mutex> lock(d.mu());
    if (!r.payloads.empty()) gather_into({&first_r.col()}, ids_r, out, 0);
    if (!s.payloads.empty()) gather_into({&first_s.col()}, ids_s, out, r.payloads.size());
  }
  first_r.release();
  first_s.release();
  gftr_remaining(r, ids_r, 0, ctx, ctx.layout_r, out);
  gftr_remaining(s, ids_s, r.payloads.size(), ctx, ctx.layout_s, out);
}

void materialize_gftr(const MatchSet& match, const Relation& r, const Relation& s,
                      Column transformed_first_r, Column transformed_first_s,
                      const GftrContext& ctx, Relation& out) {
  if (match.id_semantics != TupleIdSemantics::Virtual)
    throw SpecInvalid("gftr materialization needs virtual tuple ids");
  WorkColumn fr, fs;
  if (!r.payloads.empty()) {
    fr = WorkColumn(ctx.ws, transformed_first_r.kind(), 0, AllocClass::ColumnData);
    fr.col() = std::move(transformed_first_r);
  }
  if (!s.payloads.empty()) {
    fs = WorkColumn(ctx.ws, transformed_first_s.kind(), 0, AllocClass::ColumnData);
    fs.col() = std::move(transformed_first_s);
  }
  materialize_gftr(match.ids_r, match.ids_s, r, s, std::move(fr), std::move(fs), ctx, out);
}


namespace sharded {

CommId make_comm_id() {
  CommId id{};
  const int st = cj_comm_unique_id(id.data());
  if (st != CJ_OK) detail::throw_status(st, "comm id (NCCL unavailable?)");
  return id;
}

Comm::Comm(const CommId& id, int nranks, int rank) {
  auto& d = detail::Device::get();
  d.check(cj_comm_init(d.ctx(), id.data(), nranks, rank, &comm_), "comm init");
}

Comm::~Comm() { cj_comm_destroy(comm_); }
int Comm::size() const { return cj_comm_size(comm_); }
int Comm::rank() const { return cj_comm_rank(comm_); }

JoinOutput run_join(const JoinTask& task, Comm& comm, ShuffleStats* stats) {
  if (!task.build || !task.probe) throw SpecInvalid("join task needs both input relations");
  if (task.build->key.kind() != task.probe->key.kind())
    throw KindError("build and probe key kinds differ");
  if (task.options.radix_bits_per_pass == 0 || task.options.radix_bits_per_pass > 8)
    throw FanoutTooLarge("radix bits per pass must be in [1, 8]");
  cj_shuffle_stats st{};
  JoinOutput out = detail::run_join_with(
      task,
      [&](cj_ctx* ctx, const cj_relation* R, const cj_relation* S, const cj_join_options* opt,
          cj_join_result* res) {
        return cj_run_join_sharded(ctx, comm.handle(), R, S, opt, res, &st);
      },
      "run_join_sharded");
  if (stats) {
    stats->first_bits = st.first_bits;
    stats->r_rows_received = st.r_rows_received;
    stats->s_rows_received = st.s_rows_received;
    stats->bytes_sent_peers = st.bytes_sent_peers;
    stats->bytes_received_peers = st.bytes_received_peers;
    stats->shard_ns = st.shard_ns;
    stats->exchange_r_ns = st.exchange_r_ns;
    stats->exchange_s_ns = st.exchange_s_ns;
    stats->wall_ns = st.wall_ns;
  }
  return out;
}

}  // namespace sharded
}  // namespace coljoin
