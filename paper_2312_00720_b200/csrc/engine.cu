// Context, error plumbing, the run_join device pipeline and the C-ABI
// (include/cj_api.h).
//
// Reference: run_join (join_engine.cpp:255-361), transform_side (:68-113),
// materialize_gfur (:161-176), materialize_gftr (:180-253).
//
// Pipelines (B200 design, all device-resident):
//   PHJ-GFTR  transform: key + ALL payload columns of a side partitioned in one
//             LSD pass sequence (the reference re-partitions payloads 2..n on
//             demand, join_engine.cpp:180-213; carrying them in the same scatter
//             reads the key once per pass and skips the re-transforms).
//             find+materialise: one fused kernel writes finished output rows,
//             gathering R payloads from the staged build chunk and S payloads
//             at the (clustered) probe positions.
//   SMJ-GFTR  transform: full-width stable sort of key + all payloads;
//             find+materialise: fused merge-join kernel.
//   *-GFUR    transform: (key, id) with ids born in pass 1; find writes
//             physical ids (SMJ resolves them in the same kernel); materialise
//             gathers every payload from the untransformed relations.
//   NPHJ      global-table hash join (no partitioning), see nphj.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "cj_device.cuh"
#include "cj_internal.cuh"

namespace cj {

void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    const int code = e == cudaErrorMemoryAllocation ? CJ_ERR_OUT_OF_MEMORY : CJ_ERR_CUDA;
    fail(code, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

void scan_counts(cj_ctx* ctx, const uint64_t* in, uint64_t n, uint64_t* out, uint64_t* total_dev) {
  const uint64_t tiles = std::max<uint64_t>((n + dev::kScanTile - 1) / dev::kScanTile, 1);
  Scratch tot(ctx, tiles * 8);
  ctx->kbegin("scan", n * 16);
  dev::k_scan_tiles<0><<<(unsigned)tiles, dev::kScanThreads, 0, ctx->stream>>>(in, n, out,
                                                                               tot.as<uint64_t>());
  dev::k_scan_top<0><<<1, 1024, 0, ctx->stream>>>(tot.as<uint64_t>(), tiles, total_dev);
  if (n > 0)
    dev::k_scan_fix<0><<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(out, n,
                                                                            tot.as<uint64_t>());
  ctx->kend();
  ctx->launches += 2;
  CJ_CUDA(cudaGetLastError());
}

void raise_device_errors(cj_ctx* ctx) {
  if (ctx->err_known_clean) {  // the caller just read the error word after a sync
    ctx->err_known_clean = false;
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));  // callers rely on an idle stream after this
    return;
  }
  CJ_CUDA(cudaMemcpyAsync(ctx->host_pinned + 64, ctx->err_word, sizeof(uint32_t),
                          cudaMemcpyDeviceToHost, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  const uint32_t e = ctx->host_pinned[64];
  if (!e) return;
  CJ_CUDA(cudaMemsetAsync(ctx->err_word, 0, sizeof(uint32_t), ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  if (e & kErrOOB) fail(CJ_ERR_INDEX_OUT_OF_BOUNDS, "gather map entry past input length");
  if (e & kErrOverflow) fail(CJ_ERR_CAPACITY_EXCEEDED, "join output exceeds its capacity");
  if (e & kErrNotSorted) fail(CJ_ERR_NOT_SORTED, "keys not ascending");
  if (e & kErrDupKeys) fail(CJ_ERR_DUPLICATE_BUILD_KEYS, "pk-fk mode requires unique build keys");
  if (e & dev::kErrStall) fail(CJ_ERR_CUDA, "decoupled look-back stalled (internal error)");
}

static __global__ void k_abs_diff_sum(const uint32_t* __restrict__ ids, uint64_t n,
                               unsigned long long* out) {
  uint64_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = ids[i - 1], b = ids[i];
    acc += a > b ? a - b : b - a;
  }
  acc = dev::warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

// primitives.cpp:398-407 gather_clusteredness over a device map
double clusteredness(cj_ctx* ctx, const uint32_t* ids, uint64_t n) {
  if (n <= 1) return 1.0;
  Scratch acc(ctx, 8);
  CJ_CUDA(cudaMemsetAsync(acc.p, 0, 8, ctx->stream));
  ctx->kbegin("clusteredness", n * 4);
  k_abs_diff_sum<<<grid_for(n, 256 * 16, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
      ids, n, acc.as<unsigned long long>());
  ctx->kend();
  uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  CJ_CUDA(cudaMemcpyAsync(h, acc.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  return static_cast<double>(h[0]) / static_cast<double>(n - 1);
}

unsigned default_total_radix_bits(uint64_t build_rows) {  // task.hpp:45-50
  if (build_rows > (1ull << 20)) return 16;
  unsigned bits = 0;
  while ((build_rows >> bits) > 1024) ++bits;
  return bits > 16 ? 16 : bits;
}

PassPlan plan_bits(unsigned total_bits, unsigned per_pass) {  // task.hpp:54-63
  if (per_pass == 0 || per_pass > 8) fail(CJ_ERR_FANOUT_TOO_LARGE, "bits per pass must be in [1, 8]");
  PassPlan p;
  for (unsigned lo = 0; lo < total_bits; lo += per_pass) {
    if (p.npasses == CJ_MAX_PASSES * 3) break;
    p.lo[p.npasses] = lo;
    p.hi[p.npasses] = std::min(lo + per_pass, total_bits);
    ++p.npasses;
  }
  return p;
}

PassPlan full_width_plan(int key_bytes) { return plan_bits((unsigned)key_bytes * 8, 8); }

// The device plan for a partition over [0, total_bits): the stable LSD result
// does not depend on how the bits are split into passes, so the split is a
// performance choice — at least ceil(total / per_pass) passes (the reference's
// task.hpp:54-63 plan) and at least ceil(total / 6), of balanced width.  The
// scatter is shared-memory bound and its cost per pass falls steeply with the
// digit count: C2's 16 bits in three 6/5/5-bit passes beat two 8-bit passes
// (11.24 vs 11.43 ms per join; profiles/r01d_summary.md).
PassPlan device_plan(unsigned total_bits, unsigned per_pass) {
  if (per_pass == 0 || per_pass > 8) fail(CJ_ERR_FANOUT_TOO_LARGE, "bits per pass must be in [1, 8]");
  unsigned np = std::max((total_bits + per_pass - 1) / per_pass, (total_bits + 5) / 6);
  if (const char* e = std::getenv("CJ_PHJ_PASSES")) np = (unsigned)std::max(1, std::atoi(e));
  np = std::max(np, (total_bits + 7) / 8);
  np = std::min(np, std::max(total_bits, 1u));
  PassPlan p;
  unsigned lo = 0;
  for (unsigned i = 0; i < np && i < CJ_MAX_PASSES * 3; ++i) {
    const unsigned w = (total_bits - lo + (np - i) - 1) / (np - i);
    p.lo[p.npasses] = lo;
    p.hi[p.npasses] = lo + w;
    ++p.npasses;
    lo += w;
  }
  return p;
}

// Plan for an input already stably grouped by its low `f` key bits (the
// sharded join's received rows): pass [0, f) is marked done, the remaining
// bits [f, total) run in balanced passes of at most `max_w` bits (and at least
// ceil(rest / per_pass) of them).  Same stable layout as the full plan.
PassPlan presorted_plan(unsigned total_bits, unsigned f, unsigned max_w, unsigned per_pass) {
  if (f > total_bits) f = total_bits;
  PassPlan p;
  p.npasses = 1;
  p.lo[0] = 0;
  p.hi[0] = f;
  p.done = 1;
  const unsigned rest = total_bits - f;
  if (rest == 0) return p;
  unsigned np = std::max((rest + per_pass - 1) / per_pass, (rest + max_w - 1) / max_w);
  np = std::min(np, rest);
  unsigned lo = f;
  for (unsigned i = 0; i < np && p.npasses < CJ_MAX_PASSES * 3; ++i) {
    const unsigned w = (total_bits - lo + (np - i) - 1) / (np - i);
    p.lo[p.npasses] = lo;
    p.hi[p.npasses] = lo + w;
    ++p.npasses;
    lo += w;
  }
  return p;
}

void check_key_bytes(uint32_t kb) {
  if (kb != 4 && kb != 8) fail(CJ_ERR_KIND, "key must be a 4- or 8-byte integer column");
}

// LSD plans longer than CJ_MAX_PASSES (e.g. 20 bits at 1 bit/pass) run in
// segments; each segment is itself stable, so the composition is the plan.
void lsd_any(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int kb,
             const PassPlan& plan, const ValCols& vals, unsigned long long* key_or) {
  if (plan.npasses <= CJ_MAX_PASSES) {
    lsd_partition(ctx, keys, keys_out, n, kb, plan, vals, nullptr, key_or);
    return;
  }
  const void* cur = keys;
  ValCols v = vals;
  for (int s = 0; s < plan.npasses; s += CJ_MAX_PASSES) {
    PassPlan seg;
    seg.npasses = std::min(CJ_MAX_PASSES, plan.npasses - s);
    seg.done = std::max(0, std::min(plan.done - s, seg.npasses));
    for (int i = 0; i < seg.npasses; ++i) {
      seg.lo[i] = plan.lo[s + i];
      seg.hi[i] = plan.hi[s + i];
    }
    lsd_partition(ctx, cur, keys_out, n, kb, seg, v, nullptr, s == 0 ? key_or : nullptr);
    cur = keys_out;
    for (int c = 0; c < v.n; ++c) v.in[c] = v.out[c];
    v.gen_ids = 0;
  }
}

struct Side {
  void* keys = nullptr;
  void* cols[CJ_MAX_COLS + 1] = {};   // transformed carried columns
  uint64_t* offsets = nullptr;        // PHJ layout (device)
  unsigned long long* key_or = nullptr;  // PHJ: OR of the keys (from the first histogram)
};

struct Timer {
  cj_ctx* ctx;
  cudaEvent_t ev[4];
  explicit Timer(cj_ctx* c) : ctx(c) {
    for (auto& e : ev) CJ_CUDA(cudaEventCreate(&e));
  }
  ~Timer() {
    for (auto& e : ev) cudaEventDestroy(e);
  }
  void mark(int i) { CJ_CUDA(cudaEventRecord(ev[i], ctx->stream)); }
  uint64_t ns(int a, int b) {
    float ms = 0;
    CJ_CUDA(cudaEventElapsedTime(&ms, ev[a], ev[b]));
    return static_cast<uint64_t>(ms * 1e6);
  }
};

void validate_relation(const cj_relation* r, const char* what) {
  if (!r) fail(CJ_ERR_SPEC_INVALID, std::string("join task needs ") + what);
  check_key_bytes(r->key_bytes);
  if (r->rows > 0x7fffffffull) fail(CJ_ERR_SPEC_INVALID, "relation exceeds the 2^31-1 row cap");
  if (r->npay > CJ_MAX_COLS) fail(CJ_ERR_UNSUPPORTED, "too many payload columns");
  for (uint32_t c = 0; c < r->npay; ++c)
    if (r->pay_bytes[c] != 4 && r->pay_bytes[c] != 8)
      fail(CJ_ERR_KIND, "payload columns must be 4- or 8-byte integers");
}

// Transform one side: partition (PHJ) or sort (SMJ) the key with the carried
// columns.  gfur: carried = generated ids; gftr: carried = every payload.
Side transform(cj_ctx* ctx, const cj_relation* rel, int algo, bool gfur, unsigned total_bits,
               unsigned bits_per_pass, std::vector<void*>& owned, unsigned presorted = 0) {
  Side s;
  const uint64_t n = rel->rows;
  const int kb = (int)rel->key_bytes;
  s.keys = ctx->alloc(n * kb + kPad, cj_ctx::kColumnData, n * kb);
  owned.push_back(s.keys);
  ValCols v;
  if (gfur) {
    v.n = 1;
    v.gen_ids = 1;
    v.in[0] = nullptr;
    v.bytes[0] = 4;
    v.out[0] = ctx->alloc(n * 4 + kPad, cj_ctx::kColumnData, n * 4);
    owned.push_back(v.out[0]);
  } else {
    v.n = (int)rel->npay;
    for (uint32_t c = 0; c < rel->npay; ++c) {
      v.in[c] = rel->pay[c];
      v.bytes[c] = rel->pay_bytes[c];
      v.out[c] = ctx->alloc(n * rel->pay_bytes[c] + kPad, cj_ctx::kColumnData,
                            n * rel->pay_bytes[c]);
      owned.push_back(v.out[c]);
    }
  }
  for (int c = 0; c < v.n; ++c) s.cols[c] = v.out[c];
  struct LiveScope {  // see cj_ctx::assume_live_passes
    cj_ctx* c;
    explicit LiveScope(cj_ctx* x) : c(x) { c->assume_live_passes = true; }
    ~LiveScope() { c->assume_live_passes = false; }
  } live_scope(ctx);
  if (algo == CJ_SMJ) {
    PassPlan plan = sort_plan(ctx, rel->key, n, kb, v);
    if (presorted > 0) {  // keys above bit B are zero: sorted by [0, f >= B) is sorted
      const unsigned bits = plan.npasses ? plan.hi[plan.npasses - 1] : 0;
      plan = presorted_plan(bits, std::min(presorted, bits), 8, 8);
    }
    lsd_any(ctx, rel->key, s.keys, n, kb, plan, v);
  } else {
    s.offsets = static_cast<uint64_t*>(ctx->alloc(sizeof(uint64_t) * ((1ull << total_bits) + 1)));
    owned.push_back(s.offsets);
    if (total_bits == 0) {
      copy_columns(ctx, rel->key, s.keys, n, kb, v);
    } else {
      s.key_or = static_cast<unsigned long long*>(ctx->alloc(8));
      owned.push_back(s.key_or);
      CJ_CUDA(cudaMemsetAsync(s.key_or, 0, 8, ctx->stream));
      // a hint wider than the partition bits says nothing about them
      lsd_any(ctx, rel->key, s.keys, n, kb,
              presorted > 0 && presorted <= total_bits
                  ? presorted_plan(total_bits, presorted, 6, bits_per_pass)
                  : device_plan(total_bits, bits_per_pass), v, s.key_or);
    }
    partition_offsets(ctx, s.keys, n, kb, total_bits, s.offsets);
  }
  return s;
}

void alloc_output(cj_ctx* ctx, const cj_relation* r, const cj_relation* s, uint64_t cap,
                  bool ids, cj_join_result* res) {
  const uint64_t c = std::max<uint64_t>(cap, 1);
  constexpr int kOut = cj_ctx::kOutputData, kCol = cj_ctx::kColumnData;
  res->key = ctx->alloc(c * r->key_bytes, kOut);
  for (uint32_t i = 0; i < r->npay; ++i) res->pay[i] = ctx->alloc(c * r->pay_bytes[i], kOut);
  for (uint32_t i = 0; i < s->npay; ++i)
    res->pay[r->npay + i] = ctx->alloc(c * s->pay_bytes[i], kOut);
  if (ids) {  // the tuple-id maps: column data (join_engine.cpp:300-301), |T| entries
    res->ids_r = static_cast<uint32_t*>(ctx->alloc(c * 4, kCol, cap * 4));
    res->ids_s = static_cast<uint32_t*>(ctx->alloc(c * 4, kCol, cap * 4));
  }
}

void free_output(cj_ctx* ctx, cj_join_result* res) {
  if (res->key) ctx->release(res->key);
  res->key = nullptr;
  for (auto& p : res->pay) {
    if (p) ctx->release(p);
    p = nullptr;
  }
  if (res->ids_r) ctx->release(res->ids_r);
  if (res->ids_s) ctx->release(res->ids_s);
  res->ids_r = res->ids_s = nullptr;
}

// Device bytes this call holds (outputs, transformed columns, scratch) at
// their high-water mark in each phase — PhaseReport's per-phase peaks
// (mem_ledger.hpp:231-246) measured on the device arena instead of a ledger.
// The ledger view follows MemLedger::begin_phase (mem_ledger.hpp:40-47): bytes
// carried in from earlier phases count toward a phase's peak; each phase's
// snapshot is (column, scratch) at the high-water mark of their sum.
struct PhasePeaks {
  cj_ctx* ctx;
  uint64_t base;
  uint64_t lbase[2];
  int phase = 0;
  cj_join_result* res;
  PhasePeaks(cj_ctx* c, cj_join_result* r) : ctx(c), base(c->live), res(r) {
    c->live_peak = c->live;
    lbase[0] = c->ledger[0];
    lbase[1] = c->ledger[1];
    c->ledger_reset_peak();
  }
  uint64_t next() {  // peak since the last call; starts the next phase
    const uint64_t p = ctx->live_peak > base ? ctx->live_peak - base : 0;
    ctx->live_peak = ctx->live;
    if (phase < 3) {
      res->ledger_column_b[phase] =
          ctx->ledger_peak[1] > lbase[1] ? ctx->ledger_peak[1] - lbase[1] : 0;
      res->ledger_scratch_b[phase] =
          ctx->ledger_peak[0] > lbase[0] ? ctx->ledger_peak[0] - lbase[0] : 0;
    }
    ++phase;
    ctx->ledger_reset_peak();
    return p;
  }
};

void run_join_dev(cj_ctx* ctx, const cj_relation* R, const cj_relation* S,
                  const cj_join_options* opt, cj_join_result* res, const JoinHooks* hooks) {
  const unsigned presorted = hooks ? hooks->presorted_bits : 0;
  validate_relation(R, "a build relation");
  validate_relation(S, "a probe relation");
  if (R->key_bytes != S->key_bytes) fail(CJ_ERR_KIND, "build and probe key kinds differ");
  if (opt->radix_bits_per_pass == 0 || opt->radix_bits_per_pass > 8)
    fail(CJ_ERR_FANOUT_TOO_LARGE, "radix bits per pass must be in [1, 8]");
  if (opt->algo != CJ_SMJ && opt->algo != CJ_PHJ && opt->algo != CJ_NPHJ)
    fail(CJ_ERR_SPEC_INVALID, "unknown join algorithm");
  const int kb = (int)R->key_bytes;
  const bool gfur = opt->pattern == CJ_GFUR;
  const bool pk_fk = R->key_unique != 0;
  const unsigned total_bits = opt->total_radix_bits >= 0 ? (unsigned)opt->total_radix_bits
                                                         : default_total_radix_bits(R->rows);
  if (opt->algo == CJ_PHJ && (total_bits > 20 || total_bits > (unsigned)kb * 8))
    fail(CJ_ERR_FANOUT_TOO_LARGE, "partition fan-out capped at 2^20 and the key width");
  const bool want_ids = opt->want_ids || opt->want_stats;
  {
    // peak device footprint of the call: transformed R and S, one side's LSD
    // ping-pong scratch, the output (|S| rows for PK-FK) and find scratch
    uint64_t rb = R->key_bytes, sb = S->key_bytes, ob = R->key_bytes + 8;
    for (uint32_t c = 0; c < R->npay; ++c) rb += R->pay_bytes[c], ob += R->pay_bytes[c];
    for (uint32_t c = 0; c < S->npay; ++c) sb += S->pay_bytes[c], ob += S->pay_bytes[c];
    const uint64_t big = std::max(rb * R->rows, sb * S->rows);
    ctx->reserve(rb * R->rows + sb * S->rows + big + ob * S->rows + 4 * S->rows + (64ull << 20));
  }
  std::memset(res, 0, sizeof(*res));
  std::vector<void*> owned;
  Timer tm(ctx);
  struct Guard {
    cj_ctx* ctx;
    std::vector<void*>* v;
    ~Guard() {
      for (void* p : *v) ctx->release(p);
    }
  } guard{ctx, &owned};

  PhasePeaks peaks(ctx, res);
  if (opt->algo == CJ_NPHJ) {
    // No transform: the build relation is hashed as is (nphj.cu).
    if (hooks && hooks->before_side) {
      hooks->before_side(0);
      hooks->before_side(1);
    }
    tm.mark(0);
    tm.mark(1);
    res->peak_transform_b = peaks.next();
    OutSpec o;
    uint64_t cap = pk_fk ? S->rows : nphj_find(ctx, R->key, R->rows, S->key, S->rows, kb, o, 0, true);
    alloc_output(ctx, R, S, cap, true, res);
    o.key = res->key;
    o.ids_r = res->ids_r;
    o.ids_s = res->ids_s;
    if (!gfur) {  // GFTR: payload rows carried in the table / probe order
      o.nr = (int)R->npay;
      o.ns = (int)S->npay;
      for (uint32_t c = 0; c < R->npay; ++c) {
        o.r_src[c] = R->pay[c];
        o.r_dst[c] = res->pay[c];
        o.r_bytes[c] = R->pay_bytes[c];
      }
      for (uint32_t c = 0; c < S->npay; ++c) {
        o.s_src[c] = S->pay[c];
        o.s_dst[c] = res->pay[R->npay + c];
        o.s_bytes[c] = S->pay_bytes[c];
      }
    }
    uint64_t total;
    try {
      total = nphj_find(ctx, R->key, R->rows, S->key, S->rows, kb, o, cap, false, pk_fk);
    } catch (const Error& e) {
      if (e.code != CJ_ERR_CAPACITY_EXCEEDED || !pk_fk) throw;
      free_output(ctx, res);
      OutSpec oc;
      cap = nphj_find(ctx, R->key, R->rows, S->key, S->rows, kb, oc, 0, true);
      alloc_output(ctx, R, S, cap, true, res);
      o.key = res->key;
      o.ids_r = res->ids_r;
      o.ids_s = res->ids_s;
      for (uint32_t c = 0; c < R->npay && !gfur; ++c) o.r_dst[c] = res->pay[c];
      for (uint32_t c = 0; c < S->npay && !gfur; ++c) o.s_dst[c] = res->pay[R->npay + c];
      total = nphj_find(ctx, R->key, R->rows, S->key, S->rows, kb, o, cap, false);
    }
    tm.mark(2);
    res->peak_find_b = peaks.next();
    if (gfur) {
      const void* in[2 * CJ_MAX_COLS];
      void* out[2 * CJ_MAX_COLS];
      uint32_t by[2 * CJ_MAX_COLS];
      for (uint32_t c = 0; c < R->npay; ++c) {
        in[c] = R->pay[c];
        out[c] = res->pay[c];
        by[c] = R->pay_bytes[c];
      }
      gather_cols(ctx, in, R->rows, res->ids_r, total, out, by, (int)R->npay);
      for (uint32_t c = 0; c < S->npay; ++c) {
        in[c] = S->pay[c];
        out[c] = res->pay[R->npay + c];
        by[c] = S->pay_bytes[c];
      }
      gather_cols(ctx, in, S->rows, res->ids_s, total, out, by, (int)S->npay);
    }
    tm.mark(3);
    res->peak_materialize_b = peaks.next();
    res->device_bytes_peak =
        std::max({res->peak_transform_b, res->peak_find_b, res->peak_materialize_b});
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    raise_device_errors(ctx);
    res->rows = total;
    res->transform_ns = tm.ns(0, 1);
    res->find_ns = tm.ns(1, 2);
    res->materialize_ns = tm.ns(2, 3);
    if (opt->want_stats) {
      res->clusteredness_r = clusteredness(ctx, res->ids_r, total);
      res->clusteredness_s = clusteredness(ctx, res->ids_s, total);
    }
    if (!want_ids) {
      ctx->release(res->ids_r);
      ctx->release(res->ids_s);
      res->ids_r = res->ids_s = nullptr;
    }
    return;
  }

  // ---- transform ----------------------------------------------------------
  tm.mark(0);
  if (hooks && hooks->before_side) hooks->before_side(0);
  Side tr = transform(ctx, R, opt->algo, gfur, total_bits, opt->radix_bits_per_pass, owned,
                      presorted);
  if (hooks && hooks->before_side) hooks->before_side(1);
  Side ts = transform(ctx, S, opt->algo, gfur, total_bits, opt->radix_bits_per_pass, owned,
                      presorted);
  tm.mark(1);
  res->peak_transform_b = peaks.next();

  // ---- find (+ fused materialise for GFTR) ------------------------------------
  if (opt->algo == CJ_SMJ && opt->validate) {
    check_sorted(ctx, tr.keys, R->rows, kb, false, CJ_ERR_NOT_SORTED, "build");
    check_sorted(ctx, ts.keys, S->rows, kb, false, CJ_ERR_NOT_SORTED, "probe");
    if (pk_fk) check_sorted(ctx, tr.keys, R->rows, kb, true, CJ_ERR_DUPLICATE_BUILD_KEYS, "pk");
  }
  const uint32_t fanout = 1u << total_bits;
  auto count = [&]() -> uint64_t {
    if (opt->algo == CJ_SMJ) return smj_count(ctx, tr.keys, R->rows, ts.keys, S->rows, kb, pk_fk);
    return phj_count(ctx, tr.keys, tr.offsets, ts.keys, ts.offsets, fanout, kb,
                     opt->sub_partition_limit, tr.key_or);
  };
  // PK-FK: at most one match per probe row (sized without a count pass); a
  // mislabelled build with duplicates overflows and is re-run exactly.
  uint64_t cap = pk_fk ? S->rows : count();
  auto find = [&](uint64_t capacity) -> uint64_t {
    OutSpec o;
    o.key = res->key;
    o.ids_r = res->ids_r;
    o.ids_s = res->ids_s;
    o.padded = true;  // transformed columns carry kPad bytes of slack
    o.r_rows = R->rows;
    o.s_rows = S->rows;
    if (gfur) {
      // the physical ids carried through the transform are moved like a
      // payload column (staged by the find's bulk copies, written at the
      // output row) into ids_r / ids_s: resolve_ids (join_engine.cpp:37-45)
      o.ids_r = o.ids_s = nullptr;
      o.nr = o.ns = 1;
      o.r_src[0] = tr.cols[0];
      o.r_dst[0] = res->ids_r;
      o.r_bytes[0] = 4;
      o.s_src[0] = ts.cols[0];
      o.s_dst[0] = res->ids_s;
      o.s_bytes[0] = 4;
    } else {
      o.nr = (int)R->npay;
      o.ns = (int)S->npay;
      for (uint32_t c = 0; c < R->npay; ++c) {
        o.r_src[c] = tr.cols[c];
        o.r_dst[c] = res->pay[c];
        o.r_bytes[c] = R->pay_bytes[c];
      }
      for (uint32_t c = 0; c < S->npay; ++c) {
        o.s_src[c] = ts.cols[c];
        o.s_dst[c] = res->pay[R->npay + c];
        o.s_bytes[c] = S->pay_bytes[c];
      }
    }
    if (opt->algo == CJ_SMJ)
      return smj_find(ctx, tr.keys, R->rows, ts.keys, S->rows, kb, pk_fk, o, capacity);
    return phj_find(ctx, tr.keys, tr.offsets, ts.keys, ts.offsets, fanout, kb,
                    opt->sub_partition_limit, o, capacity, tr.key_or, pk_fk);
  };
  alloc_output(ctx, R, S, cap, want_ids || gfur, res);
  uint64_t total;
  try {
    total = find(cap);
  } catch (const Error& e) {
    if (e.code != CJ_ERR_CAPACITY_EXCEEDED || !pk_fk) throw;
    free_output(ctx, res);
    cap = count();
    alloc_output(ctx, R, S, cap, want_ids || gfur, res);
    total = find(cap);
  }
  if (ctx->timing) {  // algorithmic bytes of the find launch, now that |T| is known
    uint64_t rrow = kb, srow = kb, out_row = kb + (want_ids || gfur ? 8 : 0);
    if (!gfur) {
      for (uint32_t c = 0; c < R->npay; ++c) rrow += R->pay_bytes[c];
      for (uint32_t c = 0; c < S->npay; ++c) srow += S->pay_bytes[c];
      out_row += rrow + srow - 2 * kb;
    } else {  // the carried ids are read once, like a payload column
      rrow += 4;
      srow += 4;
    }
    const uint64_t b = rrow * R->rows + srow * S->rows + out_row * total;
    ctx->set_bytes(opt->algo == CJ_SMJ ? "smj_find" : "phj_find", b);
  }
  // the transformed sides are done with (GFTR's find wrote finished rows;
  // GFUR gathers from the untransformed relations): released at the end of
  // the find phase, as join_engine.cpp:330-335 frees the transformed keys and
  // ids
  for (void* p : owned) ctx->release(p);
  owned.clear();
  tm.mark(2);
  res->peak_find_b = peaks.next();

  // ---- materialise (GFUR: gathers from the untransformed relations) -------
  if (gfur) {
    const void* in[2 * CJ_MAX_COLS];
    void* out[2 * CJ_MAX_COLS];
    uint32_t by[2 * CJ_MAX_COLS];
    for (uint32_t c = 0; c < R->npay; ++c) {
      in[c] = R->pay[c];
      out[c] = res->pay[c];
      by[c] = R->pay_bytes[c];
    }
    gather_cols(ctx, in, R->rows, res->ids_r, total, out, by, (int)R->npay);
    for (uint32_t c = 0; c < S->npay; ++c) {
      in[c] = S->pay[c];
      out[c] = res->pay[R->npay + c];
      by[c] = S->pay_bytes[c];
    }
    gather_cols(ctx, in, S->rows, res->ids_s, total, out, by, (int)S->npay);
  }
  tm.mark(3);
  res->peak_materialize_b = peaks.next();
  res->device_bytes_peak =
      std::max({res->peak_transform_b, res->peak_find_b, res->peak_materialize_b});
  raise_device_errors(ctx);  // (one synchronisation: it reads the error word)
  res->rows = total;
  res->transform_ns = tm.ns(0, 1);
  res->find_ns = tm.ns(1, 2);
  res->materialize_ns = tm.ns(2, 3);
  if (opt->want_stats) {
    res->clusteredness_r = clusteredness(ctx, res->ids_r, total);
    res->clusteredness_s = clusteredness(ctx, res->ids_s, total);
  }
  if (!want_ids && res->ids_r) {
    ctx->release(res->ids_r);
    ctx->release(res->ids_s);
    res->ids_r = res->ids_s = nullptr;
  }
}

}  // namespace cj

// ---- cj_ctx -------------------------------------------------------------------

void* cj_ctx::alloc(uint64_t bytes, int cls, uint64_t logical) {
  void* p = nullptr;
  cj::check_cuda(cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, pool, stream), "cudaMallocAsync");
  if (logical == ~0ull) logical = bytes;
  live_sizes[p] = LiveAlloc{bytes, logical, cls};
  live += bytes;
  live_peak = std::max(live_peak, live);
  if (cls != kOutputData) {
    ledger[cls] += logical;
    if (ledger[0] + ledger[1] > ledger_peak[0] + ledger_peak[1]) ledger_reset_peak();
  }
  return p;
}

void cj_ctx::release(void* p) {
  if (!p) return;
  auto it = live_sizes.find(p);
  if (it != live_sizes.end()) {
    live -= it->second.bytes;
    if (it->second.cls != kOutputData) ledger[it->second.cls] -= it->second.logical;
    live_sizes.erase(it);
  }
  cudaFreeAsync(p, stream);
}

uint16_t cj_ctx::next_epoch() {
  if (epoch == 0xffff) {  // wrap: clear old generations
    epoch = 0;
    if (status) cj::check_cuda(cudaMemsetAsync(status, 0, status_words * 8, stream), "memset");
  }
  return ++epoch;
}

void cj_ctx::reserve(uint64_t bytes) {
  if (bytes <= pool_reserved) return;
  const uint64_t want = bytes + bytes / 4;
  void* p = nullptr;
  if (cudaMallocFromPoolAsync(&p, want, pool, stream) != cudaSuccess) {
    cudaGetLastError();  // not enough memory for one block: allocate as we go
    pool_reserved = bytes;
    return;
  }
  cj::check_cuda(cudaFreeAsync(p, stream), "cudaFreeAsync");
  pool_reserved = want;
}

uint64_t* cj_ctx::status_buffer(uint64_t words) {
  if (words > status_words) {
    if (status) cudaFreeAsync(status, stream);
    const uint64_t w = std::max<uint64_t>(words + words / 4, 1 << 16);
    status = static_cast<uint64_t*>(alloc(w * 8));
    cj::check_cuda(cudaMemsetAsync(status, 0, w * 8, stream), "memset status");
    status_words = w;
  }
  return status;
}

cudaEvent_t cj_ctx::take_event() {
  if (ev_used == ev_pool.size()) {
    cudaEvent_t e;
    cj::check_cuda(cudaEventCreate(&e), "cudaEventCreate");
    ev_pool.push_back(e);
  }
  return ev_pool[ev_used++];
}

void cj_ctx::kbegin(const char* name, uint64_t alg_bytes) {
  ++launches;
  if (!timing) return;
  KernelRec r{name, take_event(), take_event(), alg_bytes};
  cj::check_cuda(cudaEventRecord(r.a, stream), "cudaEventRecord");
  recs.push_back(r);
}

void cj_ctx::kend() {
  if (!timing || recs.empty()) return;
  cj::check_cuda(cudaEventRecord(recs.back().b, stream), "cudaEventRecord");
}

void cj_ctx::set_bytes(const char* name, uint64_t bytes) {
  for (size_t i = recs.size(); i-- > 0;)
    if (std::strcmp(recs[i].name, name) == 0) {
      recs[i].bytes = bytes;
      return;
    }
}

uint32_t* cj_ctx::ticket(int slot) {
  cj::check_cuda(cudaMemsetAsync(counters + slot, 0, sizeof(uint32_t), stream), "memset ticket");
  return counters + slot;
}

// ---- C ABI --------------------------------------------------------------------

extern "C" {

void* cj_ctx_stream(const cj_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int cj_ctx_create(int device, void* stream, cj_ctx** out) {
  if (!out) return CJ_ERR_SPEC_INVALID;
  *out = nullptr;
  cj_ctx* ctx = new cj_ctx();
  const int st = cj::guarded(ctx, [&] {
    int ndev = 0;
    CJ_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) cj::fail(CJ_ERR_CUDA, "no such CUDA device");
    CJ_CUDA(cudaSetDevice(device));
    ctx->device = device;
    CJ_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    if (stream) {
      ctx->stream = static_cast<cudaStream_t>(stream);
    } else {
      CJ_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
    }
    // a pool per ctx: concurrent ctxs (one per host thread / stream) never
    // contend for, or fragment, each other's reserved memory
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    CJ_CUDA(cudaMemPoolCreate(&ctx->pool, &props));
    uint64_t thr = UINT64_MAX;
    CJ_CUDA(cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // Optional up-front reservation (GiB) of the stream-ordered pool, so the
    // join's multi-GiB scratch never maps new memory inside a timed call.
    if (const char* rg = std::getenv("CJ_POOL_RESERVE_GB")) {
      const uint64_t bytes = (uint64_t)std::strtoull(rg, nullptr, 10) << 30;
      if (bytes) {
        void* p = nullptr;
        CJ_CUDA(cudaMallocFromPoolAsync(&p, bytes, ctx->pool, ctx->stream));
        CJ_CUDA(cudaFreeAsync(p, ctx->stream));
      }
    }
    ctx->counters = static_cast<uint32_t*>(ctx->alloc(256 * sizeof(uint32_t)));
    CJ_CUDA(cudaMemsetAsync(ctx->counters, 0, 256 * sizeof(uint32_t), ctx->stream));
    ctx->err_word = ctx->counters + 128;
    CJ_CUDA(cudaMallocHost(&ctx->host_pinned, 1 << 16));
    for (auto& e : ctx->marks) CJ_CUDA(cudaEventCreate(&e));
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
  if (st != CJ_OK) {
    std::fprintf(stderr, "cj_ctx_create: %s\n", ctx->last_error.c_str());
    delete ctx;
    return st;
  }
  *out = ctx;
  return CJ_OK;
}

int cj_ctx_destroy(cj_ctx* ctx) {
  if (!ctx) return CJ_OK;
  cudaStreamSynchronize(ctx->stream);
  if (ctx->status) cudaFreeAsync(ctx->status, ctx->stream);
  if (ctx->counters) cudaFreeAsync(ctx->counters, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto& e : ctx->marks)
    if (e) cudaEventDestroy(e);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  // released once the caller has freed every result column it still holds
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
  delete ctx;
  return CJ_OK;
}

const char* cj_last_error(const cj_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "no ctx"; }

int cj_sync(cj_ctx* ctx) {
  return cj::guarded(ctx, [&] { CJ_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int cj_free(cj_ctx* ctx, void* p) {
  return cj::guarded(ctx, [&] { ctx->release(p); });
}

int cj_alloc(cj_ctx* ctx, uint64_t bytes, void** p) {
  return cj::guarded(ctx, [&] { *p = ctx->alloc(bytes); });
}

uint64_t cj_launch_count(const cj_ctx* ctx) { return ctx ? ctx->launches : 0; }

uint64_t cj_scratch_peak(cj_ctx* ctx, int reset) {
  if (!ctx) return 0;
  const uint64_t p = ctx->scratch_peak;
  if (reset) ctx->scratch_peak = ctx->scratch_now;
  return p;
}

int cj_copy(cj_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind) {
  return cj::guarded(ctx, [&] {
    if (bytes == 0) return;
    const cudaMemcpyKind k = kind == 1   ? cudaMemcpyHostToDevice
                             : kind == 2 ? cudaMemcpyDeviceToHost
                                         : cudaMemcpyDeviceToDevice;
    CJ_CUDA(cudaMemcpyAsync(dst, src, bytes, k, ctx->stream));
    if (kind != 3) CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int cj_mark(cj_ctx* ctx, int slot) {
  return cj::guarded(ctx, [&] {
    if (slot < 0 || slot >= 16) cj::fail(CJ_ERR_SPEC_INVALID, "mark slot out of range");
    CJ_CUDA(cudaEventRecord(ctx->marks[slot], ctx->stream));
  });
}

int cj_elapsed_ms(cj_ctx* ctx, int a, int b, float* ms) {
  return cj::guarded(ctx, [&] {
    if (a < 0 || a >= 16 || b < 0 || b >= 16) cj::fail(CJ_ERR_SPEC_INVALID, "mark slot");
    CJ_CUDA(cudaEventElapsedTime(ms, ctx->marks[a], ctx->marks[b]));
  });
}

int cj_set_kernel_timing(cj_ctx* ctx, int on) {
  return cj::guarded(ctx, [&] {
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->timing = on != 0;
    ctx->recs.clear();
    ctx->ev_used = 0;
  });
}

int cj_kernel_records(cj_ctx* ctx, int max, const char** names, float* ms, uint64_t* bytes,
                      int* count) {
  return cj::guarded(ctx, [&] {
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    const int n = (int)std::min<size_t>(ctx->recs.size(), (size_t)std::max(max, 0));
    for (int i = 0; i < n; ++i) {
      const auto& r = ctx->recs[i];
      names[i] = r.name;
      CJ_CUDA(cudaEventElapsedTime(&ms[i], r.a, r.b));
      bytes[i] = r.bytes;
    }
    *count = (int)ctx->recs.size();
  });
}

int cj_histogram(cj_ctx* ctx, const void* keys, uint64_t n, uint32_t kb, uint32_t lo,
                 uint32_t hi, uint32_t* counts_host) {
  return cj::guarded(ctx, [&] {
    cj::check_key_bytes(kb);
    if (hi < lo || hi - lo > 8) cj::fail(CJ_ERR_FANOUT_TOO_LARGE, "radix pass limited to 8 bits (256 partitions)");
    if (hi > kb * 8) cj::fail(CJ_ERR_FANOUT_TOO_LARGE, "bit range exceeds key width");
    cj::PassPlan plan;
    plan.npasses = 1;
    plan.lo[0] = lo;
    plan.hi[0] = hi;
    cj::ValCols none;
    const cj::ScatterGeom g = cj::scatter_geom(ctx, n, (int)kb, none, keys);
    cj::Scratch cnt(ctx, 4ull * cj::kRadix * g.nblocks), tot(ctx, 4 * cj::kRadix),
        base(ctx, 8 * cj::kRadix);
    std::vector<uint32_t> h;
    cj::histogram_passes(ctx, keys, n, (int)kb, plan, g, cnt.as<uint32_t>(), tot.as<uint32_t>(),
                         base.as<uint64_t>(), &h);
    std::memcpy(counts_host, h.data(), sizeof(uint32_t) * (1u << (hi - lo)));
  });
}

static cj::ValCols make_vals(const void* const* in, void* const* out, const uint32_t* bytes,
                             uint32_t n, int gen_ids) {
  if (n > CJ_MAX_COLS + 1) cj::fail(CJ_ERR_UNSUPPORTED, "too many value columns");
  cj::ValCols v;
  v.n = (int)n;
  v.gen_ids = gen_ids;
  for (uint32_t c = 0; c < n; ++c) {
    v.in[c] = in ? in[c] : nullptr;
    v.out[c] = out[c];
    v.bytes[c] = bytes[c];
    if (bytes[c] != 4 && bytes[c] != 8) cj::fail(CJ_ERR_KIND, "value columns must be 4 or 8 bytes");
  }
  if (gen_ids && (n == 0 || bytes[0] != 4)) cj::fail(CJ_ERR_KIND, "generated ids are u32");
  return v;
}

int cj_radix_partition(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, uint32_t kb,
                       uint32_t lo, uint32_t hi, const void* const* vin, void* const* vout,
                       const uint32_t* vbytes, uint32_t nvals, uint64_t* offsets_host) {
  return cj::guarded(ctx, [&] {
    cj::check_key_bytes(kb);
    if (hi < lo || hi - lo > 8) cj::fail(CJ_ERR_FANOUT_TOO_LARGE, "radix pass limited to 8 bits (256 partitions)");
    if (hi > kb * 8) cj::fail(CJ_ERR_FANOUT_TOO_LARGE, "bit range exceeds key width");
    cj::ValCols v = make_vals(vin, vout, vbytes, nvals, 0);
    if (lo == hi) {  // fan-out 1 = identity (primitives.cpp:300-305)
      cj::copy_columns(ctx, keys, keys_out, n, (int)kb, v);
      if (offsets_host) {
        offsets_host[0] = 0;
        offsets_host[1] = n;
      }
      CJ_CUDA(cudaStreamSynchronize(ctx->stream));
      return;
    }
    cj::PassPlan plan;
    plan.npasses = 1;
    plan.lo[0] = lo;
    plan.hi[0] = hi;
    const cj::ScatterGeom g = cj::scatter_geom(ctx, n, (int)kb, v, keys);
    cj::Scratch cnt(ctx, 4ull * cj::kRadix * g.nblocks), tot(ctx, 4 * cj::kRadix),
        base(ctx, 8 * cj::kRadix);
    std::vector<uint32_t> h;
    cj::histogram_passes(ctx, keys, n, (int)kb, plan, g, cnt.as<uint32_t>(), tot.as<uint32_t>(),
                         base.as<uint64_t>(), &h);
    cj::scatter_pass(ctx, keys, keys_out, n, (int)kb, lo, hi, base.as<uint64_t>(),
                     cnt.as<uint32_t>(), cj::kRadix, g, v);
    if (offsets_host) {
      const uint32_t fan = 1u << (hi - lo);
      offsets_host[0] = 0;
      for (uint32_t d = 0; d < fan; ++d) offsets_host[d + 1] = offsets_host[d] + h[d];
    }
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int cj_radix_partition_passes(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n,
                              uint32_t kb, const uint32_t* plan_lo, const uint32_t* plan_hi,
                              uint32_t npasses, const void* const* vin, void* const* vout,
                              const uint32_t* vbytes, uint32_t nvals, int gen_ids) {
  return cj::guarded(ctx, [&] {
    cj::check_key_bytes(kb);
    if (npasses > 64) cj::fail(CJ_ERR_UNSUPPORTED, "plan longer than 64 passes");
    cj::PassPlan plan;
    plan.npasses = (int)npasses;
    for (uint32_t p = 0; p < npasses; ++p) {
      if (plan_hi[p] < plan_lo[p] || plan_hi[p] - plan_lo[p] > 8)
        cj::fail(CJ_ERR_FANOUT_TOO_LARGE, "radix pass limited to 8 bits (256 partitions)");
      if (plan_hi[p] > kb * 8) cj::fail(CJ_ERR_FANOUT_TOO_LARGE, "bit range exceeds key width");
      plan.lo[p] = plan_lo[p];
      plan.hi[p] = plan_hi[p];
    }
    cj::ValCols v = make_vals(vin, vout, vbytes, nvals, gen_ids);
    cj::lsd_any(ctx, keys, keys_out, n, (int)kb, plan, v);
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int cj_sort_pairs(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, uint32_t kb,
                  const void* const* vin, void* const* vout, const uint32_t* vbytes,
                  uint32_t nvals, int gen_ids) {
  return cj::guarded(ctx, [&] {
    cj::check_key_bytes(kb);
    cj::ValCols v = make_vals(vin, vout, vbytes, nvals, gen_ids);
    cj::lsd_partition(ctx, keys, keys_out, n, (int)kb, cj::sort_plan(ctx, keys, n, (int)kb, v), v);
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int cj_gather(cj_ctx* ctx, const void* const* in, uint64_t n_in, const uint32_t* map,
              uint64_t m, void* const* out, const uint32_t* bytes, uint32_t ncols) {
  return cj::guarded(ctx, [&] {
    for (uint32_t c = 0; c < ncols; ++c)
      if (bytes[c] != 4 && bytes[c] != 8) cj::fail(CJ_ERR_KIND, "gather columns must be 4 or 8 bytes");
    cj::gather_cols(ctx, in, n_in, map, m, out, bytes, (int)ncols);
    cj::raise_device_errors(ctx);
  });
}

int cj_partition_relation(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, uint32_t kb,
                          uint32_t total_bits, uint32_t bits_per_pass, const void* const* vin,
                          void* const* vout, const uint32_t* vbytes, uint32_t nvals, int gen_ids,
                          uint64_t* offsets_dev) {
  return cj::guarded(ctx, [&] {
    cj::check_key_bytes(kb);
    if (total_bits > 20) cj::fail(CJ_ERR_FANOUT_TOO_LARGE, "partition fan-out capped at 2^20");
    if (total_bits > kb * 8) cj::fail(CJ_ERR_FANOUT_TOO_LARGE, "partition bits exceed key width");
    cj::ValCols v = make_vals(vin, vout, vbytes, nvals, gen_ids);
    if (total_bits == 0) {
      cj::copy_columns(ctx, keys, keys_out, n, (int)kb, v);
    } else {
      cj::lsd_any(ctx, keys, keys_out, n, (int)kb, cj::plan_bits(total_bits, bits_per_pass), v);
    }
    cj::partition_offsets(ctx, keys_out, n, (int)kb, total_bits, offsets_dev);
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int cj_hash_find_matches(cj_ctx* ctx, const cj_partitioned* b, const cj_partitioned* p,
                         uint32_t fanout, uint32_t kb, uint32_t limit, int id_mode,
                         uint64_t* total_host, void** keys_out, uint32_t** ids_r_out,
                         uint32_t** ids_s_out) {
  return cj::guarded(ctx, [&] {
    cj::check_key_bytes(kb);
    const bool phys = id_mode == CJ_IDS_PHYSICAL;
    if (phys && (!b->carried || !p->carried))
      cj::fail(CJ_ERR_UNSUPPORTED, "physical id mode needs carried id columns on both sides");
    const uint64_t total = cj::phj_count(ctx, b->keys, b->offsets, p->keys, p->offsets, fanout,
                                         (int)kb, limit);
    void* k = ctx->alloc(std::max<uint64_t>(total, 1) * kb);
    uint32_t* ir = static_cast<uint32_t*>(ctx->alloc(std::max<uint64_t>(total, 1) * 4));
    uint32_t* is = static_cast<uint32_t*>(ctx->alloc(std::max<uint64_t>(total, 1) * 4));
    cj::OutSpec o;
    o.key = k;
    o.ids_r = ir;
    o.ids_s = is;
    if (phys) {
      o.carried_r = b->carried;
      o.carried_s = p->carried;
    }
    cj::phj_find(ctx, b->keys, b->offsets, p->keys, p->offsets, fanout, (int)kb, limit, o, total);
    *total_host = total;
    *keys_out = k;
    *ids_r_out = ir;
    *ids_s_out = is;
  });
}

int cj_merge_find_matches(cj_ctx* ctx, const void* r, uint64_t nr, const void* s, uint64_t ns,
                          uint32_t kb, int pk_fk, int validate, uint64_t* total_host,
                          void** keys_out, uint32_t** ids_r_out, uint32_t** ids_s_out) {
  return cj::guarded(ctx, [&] {
    cj::check_key_bytes(kb);
    if (validate) {
      cj::check_sorted(ctx, r, nr, (int)kb, false, CJ_ERR_NOT_SORTED, "build");
      cj::check_sorted(ctx, s, ns, (int)kb, false, CJ_ERR_NOT_SORTED, "probe");
      if (pk_fk) cj::check_sorted(ctx, r, nr, (int)kb, true, CJ_ERR_DUPLICATE_BUILD_KEYS, "pk");
    }
    const uint64_t total = cj::smj_count(ctx, r, nr, s, ns, (int)kb, pk_fk != 0);
    void* k = ctx->alloc(std::max<uint64_t>(total, 1) * kb);
    uint32_t* ir = static_cast<uint32_t*>(ctx->alloc(std::max<uint64_t>(total, 1) * 4));
    uint32_t* is = static_cast<uint32_t*>(ctx->alloc(std::max<uint64_t>(total, 1) * 4));
    cj::OutSpec o;
    o.key = k;
    o.ids_r = ir;
    o.ids_s = is;
    cj::smj_find(ctx, r, nr, s, ns, (int)kb, pk_fk != 0, o, total);
    *total_host = total;
    *keys_out = k;
    *ids_r_out = ir;
    *ids_s_out = is;
  });
}

void cj_default_options(cj_join_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->algo = CJ_PHJ;
  o->pattern = CJ_GFTR;
  o->radix_bits_per_pass = 8;
  o->total_radix_bits = -1;
  o->sub_partition_limit = 4096;
}

int cj_run_join(cj_ctx* ctx, const cj_relation* build, const cj_relation* probe,
                const cj_join_options* opt, cj_join_result* res) {
  return cj::guarded(ctx, [&] {
    try {
      cj::run_join_dev(ctx, build, probe, opt, res);
    } catch (...) {
      cj::free_output(ctx, res);
      throw;
    }
  });
}

int cj_run_join_presorted(cj_ctx* ctx, const cj_relation* build, const cj_relation* probe,
                          const cj_join_options* opt, uint32_t presorted_bits,
                          cj_join_result* res) {
  return cj::guarded(ctx, [&] {
    cj::JoinHooks h;
    h.presorted_bits = presorted_bits;
    try {
      cj::run_join_dev(ctx, build, probe, opt, res, &h);
    } catch (...) {
      cj::free_output(ctx, res);
      throw;
    }
  });
}

int cj_run_join_sequence(cj_ctx* ctx, const cj_relation* fact, const cj_relation* dims,
                         uint32_t n_dims, const cj_join_options* opt, cj_sequence_step* steps,
                         cj_join_result* last) {
  return cj::guarded(ctx, [&] {
    if (!fact || !dims || !opt || !steps) cj::fail(CJ_ERR_SPEC_INVALID, "null argument");
    if (n_dims == 0) return;
    if (fact->npay < n_dims) cj::fail(CJ_ERR_SPEC_INVALID, "fact table needs one FK column per dimension");
    if (fact->key_bytes != 4) cj::fail(CJ_ERR_SPEC_INVALID, "fact tuple ids must be a 4-byte column");
    // buffers the chain owns (intermediate outputs), released when unused
    std::vector<void*> owned;
    auto release = [&](void* p) {
      for (auto& q : owned)
        if (q == p) {
          ctx->release(p);
          q = nullptr;
        }
    };
    struct Guard {
      cj_ctx* c;
      std::vector<void*>* v;
      ~Guard() {
        for (void* p : *v)
          if (p) c->release(p);
      }
    } guard{ctx, &owned};
    // probe for join 1: (FK_1, ID)  (sequence.cpp:23-27).  GFTR: the later FK
    // columns ride along as trailing probe payloads (nfk of them), so each
    // join's output already holds the next join's FK column in output order —
    // the reference's FK fetch gather (sequence.cpp:43-55) yields the same
    // values, and a carried column costs the transform's sequential bytes
    // instead of a random gather over the fact table.
    cj_relation probe{};
    probe.key = fact->pay[0];
    probe.key_bytes = fact->pay_bytes[0];
    probe.rows = fact->rows;
    probe.npay = 1;
    probe.pay[0] = fact->key;
    probe.pay_bytes[0] = 4;
    probe.key_unique = 0;
    const bool carry = opt->pattern == CJ_GFTR && n_dims > 1 && n_dims <= CJ_MAX_COLS;
    uint32_t nfk = 0;
    if (carry)
      for (uint32_t d = 1; d < n_dims; ++d, ++nfk) {
        probe.pay[probe.npay] = fact->pay[d];
        probe.pay_bytes[probe.npay++] = fact->pay_bytes[d];
      }
    cudaEvent_t e0, e1;
    CJ_CUDA(cudaEventCreate(&e0));
    CJ_CUDA(cudaEventCreate(&e1));
    for (uint32_t i = 0; i < n_dims; ++i) {
      cj_join_result res{};
      cj::run_join_dev(ctx, &dims[i], &probe, opt, &res);
      cj_sequence_step& st = steps[i];
      st.rows = res.rows;
      st.output_columns = 1 + dims[i].npay + probe.npay - nfk;
      st.transform_ns = res.transform_ns;
      st.find_ns = res.find_ns;
      st.materialize_ns = res.materialize_ns;
      st.fk_fetch_ns = 0;
      // the probe's own columns (this chain's, not the caller's) are consumed
      if (i > 0) {
        release(const_cast<void*>(probe.key));
        for (uint32_t c = 0; c < probe.npay; ++c) release(const_cast<void*>(probe.pay[c]));
      }
      if (i + 1 == n_dims) {
        if (last) *last = res;
        else cj::free_output(ctx, &res);
        break;
      }
      // output payloads are build-side first: (P_i, ID, P_1..P_{i-1}); the
      // next probe is (FK_{i+1}, ID, P_1..P_i)  (sequence.cpp:38-62)
      const uint32_t dim_pay = dims[i].npay;
      const uint32_t kept = probe.npay - nfk;  // (ID, P_1..P_{i-1})
      void* next_fk;
      if (nfk) {  // carried: output column dim_pay + kept is FK_{i+1}
        next_fk = res.pay[dim_pay + kept];
        owned.push_back(next_fk);
      } else {
        const uint32_t* ids = static_cast<const uint32_t*>(res.pay[dim_pay]);
        next_fk = ctx->alloc(std::max<uint64_t>(res.rows * fact->pay_bytes[i + 1], 16) + cj::kPad);
        owned.push_back(next_fk);
        CJ_CUDA(cudaEventRecord(e0, ctx->stream));
        const void* in[1] = {fact->pay[i + 1]};
        void* out[1] = {next_fk};
        const uint32_t by[1] = {fact->pay_bytes[i + 1]};
        cj::gather_cols(ctx, in, fact->rows, ids, res.rows, out, by, 1);
        CJ_CUDA(cudaEventRecord(e1, ctx->stream));
        CJ_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        CJ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        st.fk_fetch_ns = static_cast<uint64_t>(ms * 1e6);
        cj::raise_device_errors(ctx);
      }
      cj_relation np{};
      np.key = next_fk;
      np.key_bytes = fact->pay_bytes[i + 1];
      np.rows = res.rows;
      np.key_unique = 0;
      if (dim_pay + probe.npay > CJ_MAX_COLS)
        cj::fail(CJ_ERR_UNSUPPORTED, "too many carried payload columns");
      // next probe payloads: (ID, P_1..P_{i-1}), P_i, then the FKs still to come
      uint32_t k = 0;
      auto take = [&](uint32_t c, uint32_t bytes) {
        np.pay[k] = res.pay[c];
        np.pay_bytes[k++] = bytes;
        owned.push_back(res.pay[c]);
      };
      for (uint32_t c = 0; c < kept; ++c) take(dim_pay + c, probe.pay_bytes[c]);
      for (uint32_t c = 0; c < dim_pay; ++c) take(c, dims[i].pay_bytes[c]);
      for (uint32_t c = kept + 1; c < probe.npay; ++c) take(dim_pay + c, probe.pay_bytes[c]);
      np.npay = k;
      if (nfk) --nfk;
      ctx->release(res.key);  // the FK key column of the output is not carried
      if (res.ids_r) ctx->release(res.ids_r);
      if (res.ids_s) ctx->release(res.ids_s);
      probe = np;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

int cj_gen_star(cj_ctx* ctx, uint64_t fact_rows, uint32_t dims, uint64_t dim_rows, uint64_t seed,
                uint32_t key_bytes, uint32_t pay_bytes, void* fact_ids, void* const* fks,
                void* const* dim_keys, void* const* dim_pays) {
  return cj::guarded(ctx, [&] {
    cj::gen_star(ctx, fact_rows, dims, dim_rows, seed, key_bytes, pay_bytes, fact_ids, fks,
                 dim_keys, dim_pays);
  });
}

int cj_result_free(cj_ctx* ctx, cj_join_result* res) {
  return cj::guarded(ctx, [&] { cj::free_output(ctx, res); });
}

namespace {
// Host-buffer joins running concurrently on one device (one ctx per host
// thread) take turns per copy direction: two uploads at once only halve each
// other's PCIe bandwidth, while an upload next to a download uses both
// directions of the link.  One lock per direction and device.
std::mutex g_h2d_mu[16], g_d2h_mu[16];
}  // namespace

int cj_run_join_host(cj_ctx* ctx, const cj_relation* build, const cj_relation* probe,
                     const cj_join_options* opt, cj_host_alloc_fn alloc, void* user,
                     cj_join_result* out, uint64_t* h2d_ns, uint64_t* d2h_ns) {
  return cj::guarded(ctx, [&] {
    std::mutex& h2d_mu = g_h2d_mu[ctx->device & 15];
    std::mutex& d2h_mu = g_d2h_mu[ctx->device & 15];
    cj::validate_relation(build, "a build relation");
    cj::validate_relation(probe, "a probe relation");
    std::vector<void*> owned;
    struct G {
      cj_ctx* c;
      std::vector<void*>* v;
      ~G() {
        for (void* p : *v) c->release(p);
      }
    } g{ctx, &owned};
    cj::Timer tm(ctx);
    auto up = [&](const cj_relation* h, cj_relation* d) {
      *d = *h;
      void* k = ctx->alloc(std::max<uint64_t>(h->rows * h->key_bytes, 16));
      owned.push_back(k);
      if (h->rows)
        CJ_CUDA(cudaMemcpyAsync(k, h->key, h->rows * h->key_bytes, cudaMemcpyHostToDevice,
                                ctx->stream));
      d->key = k;
      for (uint32_t c = 0; c < h->npay; ++c) {
        void* p = ctx->alloc(std::max<uint64_t>(h->rows * h->pay_bytes[c], 16));
        owned.push_back(p);
        if (h->rows)
          CJ_CUDA(cudaMemcpyAsync(p, h->pay[c], h->rows * h->pay_bytes[c],
                                  cudaMemcpyHostToDevice, ctx->stream));
        d->pay[c] = p;
      }
    };
    cj_relation R, S;
    {
      std::lock_guard<std::mutex> lk(h2d_mu);
      tm.mark(0);
      up(build, &R);
      up(probe, &S);
      tm.mark(1);
      CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    cj_join_result dres;
    std::memset(&dres, 0, sizeof(dres));
    cj::run_join_dev(ctx, &R, &S, opt, &dres);
    struct RG {
      cj_ctx* c;
      cj_join_result* r;
      ~RG() { cj::free_output(c, r); }
    } rg{ctx, &dres};
    *out = dres;
    const uint64_t t = dres.rows;
    std::lock_guard<std::mutex> lk(d2h_mu);
    tm.mark(2);
    auto down = [&](const void* src, uint64_t bytes) -> void* {
      void* h = alloc(std::max<uint64_t>(bytes, 1), user);
      if (!h) cj::fail(CJ_ERR_OUT_OF_MEMORY, "host output allocation failed");
      if (bytes) CJ_CUDA(cudaMemcpyAsync(h, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      return h;
    };
    out->key = down(dres.key, t * build->key_bytes);
    for (uint32_t c = 0; c < build->npay; ++c)
      out->pay[c] = down(dres.pay[c], t * build->pay_bytes[c]);
    for (uint32_t c = 0; c < probe->npay; ++c)
      out->pay[build->npay + c] = down(dres.pay[build->npay + c], t * probe->pay_bytes[c]);
    out->ids_r = dres.ids_r ? static_cast<uint32_t*>(down(dres.ids_r, t * 4)) : nullptr;
    out->ids_s = dres.ids_s ? static_cast<uint32_t*>(down(dres.ids_s, t * 4)) : nullptr;
    tm.mark(3);
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h2d_ns) *h2d_ns = tm.ns(0, 1);
    if (d2h_ns) *d2h_ns = tm.ns(2, 3);
  });
}

int cj_shard_partition(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, uint32_t kb,
                       uint32_t parts, const void* const* vin, void* const* vout,
                       const uint32_t* vbytes, uint32_t nvals, uint64_t* counts_host) {
  return cj::guarded(ctx, [&] {
    cj::check_key_bytes(kb);
    cj::ValCols v = make_vals(vin, vout, vbytes, nvals, 0);
    cj::shard_partition(ctx, keys, keys_out, n, (int)kb, parts, 0, v, counts_host);
  });
}

int cj_shard_partition_ex(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, uint32_t kb,
                          uint32_t parts, uint32_t first_bits, const void* const* vin,
                          void* const* vout, const uint32_t* vbytes, uint32_t nvals,
                          uint64_t* counts_host) {
  return cj::guarded(ctx, [&] {
    cj::check_key_bytes(kb);
    cj::ValCols v = make_vals(vin, vout, vbytes, nvals, 0);
    cj::shard_partition(ctx, keys, keys_out, n, (int)kb, parts, first_bits, v, counts_host);
  });
}

int cj_gen_shard(cj_ctx* ctx, uint64_t r_total, uint64_t s_total, uint32_t rank, uint32_t ranks,
                 uint32_t r_pay, uint32_t s_pay, uint64_t seed, void* r_key, void* const* r_pays,
                 void* s_key, void* const* s_pays) {
  return cj::guarded(ctx, [&] {
    cj::gen_shard(ctx, r_total, s_total, rank, ranks, r_pay, s_pay, seed, r_key, r_pays, s_key,
                  s_pays);
  });
}

int cj_gen_pk_fk(cj_ctx* ctx, uint64_t r_rows, uint64_t s_rows, uint32_t r_pay, uint32_t s_pay,
                 uint32_t key_bytes, uint32_t pay_bytes, double match_ratio, double zipf,
                 uint64_t seed, void* r_key, void* const* r_pays, void* s_key,
                 void* const* s_pays) {
  return cj::guarded(ctx, [&] {
    cj::gen_pk_fk(ctx, r_rows, s_rows, r_pay, s_pay, key_bytes, pay_bytes, match_ratio, zipf,
                  seed, r_key, r_pays, s_key, s_pays);
  });
}

}  // extern "C"
