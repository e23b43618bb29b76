// Internal declarations shared by the .cu translation units of
// libcoljoin_b200.so.  Not part of the public boundary (include/cj_api.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <new>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "cj_api.h"

namespace cj {

constexpr int kRadix = 256;  // digits per pass (<= 8 bits, primitives.cpp:15)

// A status error carrying a cj_status; converted at the C boundary.
struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
#define CJ_CUDA(x) ::cj::check_cuda((x), #x)

}  // namespace cj

struct cj_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaMemPool_t pool = nullptr;   // stream-ordered allocations of this ctx
  uint16_t epoch = 0;             // look-back status generation (see radix.cu)
  uint64_t launches = 0;          // kernels launched through this ctx
  uint64_t scratch_now = 0, scratch_peak = 0;  // device scratch held by operators
  // every live alloc() of this ctx, for run_join's per-phase peaks: device
  // bytes, and the MemLedger view (mem_ledger.hpp:26-100) — the logical bytes
  // of column-sized working data vs scratch; the output relation is neither
  enum : int { kScratchData = 0, kColumnData = 1, kOutputData = 2 };
  struct LiveAlloc {
    uint64_t bytes, logical;
    int cls;
  };
  std::unordered_map<void*, LiveAlloc> live_sizes;
  uint64_t live = 0, live_peak = 0;
  uint64_t ledger[2] = {0, 0};        // live logical scratch / column bytes
  uint64_t ledger_peak[2] = {0, 0};   // both, at the high-water mark of their sum
  std::string last_error;
  // persistent scratch (grown on demand, never shrunk)
  uint64_t* status = nullptr;     // decoupled look-back words
  uint64_t status_words = 0;
  uint32_t* counters = nullptr;   // tile / unit tickets, error word
  uint32_t* err_word = nullptr;   // device error flags (OOB, overflow)
  uint32_t* host_pinned = nullptr;// small pinned staging (4 KiB)
  cudaEvent_t marks[16] = {};
  // per-launch timing records (cj_set_kernel_timing): event pairs around each
  // kernel on the ctx stream, with the launch's algorithmic bytes
  struct KernelRec {
    const char* name;
    cudaEvent_t a, b;
    uint64_t bytes;
  };
  bool timing = false;
  std::vector<KernelRec> recs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t take_event();
  void kbegin(const char* name, uint64_t alg_bytes);  // before a launch
  void kend();                                       // after it
  void set_bytes(const char* name, uint64_t bytes);  // fix up the last record of `name`

  // cls: kScratchData / kColumnData / kOutputData; logical = the bytes the
  // ledger counts (default `bytes`; padded columns pass their unpadded size)
  void* alloc(uint64_t bytes, int cls = kScratchData, uint64_t logical = ~0ull);
  void ledger_reset_peak() {
    ledger_peak[0] = ledger[0];
    ledger_peak[1] = ledger[1];
  }
  void release(void* p);
  uint16_t next_epoch();          // fresh look-back generation (memsets on wrap)
  uint64_t* status_buffer(uint64_t words);
  uint32_t* ticket(int slot);     // zeroed device counter (slot < 64)
  // Grow the stream-ordered pool to hold `bytes` at once (one mapping), so a
  // join's scratch never maps new memory mid-call (multi-ms stalls otherwise).
  uint64_t pool_reserved = 0;
  void reserve(uint64_t bytes);
  // run_join's transforms: run every LSD pass without the constant-digit host
  // round trip (a constant pass is a stable copy; skipping it only saves time)
  bool assume_live_passes = false;
  // set by a caller that synchronised and read a zero error word: the next
  // raise_device_errors returns without another round trip
  bool err_known_clean = false;
};

namespace cj {

// Scoped device scratch released on the ctx stream at scope exit.
struct Scratch {
  cj_ctx* ctx;
  void* p = nullptr;
  uint64_t n = 0;
  Scratch(cj_ctx* c, uint64_t bytes) : ctx(c), p(c->alloc(bytes ? bytes : 16)), n(bytes) {
    c->scratch_now += n;
    if (c->scratch_now > c->scratch_peak) c->scratch_peak = c->scratch_now;
  }
  ~Scratch() {
    if (p) ctx->release(p);
    ctx->scratch_now -= n;
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// ---- radix.cu ---------------------------------------------------------------
struct ValCols {
  int n = 0;
  const void* in[CJ_MAX_COLS + 1] = {};
  void* out[CJ_MAX_COLS + 1] = {};
  uint32_t bytes[CJ_MAX_COLS + 1] = {};
  int gen_ids = 0;   // column 0 generated as the source index (u32)
};

struct PassPlan {
  int npasses = 0;
  uint32_t lo[64] = {}, hi[64] = {};
  int done = 0;  // leading passes the input already went through (a presorted
                 // input: the sharded join's receivers get rows grouped by the
                 // first digit); skipped, the rest run as usual
};

// Geometry of a blocked scatter pass: tile size (shared-memory budget), tile
// count, one static block of consecutive tiles per CTA, stage layout.
struct ScatterGeom {
  int items = 8;
  uint64_t tile = 4096, tiles = 1;
  uint32_t nblocks = 1;
  size_t smem = 0;
  uint32_t stage_bytes = 0, pbytes = 0;
  uint32_t voff[CJ_MAX_COLS + 1] = {};
  bool tma = false;  // all inputs 16-byte aligned (TMA bulk copies)
  int ctas_per_sm = 2, stages = 2;
  int rank = 0;      // in-warp peer search: 0 atomic-OR masks, 1 ballots
  int rb = 8;        // digit bits of the passes (8, or 9 for wide full-width sorts)
  int threads = 512; // per CTA (256: two CTAs per SM)
};
ScatterGeom scatter_geom(cj_ctx* ctx, uint64_t n, int key_bytes, const ValCols& vals,
                         const void* keys_in, int rb = 8);

// Per-block digit counts (cnt[b][p][256]) of every pass of `plan` (<= 8) in one
// read of the keys, over the blocks of geometry g.
// With totals_dev / base_dev, the last CTA also writes the digit totals and
// exclusive bases of every pass (no separate launch).
void block_hist(cj_ctx* ctx, const void* keys, uint64_t n, int key_bytes, const PassPlan& plan,
                const ScatterGeom& g, uint32_t* cnt_dev, uint32_t hparts = 0,
                uint32_t lowbits = 0, unsigned long long* key_or = nullptr,
                uint32_t* totals_dev = nullptr, uint64_t* base_dev = nullptr);

// block_hist + digit totals (totals_dev[p*256+d]) + exclusive digit bases
// (base_dev[p*256+d]); totals_host after one host round trip when non-null.
void histogram_passes(cj_ctx* ctx, const void* keys, uint64_t n, int key_bytes,
                      const PassPlan& plan, const ScatterGeom& g, uint32_t* cnt_dev,
                      uint32_t* totals_dev, uint64_t* base_dev,
                      std::vector<uint32_t>* totals_host, uint32_t hparts = 0,
                      uint32_t lowbits = 0, unsigned long long* key_or = nullptr);

// One stable scatter pass.  With per-block counts of this pass (cnt, stride
// cnt_stride) and a TMA-eligible geometry it runs the blocked kernel (no
// inter-CTA waiting); otherwise the onesweep kernel with decoupled look-back.
void scatter_pass(cj_ctx* ctx, const void* keys_in, void* keys_out, uint64_t n, int key_bytes,
                  uint32_t lo, uint32_t hi, const uint64_t* base_dev, const uint32_t* cnt,
                  uint32_t cnt_stride, const ScatterGeom& g, const ValCols& vals,
                  uint32_t hparts = 0, uint32_t lowbits = 0, int runs = 0);

// Stable partition of rows by digit = shard << lowbits | (key & (2^lowbits - 1)),
// shard = floor(mix64(key) * parts / 2^64) (the multi-GPU shuffle's send
// layout: by destination, then by the receiver's first LSD digit);
// counts_host[parts << lowbits] rows per digit.
void shard_partition(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int key_bytes,
                     uint32_t parts, uint32_t lowbits, const ValCols& vals, uint64_t* counts_host);

// Stable LSD over the plan; constant-digit passes skipped; the last executed
// pass lands in the caller's outputs.  gen_ids handled in the first pass.
void lsd_partition(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int key_bytes,
                   const PassPlan& plan, const ValCols& vals,
                   std::vector<uint32_t>* counts_host = nullptr,
                   unsigned long long* key_or = nullptr);

// Layout offsets (fanout + 1) of keys sorted by their low `bits`: binary search
// of every boundary.
void partition_offsets(cj_ctx* ctx, const void* keys_sorted, uint64_t n, int key_bytes,
                       uint32_t bits, uint64_t* offsets_dev);

void copy_columns(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int key_bytes,
                  const ValCols& vals);

// Plan of a stable full-width sort over the keys' significant bits (8- or
// 9-bit digits, whichever needs fewer passes).
PassPlan sort_plan(cj_ctx* ctx, const void* keys, uint64_t n, int key_bytes, const ValCols& vals);

// Stable LSD over a plan of any length (segments of CJ_MAX_PASSES passes), engine.cu.
void lsd_any(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int kb,
             const PassPlan& plan, const ValCols& vals, unsigned long long* key_or = nullptr);

// ---- gather.cu ----------------------------------------------------------------
void gather_cols(cj_ctx* ctx, const void* const* in, uint64_t n_in, const uint32_t* map,
                 uint64_t m, void* const* out, const uint32_t* bytes, int ncols);

// ---- join kernels ---------------------------------------------------------------
struct OutSpec {
  void* key = nullptr;             // K[]
  uint32_t* ids_r = nullptr;       // u32[]
  uint32_t* ids_s = nullptr;
  const uint32_t* carried_r = nullptr;  // physical ids: ids_r = carried_r[i]
  const uint32_t* carried_s = nullptr;
  int nr = 0, ns = 0;              // fused payload columns per side
  const void* r_src[CJ_MAX_COLS] = {};
  const void* s_src[CJ_MAX_COLS] = {};
  void* r_dst[CJ_MAX_COLS] = {};
  void* s_dst[CJ_MAX_COLS] = {};
  uint32_t r_bytes[CJ_MAX_COLS] = {};
  uint32_t s_bytes[CJ_MAX_COLS] = {};
  bool padded = false;             // keys + src columns readable 16 B past the end (TMA path)
  uint64_t r_rows = 0, s_rows = 0; // input sizes (timing records only)
};

// Allocation slack that keeps 16-byte-aligned bulk copies of any row range
// inside the allocation.
constexpr uint64_t kPad = 64;

// hash_join.cu: partitioned hash join (count + look-back + fill), outputs per
// OutSpec; capacity = rows the outputs can hold (CJ_ERR_CAPACITY_EXCEEDED
// beyond).  Returns the match count (one host sync).
// key_or (optional, device): OR of the build keys; when (OR >> log2 fanout)
// is below a unit's table size the unit uses a direct-addressed table.
uint64_t phj_find(cj_ctx* ctx, const void* bkeys, const uint64_t* boff, const void* pkeys,
                  const uint64_t* poff, uint32_t fanout, int key_bytes, uint32_t limit,
                  const OutSpec& out, uint64_t capacity,
                  const unsigned long long* key_or = nullptr, bool pk_fk = false);
// Match count only (for sizing outputs), plus optional per-reference-unit counts.
uint64_t phj_count(cj_ctx* ctx, const void* bkeys, const uint64_t* boff, const void* pkeys,
                   const uint64_t* poff, uint32_t fanout, int key_bytes, uint32_t limit,
                   const unsigned long long* key_or = nullptr);

// merge_join.cu: merge join over sorted keys; same contract.
uint64_t smj_find(cj_ctx* ctx, const void* rkeys, uint64_t nr, const void* skeys, uint64_t ns,
                  int key_bytes, bool pk_fk, const OutSpec& out, uint64_t capacity);
uint64_t smj_count(cj_ctx* ctx, const void* rkeys, uint64_t nr, const void* skeys, uint64_t ns,
                   int key_bytes, bool pk_fk);
void check_sorted(cj_ctx* ctx, const void* keys, uint64_t n, int key_bytes, bool strict,
                  int err_code, const char* what);

// nphj.cu: non-partitioned (global table) hash join.
uint64_t nphj_find(cj_ctx* ctx, const void* rkeys, uint64_t nr, const void* skeys, uint64_t ns,
                   int key_bytes, const OutSpec& out, uint64_t capacity, bool count_only,
                   bool unique = false);

// gen.cu
void gen_pk_fk(cj_ctx* ctx, uint64_t r_rows, uint64_t s_rows, uint32_t r_pay, uint32_t s_pay,
               uint32_t key_bytes, uint32_t pay_bytes, double match_ratio, double zipf,
               uint64_t seed, void* r_key, void* const* r_pays, void* s_key, void* const* s_pays);

// Exclusive scan of n u64 counts on the ctx stream; *total_dev = sum.
void scan_counts(cj_ctx* ctx, const uint64_t* in, uint64_t n, uint64_t* out, uint64_t* total_dev);

void gen_star(cj_ctx* ctx, uint64_t fact_rows, uint32_t dims, uint64_t dim_rows, uint64_t seed,
              uint32_t key_bytes, uint32_t pay_bytes, void* fact_ids, void* const* fks,
              void* const* dim_keys, void* const* dim_pays);

void gen_shard(cj_ctx* ctx, uint64_t r_total, uint64_t s_total, uint32_t rank, uint32_t ranks,
               uint32_t r_pay, uint32_t s_pay, uint64_t seed, void* r_key, void* const* r_pays,
               void* s_key, void* const* s_pays);

// ---- engine.cu ------------------------------------------------------------------
// Optional hooks of run_join_dev (the sharded join's receivers).
struct JoinHooks {
  // both sides arrive stably grouped by their low `presorted_bits` key bits:
  // the transform skips that first LSD pass
  unsigned presorted_bits = 0;
  // called (host side) before side 0 (build) / 1 (probe) is first read on the
  // ctx stream: the sharded join makes the stream wait for that side's exchange
  std::function<void(int)> before_side;
};
void run_join_dev(cj_ctx* ctx, const cj_relation* R, const cj_relation* S,
                  const cj_join_options* opt, cj_join_result* res,
                  const JoinHooks* hooks = nullptr);
void alloc_output(cj_ctx* ctx, const cj_relation* r, const cj_relation* s, uint64_t cap,
                  bool ids, cj_join_result* res);
void free_output(cj_ctx* ctx, cj_join_result* res);
unsigned default_total_radix_bits(uint64_t build_rows);
void validate_relation(const cj_relation* r, const char* what);

// Runs fn, mapping exceptions to status codes (the C boundary).
template <class F>
int guarded(cj_ctx* ctx, F&& fn) {
  try {
    fn();
    return CJ_OK;
  } catch (const Error& e) {
    if (ctx) ctx->last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->last_error = "host allocation failed";
    return CJ_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_error = e.what();
    return CJ_ERR_CUDA;
  }
}

// error word helpers: kernels OR codes into ctx->err_word; raise after sync
enum : uint32_t { kErrOOB = 1u, kErrOverflow = 2u, kErrNotSorted = 4u, kErrDupKeys = 8u };
void raise_device_errors(cj_ctx* ctx);

inline unsigned grid_for(uint64_t work, unsigned per_block, unsigned cap) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g > cap ? cap : g);
}

}  // namespace cj
