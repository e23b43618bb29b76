// Partitioned hash join find phase (K4), optionally fused with GFTR
// materialisation.
//
// Reference semantics (paths relative to the reference's proj/):
//   plan_subpartitions   hash_match.cpp:186-210  (build chunks of <= limit rows)
//   ChunkTable/scan_unit hash_match.cpp:73-121   (equal keys in insertion order)
//   hash_match_count     hash_match.cpp:212-248
//   hash_match_fill      hash_match.cpp:250-302  (order: unit, probe pos, build pos)
//
// Design (B200): work units are (partition, build chunk, probe chunk);
// splitting the probe side keeps a Zipf hot partition spread over many CTAs
// while the concatenation in unit order is exactly the reference's emission
// order.  Two implementations:
//  - run_join's path (inputs padded for bulk copies): k_phj_tma, a count pass
//    -> scan of the unit counts -> fill pass.  Each persistent CTA has a
//    producer warp that stages units (descriptor, bulk copies) and 16
//    consumer warps; the count pass builds a 16-bit open-addressing table of
//    chunk positions with CAS (duplicate keys detected exactly during
//    insertion), probes, and hands every probe row's match index to the fill,
//    which then needs neither the table nor the build keys;
//  - the operator API on arbitrary buffers: k_phj_find, one pass whose units
//    chain their output offsets by warp-cooperative decoupled look-back.
// Chunks holding duplicate keys switch to a stably sorted chunk (bitonic over
// (key, pos)) so every probe emits its matches in build insertion order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "cj_device.cuh"
#include "cj_internal.cuh"

namespace cj {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
// Probe rows per work unit; the unit sequence (partition, build chunk, probe
// chunk) concatenates to the reference's emission order for any chunk size.
uint32_t probe_chunk() {
  const char* e = std::getenv("CJ_QCHUNK");
  return e ? (uint32_t)std::max(256, std::min(16384, std::atoi(e))) : 4096u;
}
int find_ctas_per_sm() {
  const char* e = std::getenv("CJ_FIND_CTAS");
  return e ? std::max(1, std::atoi(e)) : 1;
}
int find_stages() {
  const char* e = std::getenv("CJ_FIND_STAGES");
  return e ? std::min(2, std::max(1, std::atoi(e))) : 2;
}
constexpr uint16_t kEmpty16 = 0xffffu;
constexpr uint32_t kNoMatch = 0xffffffffu;

// unit_start[p] = number of units before partition p (units with an empty
// side produce no rows and are dropped).  Grid-wide: each block scans 1024
// partitions and chains its total by decoupled look-back.
constexpr int kPlanThreads = 256, kPlanPer = 4;

struct PlanArgs2 {
  const uint64_t* boff;
  const uint64_t* poff;
  uint32_t fanout, limit, qchunk;
  uint64_t* unit_start;     // fanout + 1
  unsigned long long* stats;// [0] max build chunk (atomicMax), [1] total units
  uint64_t* status;
  uint64_t epoch;
  uint32_t* err;
};

__global__ void __launch_bounds__(kPlanThreads) k_phj_plan(const __grid_constant__ PlanArgs2 a) {
  __shared__ uint64_t wsum[kPlanThreads / 32];
  __shared__ uint64_t s_base;
  const uint32_t p0 = (blockIdx.x * kPlanThreads + threadIdx.x) * kPlanPer;
  uint64_t cnt[kPlanPer];
  uint64_t local = 0, maxc = 0;
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    const uint32_t p = p0 + i;
    cnt[i] = 0;
    if (p < a.fanout) {
      const uint64_t nb = a.boff[p + 1] - a.boff[p], ns = a.poff[p + 1] - a.poff[p];
      if (nb && ns) {
        cnt[i] = ((nb + a.limit - 1) / a.limit) * ((ns + a.qchunk - 1) / a.qchunk);
        maxc = max(maxc, dev::umin64(nb, a.limit));
      }
    }
    local += cnt[i];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t inc = dev::warp_inclusive_sum(local);
  if (lane == 31) wsum[warp] = inc;
  for (int o = 16; o > 0; o >>= 1) maxc = max(maxc, __shfl_xor_sync(0xffffffffu, maxc, o));
  if (lane == 0 && maxc) atomicMax(&a.stats[0], (unsigned long long)maxc);
  __syncthreads();
  if (warp == 0) {
    uint64_t v = lane < kPlanThreads / 32 ? wsum[lane] : 0;
    const uint64_t tot = dev::warp_sum(v);
    const uint64_t base = dev::warp_lookback(a.status, blockIdx.x, tot, a.epoch, a.err);
    if (lane == 0) {
      s_base = base;
      if (blockIdx.x == gridDim.x - 1) {
        a.unit_start[a.fanout] = base + tot;
        a.stats[1] = base + tot;
      }
    }
  }
  __syncthreads();
  uint64_t off = s_base;
  for (int w = 0; w < warp; ++w) off += wsum[w];
  uint64_t run = off + inc - local;
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    const uint32_t p = p0 + i;
    if (p < a.fanout) a.unit_start[p] = run;
    run += cnt[i];
  }
}

struct FindArgs {
  const void* bkeys;
  const uint64_t* boff;
  const void* pkeys;
  const uint64_t* poff;
  uint32_t fanout, limit, qchunk, cap_log2, max_chunk;
  const uint64_t* unit_start;
  uint64_t* status;
  uint64_t epoch;
  uint32_t* ticket;
  uint32_t* err;
  uint64_t capacity;
  int write;                 // 0: count only
  uint64_t* total_out;       // written by the last unit
  uint64_t* unit_counts;     // optional per-unit counts
  // outputs
  void* key_out;
  uint32_t* ids_r;
  uint32_t* ids_s;
  const uint32_t* carried_r;
  const uint32_t* carried_s;
  int nr, ns, stage_r;
  const void* r_src[CJ_MAX_COLS];
  const void* s_src[CJ_MAX_COLS];
  void* r_dst[CJ_MAX_COLS];
  void* s_dst[CJ_MAX_COLS];
  uint32_t r_bytes[CJ_MAX_COLS];
  uint32_t s_bytes[CJ_MAX_COLS];
  uint32_t r_stage_off[CJ_MAX_COLS];  // byte offsets of staged columns
  // TMA path: stage layout (byte offsets within one stage buffer)
  uint32_t stage_bytes, off_bk, off_pk, cap_entries;
  uint32_t off_r[CJ_MAX_COLS], off_s[CJ_MAX_COLS];
  int padded;  // every staged array is readable 16 bytes past its end
  // count / fill passes
  const void* desc;          // UnitDesc[n_units]
  uint64_t n_units;
  uint64_t* unit_off;        // exclusive output offset per unit (fill)
  uint64_t nb_rows, np_rows; // sizes of the partitioned inputs
  int stages;                // 2: prefetch the next unit while this one runs
  // count pass -> fill pass hand-off: build-chunk index of every probe row's
  // match (0xffff: none) and a per-unit duplicate flag; fill units without
  // duplicates then skip the table build and the probe entirely
  uint16_t* match_e;
  uint8_t* unit_dup;
  uint32_t off_e;            // stage offset of the match_e chunk
  int blocked;               // CTAs walk contiguous unit ranges (else round robin)
  uint32_t group;            // round robin over groups of this many consecutive units
  // dense build keys: OR of the build keys (device); a unit whose table holds
  // (OR >> dense_shift) + 1 slots addresses it directly by key >> dense_shift
  // (the partition fixes the low dense_shift bits, so a unique key owns its
  // slot: plain stores, one load per probe)
  const unsigned long long* key_or;
  uint32_t dense_shift;
  // speculative PK-FK fill (no count pass): every unit expects each probe row
  // to match once and writes at its probe offset; a unit that finds a miss or
  // a duplicate build key sets *spec_fail, later units stop, and the caller
  // runs count + fill
  uint32_t* spec_fail;
  uint32_t* spec_rows;  // probe rows of the units that matched completely (coverage check:
                        // partitions without build rows have no units)
};

// Multiplicative (Fibonacci) hashing as the reference's ChunkTable
// (hash_match.cpp:24-26); the slot never affects the output (unique chunks
// match exactly one entry, duplicate chunks are matched through their sorted
// positions), so 4-byte keys take the 32-bit product (log2cap <= 15).
template <class K>
__device__ __forceinline__ uint32_t slot_of(K k, uint32_t log2cap) {
  if constexpr (sizeof(K) == 4) return ((uint32_t)k * 0x9E3779B1u) >> (32 - log2cap);
  return (uint32_t)(((uint64_t)k * 0x9E3779B97F4A7C15ull) >> (64 - log2cap));
}

template <class K>
__device__ __forceinline__ void emit_row(const FindArgs& a, uint64_t o, uint64_t gi, uint32_t li,
                                         uint64_t j, K k, const uint8_t* rstage) {
  if (a.key_out) static_cast<K*>(a.key_out)[o] = k;
  if (a.ids_r) a.ids_r[o] = a.carried_r ? a.carried_r[gi] : (uint32_t)gi;
  if (a.ids_s) a.ids_s[o] = a.carried_s ? a.carried_s[j] : (uint32_t)j;
  for (int c = 0; c < a.nr; ++c) {
    if (a.r_bytes[c] == 4) {
      const uint32_t v = a.stage_r ? reinterpret_cast<const uint32_t*>(rstage + a.r_stage_off[c])[li]
                                   : static_cast<const uint32_t*>(a.r_src[c])[gi];
      static_cast<uint32_t*>(a.r_dst[c])[o] = v;
    } else {
      const uint64_t v = a.stage_r ? reinterpret_cast<const uint64_t*>(rstage + a.r_stage_off[c])[li]
                                   : static_cast<const uint64_t*>(a.r_src[c])[gi];
      static_cast<uint64_t*>(a.r_dst[c])[o] = v;
    }
  }
  for (int c = 0; c < a.ns; ++c) {
    if (a.s_bytes[c] == 4)
      static_cast<uint32_t*>(a.s_dst[c])[o] = __ldcs(static_cast<const uint32_t*>(a.s_src[c]) + j);
    else
      static_cast<uint64_t*>(a.s_dst[c])[o] = __ldcs(static_cast<const uint64_t*>(a.s_src[c]) + j);
  }
}

template <class K>
__global__ void __launch_bounds__(kThreads) k_phj_find(const __grid_constant__ FindArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t s_unit, s_b_lo, s_b_hi, s_q_lo, s_q_hi, s_base;
  __shared__ uint64_t s_wcount[kWarps], s_wbase[kWarps];
  __shared__ int s_dup;

  // shared layout: [bk: max_chunk K][table: 2^cap u16][res: qchunk u32][rstage]
  K* bk = reinterpret_cast<K*>(smem);
  uint16_t* tab = reinterpret_cast<uint16_t*>(smem + (size_t)a.max_chunk * sizeof(K));
  uint32_t* res = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(tab) +
                                              ((size_t)2 << a.cap_log2));
  uint8_t* rstage = reinterpret_cast<uint8_t*>(res) + (size_t)a.qchunk * 4;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t total_units = a.unit_start[a.fanout];
  const K* __restrict__ bkeys = static_cast<const K*>(a.bkeys);
  const K* __restrict__ pkeys = static_cast<const K*>(a.pkeys);

  while (true) {
    if (tid == 0) {
      const uint64_t u = atomicAdd(a.ticket, 1u);
      s_unit = u;
      if (u < total_units) {
        // partition p: unit_start[p] <= u < unit_start[p + 1]
        uint32_t lo = 0, hi = a.fanout;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (a.unit_start[mid] <= u) lo = mid; else hi = mid;
        }
        const uint32_t p = lo;
        const uint64_t b0 = a.boff[p], b1 = a.boff[p + 1], q0 = a.poff[p], q1 = a.poff[p + 1];
        const uint64_t nqc = (q1 - q0 + a.qchunk - 1) / a.qchunk;
        const uint64_t local = u - a.unit_start[p];
        const uint64_t c = local / nqc, q = local % nqc;
        s_b_lo = b0 + c * a.limit;
        s_b_hi = min(b1, s_b_lo + a.limit);
        s_q_lo = q0 + q * a.qchunk;
        s_q_hi = min(q1, s_q_lo + a.qchunk);
      }
      s_dup = 0;
    }
    __syncthreads();
    const uint64_t u = s_unit;
    if (u >= total_units) break;
    const uint64_t b_lo = s_b_lo, q_lo = s_q_lo;
    const uint32_t nb = (uint32_t)(s_b_hi - b_lo), nq = (uint32_t)(s_q_hi - q_lo);
    const uint32_t cap_log2 = nb <= 1 ? 1u : 33u - (uint32_t)__clz(nb - 1);
    const uint32_t cap = 1u << cap_log2, cmask = cap - 1;

    // 1. stage build keys (+ transformed R payloads) and clear the table
    for (uint32_t i = tid; i < nb; i += kThreads) bk[i] = bkeys[b_lo + i];
    for (uint32_t s = tid; s < cap; s += kThreads) tab[s] = kEmpty16;
    if (a.write && a.stage_r) {
      for (int c = 0; c < a.nr; ++c) {
        if (a.r_bytes[c] == 4) {
          const uint32_t* src = static_cast<const uint32_t*>(a.r_src[c]) + b_lo;
          uint32_t* dst = reinterpret_cast<uint32_t*>(rstage + a.r_stage_off[c]);
          for (uint32_t i = tid; i < nb; i += kThreads) dst[i] = src[i];
        } else {
          const uint64_t* src = static_cast<const uint64_t*>(a.r_src[c]) + b_lo;
          uint64_t* dst = reinterpret_cast<uint64_t*>(rstage + a.r_stage_off[c]);
          for (uint32_t i = tid; i < nb; i += kThreads) dst[i] = src[i];
        }
      }
    }
    __syncthreads();

    // 2. insert chunk positions; an equal key met on the way marks duplicates
    bool dup = false;
    for (uint32_t i = tid; i < nb; i += kThreads) {
      const K k = bk[i];
      uint32_t s = slot_of(k, cap_log2);
      while (true) {
        const uint16_t old = atomicCAS(&tab[s], kEmpty16, (uint16_t)i);
        if (old == kEmpty16) break;
        if (bk[old] == k) dup = true;
        s = (s + 1) & cmask;
      }
    }
    if (__syncthreads_or(dup)) s_dup = 1;
    __syncthreads();
    const bool has_dup = s_dup != 0;

    // 3. probe: warp w owns a contiguous run of 32-row rounds
    const uint32_t rounds = (nq + 31) / 32;
    const uint32_t r0 = (uint32_t)((uint64_t)rounds * warp / kWarps);
    const uint32_t r1 = (uint32_t)((uint64_t)rounds * (warp + 1) / kWarps);
    uint16_t* sidx = tab;  // duplicate path: stably sorted chunk positions
    if (has_dup) {
      // bitonic sort of chunk positions by (key, position)
      uint32_t np2 = 1;
      while (np2 < nb) np2 <<= 1;
      for (uint32_t i = tid; i < np2; i += kThreads) sidx[i] = i < nb ? (uint16_t)i : kEmpty16;
      __syncthreads();
      for (uint32_t kk = 2; kk <= np2; kk <<= 1) {
        for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
          for (uint32_t i = tid; i < np2; i += kThreads) {
            const uint32_t l = i ^ jj;
            if (l > i) {
              const uint16_t x = sidx[i], y = sidx[l];
              // sentinel (0xffff) sorts last
              bool gt;
              if (x == kEmpty16) gt = y != kEmpty16;
              else if (y == kEmpty16) gt = false;
              else gt = bk[x] > bk[y] || (bk[x] == bk[y] && x > y);
              const bool up = (i & kk) == 0;
              if (gt == up) { sidx[i] = y; sidx[l] = x; }
            }
          }
          __syncthreads();
        }
      }
    }
    uint64_t wcount = 0;
    for (uint32_t r = r0; r < r1; ++r) {
      const uint32_t jl = r * 32 + lane;
      uint32_t out = kNoMatch;
      uint32_t m = 0;
      if (jl < nq) {
        const K k = pkeys[q_lo + jl];
        if (!has_dup) {
          uint32_t s = slot_of(k, cap_log2);
          while (true) {
            const uint16_t e = tab[s];
            if (e == kEmpty16) break;
            if (bk[e] == k) { out = e; m = 1; break; }
            s = (s + 1) & cmask;
          }
        } else {
          uint32_t lo = 0, hi = nb;  // lower_bound
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (bk[sidx[mid]] < k) lo = mid + 1; else hi = mid;
          }
          uint32_t lo2 = lo, hi2 = nb;  // upper_bound
          while (lo2 < hi2) {
            const uint32_t mid = (lo2 + hi2) >> 1;
            if (bk[sidx[mid]] <= k) lo2 = mid + 1; else hi2 = mid;
          }
          m = lo2 - lo;
          out = (lo << 16) | m;
        }
        res[jl] = out;
      }
      wcount += m;
    }
    wcount = dev::warp_sum(wcount);
    if (lane == 0) s_wcount[warp] = wcount;
    __syncthreads();

    // 4. unit total -> look-back -> unit output base
    if (warp == 0) {
      uint64_t wc = lane < kWarps ? s_wcount[lane] : 0;
      const uint64_t inc = dev::warp_inclusive_sum(wc);
      if (lane < kWarps) s_wbase[lane] = inc - wc;
      const uint64_t unit_total = __shfl_sync(0xffffffffu, inc, kWarps - 1);
      const uint64_t base = dev::warp_lookback(a.status, u, unit_total, a.epoch, a.err);
      if (lane == 0) {
        s_base = base;
        if (a.unit_counts) a.unit_counts[u] = unit_total;
        if (u == total_units - 1) *a.total_out = base + unit_total;
        if (a.write && base + unit_total > a.capacity) atomicOr(a.err, kErrOverflow);
      }
    }
    __syncthreads();

    // 5. emit in probe order
    if (a.write) {
      uint64_t o = s_base + s_wbase[warp];
      for (uint32_t r = r0; r < r1; ++r) {
        const uint32_t jl = r * 32 + lane;
        const uint32_t e = jl < nq ? res[jl] : kNoMatch;
        const uint64_t j = q_lo + jl;
        if (!has_dup) {
          const bool hit = e != kNoMatch;
          const uint32_t bal = __ballot_sync(0xffffffffu, hit);
          if (hit) {
            const uint64_t oo = o + __popc(bal & dev::lanemask_lt());
            if (oo < a.capacity) emit_row<K>(a, oo, b_lo + e, e, j, bk[e], rstage);
          }
          o += __popc(bal);
        } else {
          const uint32_t m = e == kNoMatch ? 0 : (e & 0xffffu);
          const uint32_t lb = e >> 16;
          const uint32_t inc = dev::warp_inclusive_sum(m);
          uint64_t oo = o + inc - m;
          for (uint32_t t = 0; t < m; ++t, ++oo) {
            const uint32_t li = sidx[lb + t];
            if (oo < a.capacity) emit_row<K>(a, oo, b_lo + li, li, j, bk[li], rstage);
          }
          o += __shfl_sync(0xffffffffu, inc, 31);
        }
      }
    }
    __syncthreads();
  }
}

// ---- TMA-pipelined count / fill (the default for run_join) -------------------
//
// No inter-CTA waiting: a count pass writes every unit's match count, a scan
// turns them into output offsets, and the fill pass writes each unit's rows at
// its offset.  Both passes are persistent (one CTA of 512 threads per SM, unit
// u_k = blockIdx + k * gridDim) and double-buffered: a unit's build chunk (keys
// + transformed R payload slices) and probe chunk (keys + transformed S payload
// slices) are contiguous ranges, bulk-copied (cp.async.bulk, 16-byte aligned
// supersets of the ranges) into one shared-memory stage while the previous
// unit is built, probed and written from the other.  Unit descriptors are
// precomputed, so the next unit's copies are issued without a dependent lookup.
constexpr int kTmaThreads = 512;
constexpr int kTmaWarps = kTmaThreads / 32;

struct UnitDesc {
  uint64_t b_lo, b_hi, q_lo, q_hi;
  uint32_t split;  // the partition holds more build rows than the limit (several build chunks)
};

// One thread per unit: its partition by binary search over unit_start (a
// skewed partition may own millions of units; a thread per partition would
// write them serially).
__global__ void k_phj_desc(const uint64_t* __restrict__ boff, const uint64_t* __restrict__ poff,
                           const uint64_t* __restrict__ unit_start, uint32_t fanout,
                           uint32_t limit, uint32_t qchunk, uint64_t units,
                           UnitDesc* __restrict__ desc) {
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units;
       u += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = fanout;  // last p with unit_start[p] <= u
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (unit_start[mid] <= u) lo = mid; else hi = mid;
    }
    const uint32_t p = lo;
    const uint64_t l = u - unit_start[p];
    const uint64_t b0 = boff[p], b1 = boff[p + 1], q0 = poff[p], q1 = poff[p + 1];
    const uint64_t nqc = (q1 - q0 + qchunk - 1) / qchunk;
    UnitDesc d;
    d.b_lo = b0 + (l / nqc) * limit;
    d.b_hi = dev::umin64(b1, d.b_lo + limit);
    d.q_lo = q0 + (l % nqc) * qchunk;
    d.q_hi = dev::umin64(q1, d.q_lo + qchunk);
    d.split = b1 - b0 > limit ? 1u : 0u;
    desc[u] = d;
  }
}

// Rows [0, cnt) of a unit's output at ubase, column by column, consecutive
// threads on consecutive output rows: row t is (build idx, probe idx) =
// (me[t] or res[t], t) when ident, else list[t] = build idx << 16 | probe idx.
template <class K>
__device__ __forceinline__ void emit_rows(const FindArgs& a, const UnitDesc& inf,
                                          const uint8_t* st, const K* pk, const uint16_t* me,
                                          const uint32_t* res, const uint32_t* list,
                                          uint64_t ubase, uint32_t cnt, bool ident) {
  const int tid = threadIdx.x;
  const uint32_t bsh4 = (uint32_t)(inf.b_lo & 3), bsh8 = (uint32_t)(inf.b_lo & 1);
  const uint32_t qsh4 = (uint32_t)(inf.q_lo & 3), qsh8 = (uint32_t)(inf.q_lo & 1);
  // 3b. column by column, consecutive threads write consecutive output rows
  if (ubase + cnt > a.capacity) cnt = ubase < a.capacity ? (uint32_t)(a.capacity - ubase) : 0u;
  constexpr int kE = 8;
  for (uint32_t t0 = 0; t0 < cnt; t0 += kE * kTmaThreads) {
    uint32_t L[kE];
#pragma unroll
    for (int k = 0; k < kE; ++k) {
      const uint32_t t = t0 + tid + k * kTmaThreads;
      L[k] = t < cnt ? (ident ? ((me ? (uint32_t)me[t] : res[t]) << 16) | t : list[t]) : 0u;
    }
    auto each = [&](auto&& f) {
#pragma unroll
      for (int k = 0; k < kE; ++k) {
        const uint32_t t = t0 + tid + k * kTmaThreads;
        if (t < cnt) f(ubase + t, L[k] >> 16, L[k] & 0xffffu);
      }
    };
    if (a.key_out) {
      K* ko = static_cast<K*>(a.key_out);
      each([&](uint64_t oo, uint32_t, uint32_t jl) { ko[oo] = pk[jl]; });
    }
    if (a.ids_r)
      each([&](uint64_t oo, uint32_t li, uint32_t) {
        const uint64_t gi = inf.b_lo + li;
        a.ids_r[oo] = a.carried_r ? a.carried_r[gi] : (uint32_t)gi;
      });
    if (a.ids_s)
      each([&](uint64_t oo, uint32_t, uint32_t jl) {
        const uint64_t j = inf.q_lo + jl;
        a.ids_s[oo] = a.carried_s ? a.carried_s[j] : (uint32_t)j;
      });
    for (int c = 0; c < a.nr; ++c) {
      if (a.r_bytes[c] == 4) {
        const uint32_t* sv = reinterpret_cast<const uint32_t*>(st + a.off_r[c]) + bsh4;
        uint32_t* dv = static_cast<uint32_t*>(a.r_dst[c]);
        each([&](uint64_t oo, uint32_t li, uint32_t) { dv[oo] = sv[li]; });
      } else {
        const uint64_t* sv = reinterpret_cast<const uint64_t*>(st + a.off_r[c]) + bsh8;
        uint64_t* dv = static_cast<uint64_t*>(a.r_dst[c]);
        each([&](uint64_t oo, uint32_t li, uint32_t) { dv[oo] = sv[li]; });
      }
    }
    for (int c = 0; c < a.ns; ++c) {
      if (a.s_bytes[c] == 4) {
        const uint32_t* sv = reinterpret_cast<const uint32_t*>(st + a.off_s[c]) + qsh4;
        uint32_t* dv = static_cast<uint32_t*>(a.s_dst[c]);
        each([&](uint64_t oo, uint32_t, uint32_t jl) { dv[oo] = sv[jl]; });
      } else {
        const uint64_t* sv = reinterpret_cast<const uint64_t*>(st + a.off_s[c]) + qsh8;
        uint64_t* dv = static_cast<uint64_t*>(a.s_dst[c]);
        each([&](uint64_t oo, uint32_t, uint32_t jl) { dv[oo] = sv[jl]; });
      }
    }
  }
}

// GFTR/GFUR emission of a unit without duplicate build keys: compact the hits
// in probe order (list[t] = build idx << 16 | probe idx), then emit_rows.  The
// match of probe row jl is me[jl] (0xffff: none) when the count pass resolved
// it, else res[jl].
template <class K>
__device__ __forceinline__ void emit_compact(const FindArgs& a, const UnitDesc& inf,
                                             const uint8_t* st, const K* pk, const uint16_t* me,
                                             const uint32_t* res, uint32_t r0, uint32_t r1,
                                             uint32_t nq, const uint64_t* s_wbase,
                                             const uint64_t* s_wcount, uint32_t* list) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t ubase = s_wbase[0];
  uint32_t cnt = (uint32_t)(s_wbase[kTmaWarps - 1] - ubase + s_wcount[kTmaWarps - 1]);
  // every probe row matched once (PK-FK, match ratio 1; units without
  // duplicate build keys): output row t is probe row t, its build row is me[t]
  // (or res[t]); no compaction needed
  const bool ident = cnt == nq;
  if (!ident) {
    // 3a. compact the hits in probe order: list[t] = (build idx << 16) | probe idx
    uint32_t o = (uint32_t)(s_wbase[warp] - ubase);
    for (uint32_t r = r0; r < r1; ++r) {
      const uint32_t jl = r * 32 + lane;
      uint32_t e = kNoMatch;
      if (jl < nq) e = me ? (me[jl] == kEmpty16 ? kNoMatch : (uint32_t)me[jl]) : res[jl];
      const bool hit = e != kNoMatch;
      const uint32_t bal = __ballot_sync(0xffffffffu, hit);
      if (hit) list[o + __popc(bal & dev::lanemask_lt())] = (e << 16) | jl;
      o += __popc(bal);
    }
    dev::named_bar(1, kTmaThreads);  // the consumer warps of k_phj_tma
  }
  emit_rows<K>(a, inf, st, pk, me, res, list, ubase, cnt, ident);
}

// Warp-specialised like k_smj_tma: warp kTmaWarps (the producer) walks this
// CTA's units, puts each unit's descriptor (and, in the fill, the count pass's
// total and offset) in shared memory and bulk-copies its columns into a free
// stage; the 16 consumer warps take stages as the copies land (full barriers)
// and hand them back per warp (empty barriers).  Units the count pass fully
// resolved (the PK-FK fill) need no consumer-wide barrier at all; the other
// paths synchronise the consumers on named barrier 1.
template <class K, bool WRITE, int MINB>
__global__ void __launch_bounds__(kTmaThreads + 32, MINB)
k_phj_tma(const __grid_constant__ FindArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* tab = reinterpret_cast<uint32_t*>(smem + (size_t)a.stages * a.stage_bytes);
  uint32_t* res = tab + a.cap_entries;
  __shared__ UnitDesc s_desc[2];
  __shared__ bool s_pre[2];
  __shared__ uint64_t s_ucnt[2], s_ubase[2];
  __shared__ __align__(8) uint64_t full[2], empty[2];
  __shared__ uint64_t s_wcnt[2][kTmaWarps], s_wb[2][kTmaWarps];  // by unit parity
  __shared__ int s_dup;
  __shared__ int s_abort[2];  // speculative fill: the producer stopped at this stage

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t units = a.n_units;
  const UnitDesc* __restrict__ descs = reinterpret_cast<const UnitDesc*>(a.desc);
  const uint32_t kb = sizeof(K);
  const int S = a.stages;

  // Unit order: round robin over the CTAs, or (a.blocked) a contiguous range
  // of units per CTA, so the probe chunks of one build chunk (a large or
  // skewed probe partition) follow each other and reuse the build table.
  const bool blocked = a.np_rows > 0 && a.blocked;
  // blocked ranges split the probe rows evenly (unit q_lo is monotone): units
  // differ in size (a skewed partition's full chunks vs small ones)
  auto first_unit = [&](uint64_t c) -> uint64_t {  // first unit with q_lo >= c * |S| / grid
    const uint64_t target = c * a.np_rows / gridDim.x;
    uint64_t lo = 0, hi = units;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (descs[mid].q_lo < target) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const bool producer = warp == kTmaWarps;
  uint64_t u_begin = 0, u_end = units;
  if (tid == 0) {
    u_end = blocked ? (blockIdx.x + 1 == gridDim.x ? units : first_unit(blockIdx.x + 1)) : units;
    u_begin = blocked ? (blockIdx.x == 0 ? 0 : first_unit(blockIdx.x))
                      : (uint64_t)blockIdx.x * a.group;
  }
  __shared__ uint64_t s_range[2];
  if (tid == 0) {
    s_range[0] = u_begin;
    s_range[1] = u_end;
    for (int i = 0; i < 2; ++i) {
      dev::mbar_init(&full[i], 1);
      dev::mbar_init(&empty[i], kTmaWarps);
    }
    dev::fence_mbar_init();
  }
  __syncthreads();
  u_begin = s_range[0];
  u_end = s_range[1];
  // round robin over groups of a.group consecutive units: the probe chunks of
  // one build chunk (C3's wide rows: ~4 per partition) mostly land in one CTA
  // and reuse its table, while a skewed partition's many units still spread
  // over every CTA
  const uint64_t G = a.group;
  auto next_u = [&](uint64_t uu) -> uint64_t {
    if (blocked || (uu + 1) % G != 0) return uu + 1;
    return (uu / G + gridDim.x) * G;
  };

  if (producer) {  // ---- producer (one thread) ----
    if (lane != 0) return;
    auto bytes = [&](uint64_t lo, uint64_t hi, uint32_t w) {
      return (uint32_t)((dev::align_hi(hi, w) - dev::align_lo(lo, w)) * w);
    };
    // what a unit's staging needs from global memory, loaded one unit ahead
    // so the loads' latency overlaps the previous unit's wait and issue
    struct Pf {
      UnitDesc d;
      uint32_t dup;
      uint64_t cnt, base;
    };
    auto fetch = [&](uint64_t uu) {
      Pf p;
      p.d = descs[uu];
      p.dup = WRITE && a.match_e != nullptr ? a.unit_dup[uu] : 1u;
      p.cnt = WRITE && a.unit_counts ? a.unit_counts[uu] : ~0ull;
      p.base = WRITE && a.spec_fail ? p.d.q_lo : (WRITE && a.unit_off ? a.unit_off[uu] : 0ull);
      return p;
    };
    Pf nx{};
    if (u_begin < u_end) nx = fetch(u_begin);
    uint32_t k = 0;
    int pb = 0;
    uint32_t pr = 0;
    // the build chunk each stage buffer holds (keys and R payloads stay valid
    // there: later units on that stage overwrite only their probe regions), so
    // the units of one build chunk that land on the same stage copy it once
    uint64_t st_lo[4] = {~0ull, ~0ull, ~0ull, ~0ull}, st_hi[4] = {0, 0, 0, 0};
    bool st_keys[4] = {false, false, false, false};
    for (uint64_t u = u_begin; u < u_end; u = next_u(u), ++k) {
      const Pf cur = nx;
      if (next_u(u) < u_end) nx = fetch(next_u(u));
      // stage b of round r = k / S (kept incrementally: no division per tile)
      const int b = pb;
      if (k >= (uint32_t)S) dev::mbar_wait(&empty[b], pr ^ 1u);
      if (++pb == S) {
        pb = 0;
        pr ^= 1u;
      }
      const UnitDesc d = cur.d;
      if (WRITE && a.spec_fail && *reinterpret_cast<volatile uint32_t*>(a.spec_fail)) {
        // a unit failed the speculation: wake the consumers on this stage and stop
        s_abort[b] = 1;
        dev::mbar_arrive(&full[b]);
        return;
      }
      s_abort[b] = 0;
      // pre: the count pass resolved this unit's matches (match_e); no build keys needed
      const bool pre = WRITE && cur.dup == 0;
      s_desc[b] = d;
      s_pre[b] = pre;
      if (WRITE) {
        s_ucnt[b] = pre ? cur.cnt : ~0ull;
        s_ubase[b] = cur.base;
      }
      uint8_t* st = smem + (size_t)b * a.stage_bytes;
      const bool same = st_lo[b] == d.b_lo && st_hi[b] == d.b_hi;
      const bool need_keys = !pre && !(same && st_keys[b]);
      const bool need_r = WRITE && !same;
      st_keys[b] = same ? (st_keys[b] || !pre) : !pre;
      st_lo[b] = d.b_lo;
      st_hi[b] = d.b_hi;
      uint32_t total = bytes(d.q_lo, d.q_hi, kb);
      if (need_keys) total += bytes(d.b_lo, d.b_hi, kb);
      if (WRITE) {
        if (need_r)
          for (int c = 0; c < a.nr; ++c) total += bytes(d.b_lo, d.b_hi, a.r_bytes[c]);
        for (int c = 0; c < a.ns; ++c) total += bytes(d.q_lo, d.q_hi, a.s_bytes[c]);
        if (pre) total += bytes(d.q_lo, d.q_hi, 2);
      }
      dev::fence_proxy_async();
      dev::mbar_expect_tx(&full[b], total);
      auto copy = [&](uint32_t off, const void* base, uint64_t lo, uint64_t hi, uint32_t w) {
        dev::tma_load_1d(st + off, static_cast<const uint8_t*>(base) + dev::align_lo(lo, w) * w,
                         bytes(lo, hi, w), &full[b]);
      };
      if (need_keys) copy(a.off_bk, a.bkeys, d.b_lo, d.b_hi, kb);
      copy(a.off_pk, a.pkeys, d.q_lo, d.q_hi, kb);
      if (WRITE) {
        if (need_r)
          for (int c = 0; c < a.nr; ++c) copy(a.off_r[c], a.r_src[c], d.b_lo, d.b_hi, a.r_bytes[c]);
        for (int c = 0; c < a.ns; ++c) copy(a.off_s[c], a.s_src[c], d.q_lo, d.q_hi, a.s_bytes[c]);
        if (pre) copy(a.off_e, a.match_e, d.q_lo, d.q_hi, 2);
      }
    }
    return;
  }

  // ---- consumers ----
  auto sync_c = [] { dev::named_bar(1, kTmaThreads); };
  auto release = [&](int b) {  // this warp is done with stage b
    __syncwarp();
    if (lane == 0) dev::mbar_arrive(&empty[b]);
  };
  uint64_t built_lo = ~0ull, built_hi = 0;  // build chunk whose table is in shared memory
  uint32_t k = 0;
  int cb = 0;
  uint32_t cr = 0;
  const uint64_t key_hi = a.key_or ? (uint64_t)(*a.key_or) >> a.dense_shift : ~0ull;
  const uint32_t ds = a.dense_shift;
  // Direct-addressed tables hold (tag << 16) | chunk index; a new build chunk
  // takes a new tag, so the table is cleared only when the region was last
  // used otherwise (CAS table, sorted positions) or the tags wrap.
  uint32_t utag = 0;
  bool tab_tagged = false;
  for (uint64_t u = u_begin; u < u_end; u = next_u(u), ++k) {
    const int b = cb;
    const uint32_t cphase = cr;
    if (++cb == S) {
      cb = 0;
      cr ^= 1u;
    }
    uint64_t* s_wcount = s_wcnt[k & 1u];
    uint64_t* s_wbase = s_wb[k & 1u];
    dev::mbar_wait(&full[b], cphase);
    if (WRITE && s_abort[b]) break;
    const UnitDesc inf = s_desc[b];
    const bool pre = s_pre[b];
    const bool reuse = inf.b_lo == built_lo && inf.b_hi == built_hi;
    const uint32_t nb = (uint32_t)(inf.b_hi - inf.b_lo), nq = (uint32_t)(inf.q_hi - inf.q_lo);
    uint8_t* st = smem + (size_t)b * a.stage_bytes;
    const K* bk = reinterpret_cast<const K*>(st + a.off_bk) + (inf.b_lo - dev::align_lo(inf.b_lo, kb));
    const K* pk = reinterpret_cast<const K*>(st + a.off_pk) + (inf.q_lo - dev::align_lo(inf.q_lo, kb));
    const uint32_t rounds = (nq + 31) / 32;
    const uint32_t r0 = (uint32_t)((uint64_t)rounds * warp / kTmaWarps);
    const uint32_t r1 = (uint32_t)((uint64_t)rounds * (warp + 1) / kTmaWarps);
    // the speculative fill alternates its probe results between res and the
    // list region by unit parity, so a unit needs no barrier at its end
    const bool spec = WRITE && a.spec_fail != nullptr;
    uint32_t* const rs = spec ? res + (k & 1u) * a.qchunk : res;
    if (pre) {
      // matches resolved by the count pass
      const uint16_t* me = reinterpret_cast<const uint16_t*>(st + a.off_e) +
                           (inf.q_lo - dev::align_lo(inf.q_lo, 2));
      const uint64_t ubase = s_ubase[b];
      if (s_ucnt[b] == nq) {
        // every probe row matched once: the output rows are the probe rows in
        // order; no count, scan or compaction, no consumer-wide barrier
        emit_rows<K>(a, inf, st, pk, me, nullptr, nullptr, ubase, nq, true);
        release(b);
        continue;
      }
      uint64_t wc = 0;
      for (uint32_t r = r0; r < r1; ++r) {
        const uint32_t jl = r * 32 + lane;
        const bool hit = jl < nq && me[jl] != kEmpty16;
        wc += __popc(__ballot_sync(0xffffffffu, hit));
      }
      if (lane == 0) s_wcount[warp] = wc;
      sync_c();
      if (warp == 1) {
        const uint64_t c = lane < kTmaWarps ? s_wcount[lane] : 0;
        const uint64_t inc = dev::warp_inclusive_sum(c);
        if (lane < kTmaWarps) s_wbase[lane] = ubase + inc - c;
      }
      sync_c();
      emit_compact<K>(a, inf, st, pk, me, nullptr, r0, r1, nq, s_wbase, s_wcount, res + a.qchunk);
      release(b);
      sync_c();  // res / list are rewritten by the next unit
      continue;
    }
    // smallest power of two >= 2 nb (at least 2)
    const uint32_t cap_log2 = nb <= 1 ? 1u : 33u - (uint32_t)__clz(nb - 1);
    const uint32_t cap = 1u << cap_log2, cmask = cap - 1;
    // dense keys: slot = key >> dense_shift < cap for every build key
    const bool dense = key_hi < cap;
    // A tagged direct-addressed table needs no clear and so no barrier before
    // the inserts: every consumer passed the previous unit's post-probe
    // barrier before reaching this point, so nobody still reads the table.
    bool cleared = false;
    if (!reuse) {
      if (tid == 0) s_dup = 0;
      if (dense) {
        if (!tab_tagged || utag == 0xfffeu) {
          for (uint32_t i = tid; i < a.cap_entries; i += kTmaThreads) tab[i] = 0;
          utag = 0;
          tab_tagged = true;
          cleared = true;
        }
        ++utag;
      } else {
        for (uint32_t i = tid; i < cap; i += kTmaThreads) tab[i] = kNoMatch;
        tab_tagged = false;
        cleared = true;
      }
    }
    if (cleared) sync_c();

    // 1. insert chunk positions (CAS); meeting an equal key marks duplicates
    //    (a plain-store first round measured slower: profiles/r01b_summary.md).
    //    The previous unit of this CTA left the same build chunk's table (or
    //    its sorted positions) in shared memory: reuse it.
    bool dup = false;
    const uint32_t tagged = utag << 16;
    if (dense) {
      if (!reuse) {
        for (uint32_t i = tid; i < nb; i += kTmaThreads) tab[(uint32_t)(bk[i] >> ds)] = tagged | i;
        sync_c();
        // equal keys share a slot: one of them does not find itself there
        // (the speculative fill checks this after its probe: a duplicate
        // fails the unit either way)
        if (!spec)
          for (uint32_t i = tid; i < nb; i += kTmaThreads)
            if (tab[(uint32_t)(bk[i] >> ds)] != (tagged | i)) dup = true;
      }
    } else {
      for (uint32_t i = reuse ? nb : tid; i < nb; i += kTmaThreads) {
        const K key = bk[i];
        uint32_t sl = slot_of(key, cap_log2);
        while (true) {
          const uint32_t old = atomicCAS(&tab[sl], kNoMatch, i);
          if (old == kNoMatch) break;
          if (bk[old] == key) dup = true;
          sl = (sl + 1) & cmask;
        }
      }
    }
    // the OR-barrier also orders the inserts before the probes; a reused
    // table's flag was stored by the unit that built it
    const bool late_verify = spec && dense;
    bool any_dup = false;
    if (!late_verify) {
      any_dup = dev::named_bar_or(1, kTmaThreads, dup);
      if (any_dup && tid == 0) s_dup = 1;
    }
    const bool has_dup = reuse ? s_dup != 0 : any_dup;
    // a probe row of a split partition meets several build chunks, one unit
    // each, and matches in at most one: its match index cannot be handed to
    // the fill (the fill rebuilds those units' tables)
    if (!WRITE && a.unit_dup && tid == 0) a.unit_dup[u] = has_dup || inf.split ? 1 : 0;
    uint16_t* sidx = reinterpret_cast<uint16_t*>(tab);
    built_lo = inf.b_lo;
    built_hi = inf.b_hi;
    if (has_dup) tab_tagged = false;  // the region holds sorted positions now
    if (has_dup && !reuse) {  // stably sorted chunk positions: bitonic over (key, position)
      uint32_t np2 = 1;
      while (np2 < nb) np2 <<= 1;
      for (uint32_t i = tid; i < np2; i += kTmaThreads) sidx[i] = i < nb ? (uint16_t)i : kEmpty16;
      sync_c();
      for (uint32_t kk = 2; kk <= np2; kk <<= 1) {
        for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
          for (uint32_t i = tid; i < np2; i += kTmaThreads) {
            const uint32_t l = i ^ jj;
            if (l > i) {
              const uint16_t x = sidx[i], y = sidx[l];
              bool gt;
              if (x == kEmpty16) gt = y != kEmpty16;
              else if (y == kEmpty16) gt = false;
              else gt = bk[x] > bk[y] || (bk[x] == bk[y] && x > y);
              if (gt == ((i & kk) == 0)) { sidx[i] = y; sidx[l] = x; }
            }
          }
          sync_c();
        }
      }
    }

    // 2. probe from shared memory; warp w owns a contiguous run of rounds
    uint32_t wcount = 0;  // <= qchunk per unit
    uint16_t* const me_out = !WRITE && a.match_e && !inf.split ? a.match_e + inf.q_lo : nullptr;
    uint32_t r = r0;
    if (!has_dup && dense) {
      // direct-addressed table: the slot's entry is the match (same partition,
      // same high bits: the same key)
      for (; r < r1; ++r) {
        const uint32_t jl = r * 32 + lane;
        if (jl >= nq) continue;
        const uint64_t hi = (uint64_t)(pk[jl] >> ds);
        const uint32_t e = hi < cap ? tab[(uint32_t)hi] : 0u;
        const uint32_t m = (e >> 16) == utag;
        const uint32_t out = m ? (e & 0xffffu) : kNoMatch;
        if (WRITE) rs[jl] = out;
        else if (me_out) me_out[jl] = (uint16_t)(m ? out : kEmpty16);
        wcount += m;
      }
    }
    if (!has_dup) {
      // four rounds at a time: the first table probe and the build-key check of
      // every round are independent loads (collisions take the loop)
      for (; r + 4 <= r1; r += 4) {
        K key[4];
        uint32_t sl[4], e[4];
        bool in[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t jl = (r + u) * 32 + lane;
          in[u] = jl < nq;
          key[u] = in[u] ? pk[jl] : K(0);
          sl[u] = slot_of(key[u], cap_log2);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) e[u] = tab[sl[u]];
        K bkey[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) bkey[u] = e[u] != kNoMatch ? bk[e[u]] : K(0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (!in[u]) continue;
          const uint32_t jl = (r + u) * 32 + lane;
          uint32_t out = kNoMatch, m = 0;
          uint32_t ee = e[u], ss = sl[u];
          K bb = bkey[u];
          while (ee != kNoMatch) {
            if (bb == key[u]) {
              out = ee;
              m = 1;
              break;
            }
            ss = (ss + 1) & cmask;
            ee = tab[ss];
            if (ee != kNoMatch) bb = bk[ee];
          }
          if (WRITE) rs[jl] = out;
          else if (me_out) me_out[jl] = (uint16_t)(out == kNoMatch ? kEmpty16 : out);
          wcount += m;
        }
      }
    }
    for (; r < r1; ++r) {
      const uint32_t jl = r * 32 + lane;
      if (jl < nq) {
        const K key = pk[jl];
        uint32_t out = kNoMatch, m = 0;
        if (!has_dup) {
          uint32_t sl = slot_of(key, cap_log2);
          while (true) {
            const uint32_t e = tab[sl];
            if (e == kNoMatch) break;
            if (bk[e] == key) { out = e; m = 1; break; }
            sl = (sl + 1) & cmask;
          }
        } else {
          uint32_t lo = 0, hi = nb;
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (bk[sidx[mid]] < key) lo = mid + 1; else hi = mid;
          }
          uint32_t lo2 = lo, hi2 = nb;
          while (lo2 < hi2) {
            const uint32_t mid = (lo2 + hi2) >> 1;
            if (bk[sidx[mid]] <= key) lo2 = mid + 1; else hi2 = mid;
          }
          m = lo2 - lo;
          out = (lo << 16) | m;
        }
        if (WRITE) rs[jl] = out;
        else if (me_out && !has_dup) me_out[jl] = (uint16_t)(out == kNoMatch ? kEmpty16 : out);
        wcount += m;
      }
    }
    if (WRITE && a.spec_fail) {
      // speculation: this unit's rows go to its probe offset only if every
      // probe row matched exactly once — one OR-barrier over "a row of mine
      // missed" replaces the count, its barrier and the scan (the output rows
      // are then the probe rows in order)
      const uint32_t full = nq >> 5, rem = nq & 31;
      uint32_t mine = r0 < min(r1, full) ? min(r1, full) - r0 : 0u;
      if (full >= r0 && full < r1 && (uint32_t)lane < rem) ++mine;
      if (late_verify && !reuse)
        for (uint32_t i = tid; i < nb; i += kTmaThreads)
          if (tab[(uint32_t)(bk[i] >> ds)] != (tagged | i)) dup = true;
      if (dev::named_bar_or(1, kTmaThreads, has_dup || dup || wcount != mine)) {
        if (tid == 0) atomicExch(a.spec_fail, 1u);
      } else {
        if (tid == 0) atomicAdd(a.spec_rows, nq);
        emit_rows<K>(a, inf, st, pk, nullptr, rs, nullptr, s_ubase[b], nq, true);
      }
      release(b);
      continue;
    }
    wcount = (uint32_t)dev::warp_sum((uint64_t)wcount);
    if (lane == 0) s_wcount[warp] = wcount;
    sync_c();  // every probe of this unit is done: the table may be rebuilt after this
    if (!WRITE) release(b);
    if (warp == 1) {
      const uint64_t wc = lane < kTmaWarps ? s_wcount[lane] : 0;
      const uint64_t inc = dev::warp_inclusive_sum(wc);
      if (lane < kTmaWarps) s_wbase[lane] = s_ubase[b] + inc - wc;
      if (!WRITE && lane == kTmaWarps - 1) a.unit_counts[u] = inc;
    }
    if (!WRITE) continue;
    sync_c();
    // 3. emit finished rows in probe order at the unit's offset
    const uint32_t bsh4 = (uint32_t)(inf.b_lo & 3), bsh8 = (uint32_t)(inf.b_lo & 1);
    const uint32_t qsh4 = (uint32_t)(inf.q_lo & 3), qsh8 = (uint32_t)(inf.q_lo & 1);
    auto write_row = [&](uint64_t oo, uint32_t li, uint32_t jl, K key) {
      const uint64_t gi = inf.b_lo + li, j = inf.q_lo + jl;
      if (a.key_out) static_cast<K*>(a.key_out)[oo] = key;
      if (a.ids_r) a.ids_r[oo] = a.carried_r ? a.carried_r[gi] : (uint32_t)gi;
      if (a.ids_s) a.ids_s[oo] = a.carried_s ? a.carried_s[j] : (uint32_t)j;
      for (int c = 0; c < a.nr; ++c) {
        if (a.r_bytes[c] == 4)
          static_cast<uint32_t*>(a.r_dst[c])[oo] = reinterpret_cast<const uint32_t*>(st + a.off_r[c])[bsh4 + li];
        else
          static_cast<uint64_t*>(a.r_dst[c])[oo] = reinterpret_cast<const uint64_t*>(st + a.off_r[c])[bsh8 + li];
      }
      for (int c = 0; c < a.ns; ++c) {
        if (a.s_bytes[c] == 4)
          static_cast<uint32_t*>(a.s_dst[c])[oo] = reinterpret_cast<const uint32_t*>(st + a.off_s[c])[qsh4 + jl];
        else
          static_cast<uint64_t*>(a.s_dst[c])[oo] = reinterpret_cast<const uint64_t*>(st + a.off_s[c])[qsh8 + jl];
      }
    };
    if (!has_dup) {
      emit_compact<K>(a, inf, st, pk, nullptr, res, r0, r1, nq, s_wbase, s_wcount, res + a.qchunk);
      release(b);
      sync_c();
      continue;
    }
    uint64_t o = s_wbase[warp];
    for (uint32_t r = r0; r < r1; ++r) {
      const uint32_t jl = r * 32 + lane;
      const uint32_t e = jl < nq ? res[jl] : kNoMatch;
      const uint32_t m = e == kNoMatch ? 0 : (e & 0xffffu);
      const uint32_t lb = e >> 16;
      const uint32_t inc = dev::warp_inclusive_sum(m);
      uint64_t oo = o + inc - m;
      for (uint32_t t = 0; t < m; ++t, ++oo) {
        const uint32_t li = sidx[lb + t];
        if (oo < a.capacity) write_row(oo, li, jl, bk[li]);
      }
      o += __shfl_sync(0xffffffffu, inc, 31);
    }
    release(b);
    sync_c();
  }
}

struct Plan {
  uint64_t total_units = 0;
  uint64_t max_chunk = 0;
};

Plan make_plan(cj_ctx* ctx, const uint64_t* boff, const uint64_t* poff, uint32_t fanout,
               uint32_t limit, uint64_t* unit_start, uint32_t qchunk) {
  Scratch st(ctx, 2 * sizeof(uint64_t));
  CJ_CUDA(cudaMemsetAsync(st.p, 0, 2 * sizeof(uint64_t), ctx->stream));
  const uint32_t blocks = (fanout + kPlanThreads * kPlanPer - 1) / (kPlanThreads * kPlanPer);
  PlanArgs2 pa{boff, poff, fanout, limit, qchunk, unit_start,
               st.as<unsigned long long>(), ctx->status_buffer(blocks), 0, ctx->err_word};
  pa.epoch = ctx->next_epoch();
  ctx->kbegin("phj_plan", 16ull * fanout);
  k_phj_plan<<<blocks, kPlanThreads, 0, ctx->stream>>>(pa);
  ctx->kend();
  CJ_CUDA(cudaGetLastError());
  uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  CJ_CUDA(cudaMemcpyAsync(h, st.p, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  return Plan{h[1], h[0]};
}

void atomicOr_host_overflow(cj_ctx* ctx) {
  const uint32_t v = kErrOverflow;
  CJ_CUDA(cudaMemcpyAsync(ctx->err_word, &v, 4, cudaMemcpyHostToDevice, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
}

template <class K>
bool tma_layout(FindArgs& a, size_t* smem_out) {
  auto up = [](size_t x) { return (x + 127) & ~size_t(127); };
  const uint32_t kb = sizeof(K);
  size_t off = 0;
  a.off_bk = (uint32_t)off;
  off = up(off + (size_t)(a.max_chunk + 8) * kb);
  for (int c = 0; c < a.nr; ++c) {
    a.off_r[c] = (uint32_t)off;
    off = up(off + (size_t)(a.max_chunk + 8) * a.r_bytes[c]);
  }
  a.off_pk = (uint32_t)off;
  off = up(off + (size_t)(a.qchunk + 8) * kb);
  for (int c = 0; c < a.ns; ++c) {
    a.off_s[c] = (uint32_t)off;
    off = up(off + (size_t)(a.qchunk + 8) * a.s_bytes[c]);
  }
  if (a.write && a.match_e) {
    a.off_e = (uint32_t)off;
    off = up(off + (size_t)(a.qchunk + 8) * 2);
  }
  a.stage_bytes = (uint32_t)off;
  a.cap_entries = 1u << a.cap_log2;
  // + res[qchunk] probe results + list[qchunk] compacted hits (fill only)
  const size_t smem = (size_t)a.stages * off + up(4 * (size_t)a.cap_entries) +
                      (a.write ? (size_t)a.qchunk * 8 : 0);
  *smem_out = smem;
  // + < 2 KB of static shared memory per CTA
  return smem <= (size_t)(a.write ? 225 / find_ctas_per_sm() - 2 : 225) * 1024;
}

// Probe rows per work unit: the largest (<= 8192, multiple of 128) whose two
// stages fit shared memory, so a probe partition is rarely split into a second
// unit that rebuilds the same build table for a few rows (C2: partitions of
// 4096 +- 64 rows; a 4096 chunk splits half of them).  CJ_QCHUNK overrides.
template <class K>
uint32_t choose_qchunk(FindArgs a) {
  if (std::getenv("CJ_QCHUNK")) return probe_chunk();
  size_t smem = 0;
  for (uint32_t q = 8192; q >= 1024; q -= 128) {
    a.qchunk = q;
    if (tma_layout<K>(a, &smem)) return q;
  }
  return probe_chunk();
}

// The fill at one CTA per SM (default), or two (CJ_FIND_CTAS=2: half the
// shared memory each, probe chunks sized to fit, <= 60 registers).
template <class K>
void launch_fill(cj_ctx* ctx, const FindArgs& a, unsigned grid, size_t smem) {
  if (find_ctas_per_sm() >= 2) {
    CJ_CUDA(cudaFuncSetAttribute(k_phj_tma<K, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    k_phj_tma<K, true, 2><<<grid, kTmaThreads + 32, smem, ctx->stream>>>(a);
  } else {
    CJ_CUDA(cudaFuncSetAttribute(k_phj_tma<K, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    k_phj_tma<K, true, 1><<<grid, kTmaThreads + 32, smem, ctx->stream>>>(a);
  }
}

template <class K>
uint64_t run_find(cj_ctx* ctx, FindArgs a, uint64_t total_units) {
  Scratch tot(ctx, sizeof(uint64_t));
  CJ_CUDA(cudaMemsetAsync(tot.p, 0, sizeof(uint64_t), ctx->stream));
  a.total_out = tot.as<uint64_t>();
  a.status = ctx->status_buffer(total_units);
  a.epoch = ctx->next_epoch();
  a.ticket = ctx->ticket(1);
  a.err = ctx->err_word;
  uint32_t cap_log2 = 1;
  while ((1ull << cap_log2) < 2ull * a.max_chunk) ++cap_log2;
  a.cap_log2 = cap_log2;
  size_t tma_smem = 0;
  const char* mode = std::getenv("CJ_FIND");
  const bool want_tma = !(mode && std::strcmp(mode, "ldg") == 0);
  // count pass -> fill pass hand-off (see FindArgs::match_e)
  const char* me_env = std::getenv("CJ_FIND_HANDOFF");
  const bool handoff = a.write && a.padded && a.desc && !(me_env && std::strcmp(me_env, "0") == 0);
  Scratch me_buf(ctx, handoff ? a.np_rows * 2 + kPad : 0);
  Scratch dup_buf(ctx, handoff ? total_units + 16 : 0);
  if (handoff) {
    a.match_e = me_buf.as<uint16_t>();
    a.unit_dup = dup_buf.as<uint8_t>();
  }
  if (want_tma && a.padded && a.desc && tma_layout<K>(a, &tma_smem)) {
    // count pass (keys only) -> scan -> fill pass; no inter-CTA waiting
    const uint64_t U = total_units;
    uint64_t total = 0;
    if (U > 0 && a.write && a.spec_fail) {
      // PK-FK speculation: one fill pass, each unit at its probe offset
      FindArgs as = a;
      as.match_e = nullptr;
      as.unit_dup = nullptr;
      as.unit_counts = nullptr;
      as.unit_off = nullptr;
      size_t smem_s = 0;
      tma_layout<K>(as, &smem_s);
      const unsigned grid =
          (unsigned)std::min<uint64_t>((uint64_t)ctx->num_sms * find_ctas_per_sm(), U);
      ctx->kbegin("phj_find", 0);
      launch_fill<K>(ctx, as, grid, smem_s);
      ctx->kend();
      CJ_CUDA(cudaGetLastError());
      uint32_t* h = ctx->host_pinned;
      CJ_CUDA(cudaMemcpyAsync(h, a.spec_fail, 4, cudaMemcpyDeviceToHost, ctx->stream));
      CJ_CUDA(cudaMemcpyAsync(h + 1, a.spec_rows, 4, cudaMemcpyDeviceToHost, ctx->stream));
      CJ_CUDA(cudaMemcpyAsync(h + 2, ctx->err_word, 4, cudaMemcpyDeviceToHost, ctx->stream));
      CJ_CUDA(cudaStreamSynchronize(ctx->stream));
      // every unit matched completely AND the units covered every probe row
      if (h[0] == 0 && h[1] == a.np_rows) {
        ctx->err_known_clean = h[2] == 0;
        return a.np_rows;
      }
    }
    a.spec_fail = nullptr;
    if (U > 0) {
      Scratch counts(ctx, U * 8), offs(ctx, U * 8);
      FindArgs ac = a;
      ac.nr = ac.ns = 0;
      ac.write = 0;
      ac.unit_counts = counts.as<uint64_t>();
      size_t smem_c = 0;
      tma_layout<K>(ac, &smem_c);
      // the count pass needs little shared memory: two CTAs per SM hide latency
      const char* ec = std::getenv("CJ_COUNT_CTAS");
      const unsigned grid_c = (unsigned)std::min<uint64_t>(
          (uint64_t)ctx->num_sms * (ec ? std::max(1, std::atoi(ec)) : 2), U);
      const unsigned grid =
          (unsigned)std::min<uint64_t>((uint64_t)ctx->num_sms * find_ctas_per_sm(), U);
      CJ_CUDA(cudaFuncSetAttribute(k_phj_tma<K, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_c));
      ctx->kbegin("phj_count", (uint64_t)(sizeof(K)) * (a.nb_rows + a.np_rows));
      k_phj_tma<K, false, 2><<<grid_c, kTmaThreads + 32, smem_c, ctx->stream>>>(ac);
      ctx->kend();
      scan_counts(ctx, counts.as<uint64_t>(), U, offs.as<uint64_t>(), a.total_out);
      CJ_CUDA(cudaGetLastError());
      if (a.write) {
        // the fill is launched without waiting for the total: every write is
        // bounded by the capacity on the device, and an overflow is reported
        // (CapacityExceeded) after the single synchronisation below
        a.unit_off = offs.as<uint64_t>();
        a.unit_counts = std::getenv("CJ_FIND_FAST") && std::strcmp(std::getenv("CJ_FIND_FAST"), "0") == 0
                            ? nullptr : counts.as<uint64_t>();
        ctx->kbegin("phj_find", 0);
        launch_fill<K>(ctx, a, grid, tma_smem);
        ctx->kend();
        CJ_CUDA(cudaGetLastError());
      }
      uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
      CJ_CUDA(cudaMemcpyAsync(h, a.total_out, 8, cudaMemcpyDeviceToHost, ctx->stream));
      CJ_CUDA(cudaStreamSynchronize(ctx->stream));
      total = h[0];
      if (a.write && total > a.capacity) atomicOr_host_overflow(ctx);
    }
    return total;
  } else {
    size_t stage = 0;
    if (a.write && a.nr > 0) {
      for (int c = 0; c < a.nr; ++c) {
        a.r_stage_off[c] = (uint32_t)stage;
        stage += (size_t)a.max_chunk * a.r_bytes[c];
        stage = (stage + 15) & ~size_t(15);
      }
    }
    size_t smem = (size_t)a.max_chunk * sizeof(K);
    smem = (smem + 15) & ~size_t(15);
    smem += (size_t)2 << cap_log2;
    smem += (size_t)a.qchunk * 4;
    a.stage_r = 0;
    if (stage && smem + stage <= 160 * 1024) {
      a.stage_r = 1;
      smem += stage;
    }
    if (smem > 200 * 1024) fail(CJ_ERR_CAPACITY_EXCEEDED, "hash join: build chunk exceeds shared memory");
    CJ_CUDA(cudaFuncSetAttribute(k_phj_find<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    int per_sm = 0;
    CJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_phj_find<K>, kThreads, smem));
    per_sm = std::max(per_sm, 1);
    const uint64_t grid = std::min<uint64_t>((uint64_t)ctx->num_sms * per_sm, total_units);
    if (total_units > 0) {
      ctx->kbegin(a.write ? "phj_find" : "phj_count", 0);
      k_phj_find<K><<<(unsigned)grid, kThreads, smem, ctx->stream>>>(a);
      ctx->kend();
      CJ_CUDA(cudaGetLastError());
    }
  }
  uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  CJ_CUDA(cudaMemcpyAsync(h, tot.p, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  return h[0];
}

// Precomputed unit descriptors for the TMA passes.
void build_desc(cj_ctx* ctx, FindArgs& a, uint64_t total_units, Scratch& desc) {
  if (total_units == 0) return;
  ctx->kbegin("phj_desc", total_units * 32);
  k_phj_desc<<<grid_for(total_units, 256, 4096), 256, 0, ctx->stream>>>(
      a.boff, a.poff, a.unit_start, a.fanout, a.limit, a.qchunk, total_units, desc.as<UnitDesc>());
  ctx->kend();
  CJ_CUDA(cudaGetLastError());
  a.desc = desc.p;
  a.n_units = total_units;
}

FindArgs base_args(const void* bkeys, const uint64_t* boff, const void* pkeys,
                   const uint64_t* poff, uint32_t fanout, uint32_t limit) {
  FindArgs a{};
  a.bkeys = bkeys;
  a.boff = boff;
  a.pkeys = pkeys;
  a.poff = poff;
  a.fanout = fanout;
  a.limit = limit;
  a.qchunk = probe_chunk();
  a.stages = find_stages();
  const char* order = std::getenv("CJ_FIND_ORDER");
  a.blocked = order && std::strcmp(order, "blocked") == 0;
  const char* grp = std::getenv("CJ_FIND_GROUP");
  a.group = grp ? (uint32_t)std::max(1, std::atoi(grp)) : 4;
  return a;
}

// CJ_DENSE=0 turns the direct-addressed tables off (experiments)
bool dense_keys() {
  const char* e = std::getenv("CJ_DENSE");
  return !(e && std::strcmp(e, "0") == 0);
}

void check_limit(uint32_t limit) {
  if (limit == 0) fail(CJ_ERR_SPEC_INVALID, "sub-partition limit must be positive");
  if (limit > 16384)
    fail(CJ_ERR_UNSUPPORTED, "sub-partition limit above 16384 rows is not supported on the device");
}

}  // namespace

uint32_t log2_of(uint32_t fanout) {
  uint32_t b = 0;
  while ((1u << b) < fanout) ++b;
  return b;
}

uint64_t phj_find(cj_ctx* ctx, const void* bkeys, const uint64_t* boff, const void* pkeys,
                  const uint64_t* poff, uint32_t fanout, int key_bytes, uint32_t limit,
                  const OutSpec& out, uint64_t capacity, const unsigned long long* key_or,
                  bool pk_fk) {
  check_limit(limit);
  Scratch us(ctx, sizeof(uint64_t) * ((uint64_t)fanout + 1));
  Plan plan = make_plan(ctx, boff, poff, fanout, limit, us.as<uint64_t>(), probe_chunk());
  FindArgs a = base_args(bkeys, boff, pkeys, poff, fanout, limit);
  a.unit_start = us.as<uint64_t>();
  a.max_chunk = (uint32_t)std::max<uint64_t>(plan.max_chunk, 1);
  a.write = 1;
  a.key_or = dense_keys() ? key_or : nullptr;
  a.dense_shift = log2_of(fanout);
  // speculate that every probe row finds its key (PK-FK): skips the count
  // pass when it holds (C2, C4); a miss falls back to count + fill
  const char* se = std::getenv("CJ_SPECULATE");
  if (pk_fk && capacity >= out.s_rows && !(se && std::strcmp(se, "0") == 0)) {
    a.spec_fail = ctx->ticket(3);
    a.spec_rows = ctx->ticket(5);
  }
  a.capacity = capacity;
  a.padded = out.padded ? 1 : 0;
  a.nb_rows = out.r_rows;
  a.np_rows = out.s_rows;
  a.nr = out.nr;
  a.ns = out.ns;
  for (int c = 0; c < out.nr; ++c) a.r_bytes[c] = out.r_bytes[c];
  for (int c = 0; c < out.ns; ++c) a.s_bytes[c] = out.s_bytes[c];
  if (a.padded) {
    uint32_t cap_log2 = 1;
    while ((1ull << cap_log2) < 2ull * a.max_chunk) ++cap_log2;
    a.cap_log2 = cap_log2;
    a.match_e = reinterpret_cast<uint16_t*>(16);  // layout with the hand-off chunk
    const uint32_t q = key_bytes == 4 ? choose_qchunk<uint32_t>(a) : choose_qchunk<uint64_t>(a);
    a.match_e = nullptr;
    if (q != a.qchunk) {
      a.qchunk = q;
      plan = make_plan(ctx, boff, poff, fanout, limit, us.as<uint64_t>(), q);
    }
  }
  Scratch desc(ctx, std::max<uint64_t>(plan.total_units, 1) * sizeof(UnitDesc));
  if (a.padded) build_desc(ctx, a, plan.total_units, desc);
  a.key_out = out.key;
  a.ids_r = out.ids_r;
  a.ids_s = out.ids_s;
  a.carried_r = out.carried_r;
  a.carried_s = out.carried_s;
  a.nr = out.nr;
  a.ns = out.ns;
  for (int c = 0; c < out.nr; ++c) {
    a.r_src[c] = out.r_src[c];
    a.r_dst[c] = out.r_dst[c];
    a.r_bytes[c] = out.r_bytes[c];
  }
  for (int c = 0; c < out.ns; ++c) {
    a.s_src[c] = out.s_src[c];
    a.s_dst[c] = out.s_dst[c];
    a.s_bytes[c] = out.s_bytes[c];
  }
  const uint64_t total = key_bytes == 4 ? run_find<uint32_t>(ctx, a, plan.total_units)
                                        : run_find<uint64_t>(ctx, a, plan.total_units);
  raise_device_errors(ctx);
  return total;
}

uint64_t phj_count(cj_ctx* ctx, const void* bkeys, const uint64_t* boff, const void* pkeys,
                   const uint64_t* poff, uint32_t fanout, int key_bytes, uint32_t limit,
                   const unsigned long long* key_or) {
  check_limit(limit);
  Scratch us(ctx, sizeof(uint64_t) * ((uint64_t)fanout + 1));
  const Plan plan = make_plan(ctx, boff, poff, fanout, limit, us.as<uint64_t>(), probe_chunk());
  FindArgs a = base_args(bkeys, boff, pkeys, poff, fanout, limit);
  a.unit_start = us.as<uint64_t>();
  a.max_chunk = (uint32_t)std::max<uint64_t>(plan.max_chunk, 1);
  a.write = 0;
  a.key_or = dense_keys() ? key_or : nullptr;
  a.dense_shift = log2_of(fanout);
  return key_bytes == 4 ? run_find<uint32_t>(ctx, a, plan.total_units)
                        : run_find<uint64_t>(ctx, a, plan.total_units);
}

}  // namespace cj
