// Partitioned hash join find phase (K4), optionally fused with GFTR
// materialisation.
//
// Reference semantics (paths relative to the reference's proj/):
//   plan_subpartitions   hash_match.cpp:186-210  (build chunks of <= limit rows)
//   ChunkTable/scan_unit hash_match.cpp:73-121   (equal keys in insertion order)
//   hash_match_count     hash_match.cpp:212-248
//   hash_match_fill      hash_match.cpp:250-302  (order: unit, probe pos, build pos)
//
// Design (B200): work units are (partition, build chunk, probe chunk of <= 4096
// rows); splitting the probe side keeps a Zipf hot partition spread over many
// CTAs while the concatenation in unit order is exactly the reference's
// emission order.  A persistent CTA takes unit tickets in order, stages the
// build chunk's keys (and, fused, its transformed payload columns) in shared
// memory, builds a 16-bit open-addressing table of chunk positions with CAS
// (duplicate keys are detected exactly during insertion), probes, publishes
// the unit's match count and resolves its output offset by warp-cooperative
// decoupled look-back, then writes its rows in probe order.  Chunks holding
// duplicate keys switch to a stably sorted chunk (bitonic over (key, pos)) so
// every probe emits its matches in build insertion order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "cj_device.cuh"
#include "cj_internal.cuh"

namespace cj {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kProbeChunk = 4096;
constexpr uint16_t kEmpty16 = 0xffffu;
constexpr uint32_t kNoMatch = 0xffffffffu;

struct PlanArgs {
  const uint64_t* boff;
  const uint64_t* poff;
  uint32_t fanout, limit, qchunk;
  uint64_t* unit_start;   // fanout + 1
  uint64_t* stats;        // [0] max build chunk, [1] total units
};

// unit_start[p] = number of units before partition p (units with an empty
// side produce no rows and are dropped).
__global__ void __launch_bounds__(1024) k_phj_plan(const PlanArgs a) {
  __shared__ uint64_t wsum[32];
  const uint32_t per = (a.fanout + blockDim.x - 1) / blockDim.x;
  const uint32_t p0 = min(a.fanout, threadIdx.x * per), p1 = min(a.fanout, p0 + per);
  uint64_t local = 0, maxc = 0;
  for (uint32_t p = p0; p < p1; ++p) {
    const uint64_t nb = a.boff[p + 1] - a.boff[p], ns = a.poff[p + 1] - a.poff[p];
    if (nb && ns) {
      local += ((nb + a.limit - 1) / a.limit) * ((ns + a.qchunk - 1) / a.qchunk);
      maxc = max(maxc, dev::umin64(nb, a.limit));
    }
  }
  const uint64_t inc = dev::warp_inclusive_sum(local);
  if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = inc;
  __syncthreads();
  uint64_t off = 0;
  for (unsigned w = 0; w < (threadIdx.x >> 5); ++w) off += wsum[w];
  uint64_t run = off + inc - local;
  for (uint32_t p = p0; p < p1; ++p) {
    a.unit_start[p] = run;
    const uint64_t nb = a.boff[p + 1] - a.boff[p], ns = a.poff[p + 1] - a.poff[p];
    if (nb && ns) run += ((nb + a.limit - 1) / a.limit) * ((ns + a.qchunk - 1) / a.qchunk);
  }
  if (threadIdx.x == blockDim.x - 1) {
    a.unit_start[a.fanout] = run;
    a.stats[1] = run;
  }
  // block max of chunk sizes
  for (int o = 16; o > 0; o >>= 1) maxc = max(maxc, __shfl_xor_sync(0xffffffffu, maxc, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = maxc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t m = 0;
    for (unsigned w = 0; w < blockDim.x / 32; ++w) m = max(m, wsum[w]);
    a.stats[0] = m;
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
};

template <class K>
__device__ __forceinline__ uint32_t slot_of(K k, uint32_t log2cap) {
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
    uint32_t cap_log2 = 1;
    while ((1u << cap_log2) < 2 * nb) ++cap_log2;
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

struct Plan {
  uint64_t total_units = 0;
  uint64_t max_chunk = 0;
};

Plan make_plan(cj_ctx* ctx, const uint64_t* boff, const uint64_t* poff, uint32_t fanout,
               uint32_t limit, uint64_t* unit_start) {
  Scratch st(ctx, 2 * sizeof(uint64_t));
  PlanArgs pa{boff, poff, fanout, limit, kProbeChunk, unit_start, st.as<uint64_t>()};
  ctx->kbegin("phj_plan", 16ull * fanout);
  k_phj_plan<<<1, 1024, 0, ctx->stream>>>(pa);
  ctx->kend();
  CJ_CUDA(cudaGetLastError());
  uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  CJ_CUDA(cudaMemcpyAsync(h, st.p, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  return Plan{h[1], h[0]};
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
  uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  CJ_CUDA(cudaMemcpyAsync(h, tot.p, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  return h[0];
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
  a.qchunk = kProbeChunk;
  return a;
}

void check_limit(uint32_t limit) {
  if (limit == 0) fail(CJ_ERR_SPEC_INVALID, "sub-partition limit must be positive");
  if (limit > 16384)
    fail(CJ_ERR_UNSUPPORTED, "sub-partition limit above 16384 rows is not supported on the device");
}

}  // namespace

uint64_t phj_find(cj_ctx* ctx, const void* bkeys, const uint64_t* boff, const void* pkeys,
                  const uint64_t* poff, uint32_t fanout, int key_bytes, uint32_t limit,
                  const OutSpec& out, uint64_t capacity) {
  check_limit(limit);
  Scratch us(ctx, sizeof(uint64_t) * ((uint64_t)fanout + 1));
  const Plan plan = make_plan(ctx, boff, poff, fanout, limit, us.as<uint64_t>());
  FindArgs a = base_args(bkeys, boff, pkeys, poff, fanout, limit);
  a.unit_start = us.as<uint64_t>();
  a.max_chunk = (uint32_t)std::max<uint64_t>(plan.max_chunk, 1);
  a.write = 1;
  a.capacity = capacity;
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
                   const uint64_t* poff, uint32_t fanout, int key_bytes, uint32_t limit) {
  check_limit(limit);
  Scratch us(ctx, sizeof(uint64_t) * ((uint64_t)fanout + 1));
  const Plan plan = make_plan(ctx, boff, poff, fanout, limit, us.as<uint64_t>());
  FindArgs a = base_args(bkeys, boff, pkeys, poff, fanout, limit);
  a.unit_start = us.as<uint64_t>();
  a.max_chunk = (uint32_t)std::max<uint64_t>(plan.max_chunk, 1);
  a.write = 0;
  return key_bytes == 4 ? run_find<uint32_t>(ctx, a, plan.total_units)
                        : run_find<uint64_t>(ctx, a, plan.total_units);
}

}  // namespace cj
