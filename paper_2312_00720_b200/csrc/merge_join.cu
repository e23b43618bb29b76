// Sort-merge join find phase (K5), optionally fused with GFTR
// materialisation.
//
// Reference semantics (paths relative to the reference's proj/):
//   merge_path_split / diagonal_intersect  merge_match.cpp:30-48, 75-102
//   walk_part                              merge_match.cpp:53-71
//   merge_match_count / merge_match_fill   merge_match.cpp:104-155
// Output: every (i, j) with r[i] == s[j] in (s-position, r-position) order,
// output key = s[j]; pk_fk emits only the lower bound (merge_match.cpp:65-68).
//
// Design (B200): tiles of 2048 consecutive probe (s) positions.  A tile's r
// window [lower_bound(s[j0]), upper_bound(s[j1-1])) bounds the keys it can
// match (merge path: equal work per tile on the s side).  run_join's path is
// k_smj_tma: a count pass (window staged in shared memory, every probe's
// lower bound by interpolation + galloping, PK-FK window indices handed to
// the fill) -> scan of the tile counts -> fill pass; both warp-specialised
// (a producer warp stages tiles, 16 consumer warps release them per warp).
// The operator API on arbitrary buffers uses k_smj_find, one pass whose
// tiles chain their output offsets by warp-cooperative decoupled look-back.
// Windows larger than shared memory fall back to global binary searches
// (correct, slower; only for sparse probes).
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
constexpr uint32_t kTileS = 2048;

struct SmjArgs {
  const void* r;
  uint64_t nr;
  const void* s;
  uint64_t ns;
  int pk_fk;
  uint32_t wmax;          // shared-memory r window capacity (keys)
  uint64_t tiles;
  uint64_t* status;
  uint64_t epoch;
  uint32_t* ticket;
  uint32_t* err;
  uint64_t capacity;
  int write;
  uint64_t* total_out;
  void* key_out;
  uint32_t* ids_r;
  uint32_t* ids_s;
  const uint32_t* carried_r;
  const uint32_t* carried_s;
  int nr_cols, ns_cols;
  const void* r_src[CJ_MAX_COLS];
  const void* s_src[CJ_MAX_COLS];
  void* r_dst[CJ_MAX_COLS];
  void* s_dst[CJ_MAX_COLS];
  uint32_t r_bytes[CJ_MAX_COLS];
  uint32_t s_bytes[CJ_MAX_COLS];
  // TMA count / fill passes
  const void* desc;          // SmjDesc[tiles]
  uint64_t* tile_counts;
  uint64_t* tile_off;
  uint32_t stage_bytes, off_rk, off_sk, off_r[CJ_MAX_COLS], off_s[CJ_MAX_COLS];
  int padded;
  // count -> fill hand-off for PK-FK tiles (see k_smj_tma)
  uint16_t* match_e;
  uint8_t* tile_pre;
  uint32_t off_e;
  int nstages;               // TMA stage ring depth (2..kSmjMaxStages)
  // speculative PK-FK fill (no count pass): every probe row is expected to
  // find its key, so tile t writes its rows at its first probe row; a tile
  // with a miss sets *spec_fail and the caller runs count + fill
  uint32_t* spec_fail;
  uint32_t* spec_rows;       // probe rows of the tiles that matched completely
};

template <class K>
__device__ __forceinline__ uint64_t g_lower_bound(const K* __restrict__ r, uint64_t lo,
                                                  uint64_t hi, K k) {
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (r[mid] < k) lo = mid + 1; else hi = mid;
  }
  return lo;
}
template <class K>
__device__ __forceinline__ uint64_t g_upper_bound(const K* __restrict__ r, uint64_t lo,
                                                  uint64_t hi, K k) {
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (r[mid] <= k) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <class K>
__device__ __forceinline__ void emit(const SmjArgs& a, uint64_t o, uint64_t i, uint64_t j, K k) {
  if (a.key_out) static_cast<K*>(a.key_out)[o] = k;
  if (a.ids_r) a.ids_r[o] = a.carried_r ? a.carried_r[i] : (uint32_t)i;
  if (a.ids_s) a.ids_s[o] = a.carried_s ? a.carried_s[j] : (uint32_t)j;
  for (int c = 0; c < a.nr_cols; ++c) {
    if (a.r_bytes[c] == 4)
      static_cast<uint32_t*>(a.r_dst[c])[o] = static_cast<const uint32_t*>(a.r_src[c])[i];
    else
      static_cast<uint64_t*>(a.r_dst[c])[o] = static_cast<const uint64_t*>(a.r_src[c])[i];
  }
  for (int c = 0; c < a.ns_cols; ++c) {
    if (a.s_bytes[c] == 4)
      static_cast<uint32_t*>(a.s_dst[c])[o] = __ldcs(static_cast<const uint32_t*>(a.s_src[c]) + j);
    else
      static_cast<uint64_t*>(a.s_dst[c])[o] = __ldcs(static_cast<const uint64_t*>(a.s_src[c]) + j);
  }
}

template <class K>
__global__ void __launch_bounds__(kThreads) k_smj_find(const __grid_constant__ SmjArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  K* rk = reinterpret_cast<K*>(smem);                          // [wmax]
  uint32_t* loff = reinterpret_cast<uint32_t*>(smem + (size_t)a.wmax * sizeof(K));  // [kTileS]
  uint32_t* mcnt = loff + kTileS;                              // [kTileS]
  __shared__ uint64_t s_tile, s_lb0, s_w, s_base;
  __shared__ uint64_t s_wcount[kWarps], s_wbase[kWarps];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const K* __restrict__ r = static_cast<const K*>(a.r);
  const K* __restrict__ s = static_cast<const K*>(a.s);
  while (true) {
    if (tid == 0) {
      const uint64_t t = atomicAdd(a.ticket, 1u);
      s_tile = t;
      if (t < a.tiles) {
        const uint64_t j0 = t * kTileS, j1 = dev::umin64(a.ns, j0 + kTileS);
        const uint64_t lb0 = g_lower_bound<K>(r, 0, a.nr, s[j0]);
        const uint64_t ub1 = g_upper_bound<K>(r, lb0, a.nr, s[j1 - 1]);
        s_lb0 = lb0;
        s_w = ub1 - lb0;
      }
    }
    __syncthreads();
    const uint64_t t = s_tile;
    if (t >= a.tiles) break;
    const uint64_t j0 = t * kTileS;
    const uint32_t nq = (uint32_t)dev::umin64(kTileS, a.ns - j0);
    const uint64_t lb0 = s_lb0, w = s_w;
    const bool windowed = w <= a.wmax;
    if (windowed)
      for (uint32_t i = tid; i < w; i += kThreads) rk[i] = r[lb0 + i];
    __syncthreads();

    const uint32_t rounds = (nq + 31) / 32;
    const uint32_t r0 = rounds * warp / kWarps, r1 = rounds * (warp + 1) / kWarps;
    uint64_t wc = 0;
    for (uint32_t rr = r0; rr < r1; ++rr) {
      const uint32_t jl = rr * 32 + lane;
      if (jl < nq) {
        const K k = s[j0 + jl];
        uint64_t lb, m = 0;
        if (windowed) {
          uint32_t lo = 0, hi = (uint32_t)w;
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (rk[mid] < k) lo = mid + 1; else hi = mid;
          }
          lb = lo;
          if (lo < w && rk[lo] == k) {
            if (a.pk_fk) {
              m = 1;
            } else {
              uint32_t lo2 = lo + 1, hi2 = (uint32_t)w;
              while (lo2 < hi2) {
                const uint32_t mid = (lo2 + hi2) >> 1;
                if (rk[mid] <= k) lo2 = mid + 1; else hi2 = mid;
              }
              m = lo2 - lo;
            }
          }
        } else {
          const uint64_t g = g_lower_bound<K>(r, lb0, lb0 + w, k);
          lb = g - lb0;
          if (g < a.nr && r[g] == k)
            m = a.pk_fk ? 1 : g_upper_bound<K>(r, g, lb0 + w, k) - g;
        }
        loff[jl] = (uint32_t)lb;
        mcnt[jl] = (uint32_t)m;
        wc += m;
      }
    }
    wc = dev::warp_sum(wc);
    if (lane == 0) s_wcount[warp] = wc;
    __syncthreads();
    if (warp == 0) {
      const uint64_t v = lane < kWarps ? s_wcount[lane] : 0;
      const uint64_t inc = dev::warp_inclusive_sum(v);
      if (lane < kWarps) s_wbase[lane] = inc - v;
      const uint64_t tot = __shfl_sync(0xffffffffu, inc, kWarps - 1);
      const uint64_t base = dev::warp_lookback(a.status, t, tot, a.epoch, a.err);
      if (lane == 0) {
        s_base = base;
        if (t == a.tiles - 1) *a.total_out = base + tot;
        if (a.write && base + tot > a.capacity) atomicOr(a.err, kErrOverflow);
      }
    }
    __syncthreads();
    if (a.write) {
      uint64_t o = s_base + s_wbase[warp];
      for (uint32_t rr = r0; rr < r1; ++rr) {
        const uint32_t jl = rr * 32 + lane;
        const uint32_t m = jl < nq ? mcnt[jl] : 0;
        const uint32_t inc = dev::warp_inclusive_sum(m);
        uint64_t oo = o + inc - m;
        if (m) {
          const uint64_t j = j0 + jl;
          const K k = s[j];
          const uint64_t i0 = lb0 + loff[jl];
          for (uint32_t q = 0; q < m; ++q, ++oo)
            if (oo < a.capacity) emit<K>(a, oo, i0 + q, j, k);
        }
        o += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
  }
}

// ---- TMA-pipelined count / fill (the default for run_join) ------------------
//
// Tiles of 2048 probe rows; a bounds kernel finds every tile's r window with
// one binary search per tile (all tiles in parallel).  Count and fill passes
// are persistent (one or two CTAs per SM, tile t_k = blockIdx + k * gridDim)
// and bulk-copy the window (keys + transformed R payloads) and the probe tile
// (keys + transformed S payloads) into a ring of shared-memory stages while
// earlier tiles are merged; nothing is chained across CTAs: counts -> scan ->
// fill.
constexpr int kTmaThreads = 512;
constexpr int kTmaWarps = kTmaThreads / 32;

struct SmjDesc {
  uint64_t r_lo, r_hi, s_lo, s_hi;
};

template <class K>
__global__ void k_smj_bounds(const K* __restrict__ r, uint64_t nr, const K* __restrict__ s,
                             uint64_t ns, uint64_t tiles, SmjDesc* __restrict__ desc,
                             uint64_t wide_lim, uint32_t* __restrict__ wide,
                             uint32_t* __restrict__ miss) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tiles;
       t += (uint64_t)gridDim.x * blockDim.x) {
    SmjDesc d;
    d.s_lo = t * kTileS;
    d.s_hi = dev::umin64(ns, d.s_lo + kTileS);
    d.r_lo = g_lower_bound<K>(r, 0, nr, s[d.s_lo]);
    d.r_hi = g_upper_bound<K>(r, d.r_lo, nr, s[d.s_hi - 1]);
    desc[t] = d;
    if (wide && d.r_hi - d.r_lo > wide_lim) atomicAdd(wide, 1u);
    // a tile's first or last probe key absent from r: not every probe matches
    // (the PK-FK speculation would fail; it is not tried)
    if (miss && (d.r_hi == d.r_lo || r[d.r_lo] != s[d.s_lo] || r[d.r_hi - 1] != s[d.s_hi - 1]))
      atomicOr(miss, 1u);
  }
}

// Galloping lower/upper bound in a shared-memory run starting at `from`
// (monotone probes: the next probe's bound is at or after the previous one).
template <class K, bool UPPER>
__device__ __forceinline__ uint32_t gallop(const K* __restrict__ r, uint32_t from, uint32_t n, K k) {
  auto before = [&](uint32_t i) { return UPPER ? !(k < r[i]) : r[i] < k; };
  if (from >= n || !before(from)) return from;
  uint32_t lo = from + 1, step = 1;  // r[lo - 1] is before k
  while (lo + step <= n && before(lo + step - 1)) {
    lo += step;
    step <<= 1;
  }
  uint32_t hi = min(n, lo + step - 1);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (before(mid)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Persistent CTAs take tiles of kTileS probe positions; each thread owns four
// consecutive probes (one binary search, then galloping), so a warp owns 128
// consecutive probes and emission keeps probe order.  WRITE=false: per-tile
// match counts and, for PK-FK tiles whose r window fits shared memory, the
// window index of every probe's match (match_e, 0xffff: none) so the fill pass
// skips the search and the r keys.  WRITE=true: compact the hits of the tile
// (list[t] = window idx << 16 | probe idx) and write column by column.
constexpr uint32_t kSmjPer = kTileS / kTmaThreads;  // probes per thread (4)
constexpr uint32_t kSmjList = 2 * kTileS;            // compacted rows per tile in shared memory

// Rows [0, cnt) of a tile's output at tbase, column by column, consecutive
// threads on consecutive output rows; row_of(t) = r window idx << 16 | probe idx.
template <class K, class RowOf>
__device__ __forceinline__ void smj_emit_rows(const SmjArgs& a, const SmjDesc& d, const uint8_t* st,
                                              const K* sk, uint64_t tbase, uint32_t cnt,
                                              RowOf row_of) {
  const int tid = threadIdx.x;
  const uint32_t ssh4 = (uint32_t)(d.s_lo & 3), ssh8 = (uint32_t)(d.s_lo & 1);
  const uint32_t rsh4 = (uint32_t)(d.r_lo & 3), rsh8 = (uint32_t)(d.r_lo & 1);
  if (tbase + cnt > a.capacity) cnt = tbase < a.capacity ? (uint32_t)(a.capacity - tbase) : 0u;
  constexpr int kE = kSmjList / kTmaThreads;
  uint32_t L[kE];
#pragma unroll
  for (int k = 0; k < kE; ++k) {
    const uint32_t tt = tid + k * kTmaThreads;
    L[k] = tt < cnt ? row_of(tt) : 0u;
  }
  auto each = [&](auto&& f) {
#pragma unroll
    for (int k = 0; k < kE; ++k) {
      const uint32_t tt = tid + k * kTmaThreads;
      if (tt < cnt) f(tbase + tt, L[k] >> 16, L[k] & 0xffffu);
    }
  };
  if (a.key_out) {
    K* ko = static_cast<K*>(a.key_out);
    each([&](uint64_t oo, uint32_t, uint32_t jl) { ko[oo] = sk[jl]; });
  }
  if (a.ids_r)
    each([&](uint64_t oo, uint32_t li, uint32_t) {
      const uint64_t i = d.r_lo + li;
      a.ids_r[oo] = a.carried_r ? a.carried_r[i] : (uint32_t)i;
    });
  if (a.ids_s)
    each([&](uint64_t oo, uint32_t, uint32_t jl) {
      const uint64_t j = d.s_lo + jl;
      a.ids_s[oo] = a.carried_s ? a.carried_s[j] : (uint32_t)j;
    });
  for (int c = 0; c < a.nr_cols; ++c) {
    if (a.r_bytes[c] == 4) {
      const uint32_t* sv = reinterpret_cast<const uint32_t*>(st + a.off_r[c]) + rsh4;
      uint32_t* dv = static_cast<uint32_t*>(a.r_dst[c]);
      each([&](uint64_t oo, uint32_t li, uint32_t) { dv[oo] = sv[li]; });
    } else {
      const uint64_t* sv = reinterpret_cast<const uint64_t*>(st + a.off_r[c]) + rsh8;
      uint64_t* dv = static_cast<uint64_t*>(a.r_dst[c]);
      each([&](uint64_t oo, uint32_t li, uint32_t) { dv[oo] = sv[li]; });
    }
  }
  for (int c = 0; c < a.ns_cols; ++c) {
    if (a.s_bytes[c] == 4) {
      const uint32_t* sv = reinterpret_cast<const uint32_t*>(st + a.off_s[c]) + ssh4;
      uint32_t* dv = static_cast<uint32_t*>(a.s_dst[c]);
      each([&](uint64_t oo, uint32_t, uint32_t jl) { dv[oo] = sv[jl]; });
    } else {
      const uint64_t* sv = reinterpret_cast<const uint64_t*>(st + a.off_s[c]) + ssh8;
      uint64_t* dv = static_cast<uint64_t*>(a.s_dst[c]);
      each([&](uint64_t oo, uint32_t, uint32_t jl) { dv[oo] = sv[jl]; });
    }
  }
}

// Warp-specialised: warp kTmaWarps (the producer) walks this CTA's tiles, reads
// each tile's descriptor (and, in the fill, the count pass's total and offset)
// into shared memory and bulk-copies the tile into a free stage; the 16
// consumer warps take stages as their copies land (full barriers) and hand
// them back per warp (empty barriers), so a warp that finishes a tile early
// starts the next one instead of waiting for the slowest warp.  Consumer-wide
// steps of the general path synchronise on named barrier 1 (512 threads).
constexpr int kSmjMaxStages = 4;

template <class K, bool WRITE>
__global__ void __launch_bounds__(kTmaThreads + 32, 1) k_smj_tma(const __grid_constant__ SmjArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int NS = a.nstages;
  uint32_t* loff = reinterpret_cast<uint32_t*>(smem + NS * (size_t)a.stage_bytes);
  uint32_t* mcnt = loff + kTileS;
  uint32_t* list = mcnt + kTileS;  // [kSmjList] (WRITE)
  __shared__ SmjDesc s_desc[kSmjMaxStages];
  __shared__ bool s_pre[kSmjMaxStages];
  __shared__ uint64_t s_fcnt[kSmjMaxStages], s_fbase[kSmjMaxStages];
  __shared__ int s_abort[kSmjMaxStages];  // speculative fill: the producer stopped at this stage
  __shared__ __align__(8) uint64_t full[kSmjMaxStages], empty[kSmjMaxStages];
  __shared__ uint64_t s_wcnt[2][kTmaWarps], s_wb[2][kTmaWarps];  // by tile parity
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const SmjDesc* __restrict__ descs = static_cast<const SmjDesc*>(a.desc);
  const K* __restrict__ rg = static_cast<const K*>(a.r);
  const uint32_t kb = sizeof(K);
  const uint64_t g = gridDim.x;
  auto bytes = [&](uint64_t lo, uint64_t hi, uint32_t w) {
    return hi > lo ? (uint32_t)((dev::align_hi(hi, w) - dev::align_lo(lo, w)) * w) : 0u;
  };
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      dev::mbar_init(&full[i], 1);
      dev::mbar_init(&empty[i], kTmaWarps);
    }
    dev::fence_mbar_init();
  }
  __syncthreads();

  if (warp == kTmaWarps) {  // ---- producer ----
    if (lane != 0) return;
    // what a tile's staging needs from global memory, loaded one tile ahead
    // so the loads' latency overlaps the previous tile's wait and issue
    struct Pf {
      SmjDesc d;
      uint32_t pre;
      uint64_t cnt, base;
    };
    auto fetch = [&](uint64_t tt) {
      Pf p;
      p.d = descs[tt];
      p.pre = WRITE && a.match_e != nullptr ? a.tile_pre[tt] : 0u;
      p.cnt = WRITE && a.tile_counts != nullptr ? a.tile_counts[tt] : ~0ull;
      p.base = WRITE && a.tile_counts != nullptr ? a.tile_off[tt] : 0ull;
      return p;
    };
    Pf nx{};
    if (blockIdx.x < a.tiles) nx = fetch(blockIdx.x);
    uint32_t k = 0;
    int pb = 0;
    uint32_t pr = 0;
    for (uint64_t t = blockIdx.x; t < a.tiles; t += g, ++k) {
      const Pf cur = nx;
      if (t + g < a.tiles) nx = fetch(t + g);
      // stage b of round r = k / NS (kept incrementally: no division per tile)
      const int b = pb;
      if (k >= (uint32_t)NS) dev::mbar_wait(&empty[b], pr ^ 1u);
      if (++pb == NS) {
        pb = 0;
        pr ^= 1u;
      }
      const SmjDesc d = cur.d;
      if (WRITE && a.spec_fail && *reinterpret_cast<volatile uint32_t*>(a.spec_fail)) {
        // a tile failed the speculation: wake the consumers on this stage and stop
        s_abort[b] = 1;
        dev::mbar_arrive(&full[b]);
        return;
      }
      s_abort[b] = 0;
      const bool pre = cur.pre != 0;
      s_desc[b] = d;
      s_pre[b] = pre;
      if (WRITE) {
        s_fcnt[b] = pre ? cur.cnt : ~0ull;
        s_fbase[b] = cur.base;
      }
      uint8_t* st = smem + (size_t)b * a.stage_bytes;
      const bool win = d.r_hi - d.r_lo <= a.wmax;
      uint32_t total = bytes(d.s_lo, d.s_hi, kb);
      if (win && !pre) total += bytes(d.r_lo, d.r_hi, kb);
      if (WRITE) {
        if (win)
          for (int c = 0; c < a.nr_cols; ++c) total += bytes(d.r_lo, d.r_hi, a.r_bytes[c]);
        for (int c = 0; c < a.ns_cols; ++c) total += bytes(d.s_lo, d.s_hi, a.s_bytes[c]);
        if (pre) total += bytes(d.s_lo, d.s_hi, 2);
      }
      dev::fence_proxy_async();
      dev::mbar_expect_tx(&full[b], total);
      auto copy = [&](uint32_t off, const void* base, uint64_t lo, uint64_t hi, uint32_t w) {
        if (hi > lo)
          dev::tma_load_1d(st + off, static_cast<const uint8_t*>(base) + dev::align_lo(lo, w) * w,
                           bytes(lo, hi, w), &full[b]);
      };
      copy(a.off_sk, a.s, d.s_lo, d.s_hi, kb);
      if (win && !pre) copy(a.off_rk, a.r, d.r_lo, d.r_hi, kb);
      if (WRITE) {
        if (win)
          for (int c = 0; c < a.nr_cols; ++c) copy(a.off_r[c], a.r_src[c], d.r_lo, d.r_hi, a.r_bytes[c]);
        for (int c = 0; c < a.ns_cols; ++c) copy(a.off_s[c], a.s_src[c], d.s_lo, d.s_hi, a.s_bytes[c]);
        if (pre) copy(a.off_e, a.match_e, d.s_lo, d.s_hi, 2);
      }
    }
    return;
  }

  // ---- consumers ----
  auto consumers_sync = [] { dev::named_bar(1, kTmaThreads); };
  auto release = [&](int b) {  // this warp is done with stage b
    __syncwarp();
    if (lane == 0) dev::mbar_arrive(&empty[b]);
  };
  uint32_t k = 0;
  int cb = 0;
  uint32_t cr = 0;
  for (uint64_t t = blockIdx.x; t < a.tiles; t += g, ++k) {
    const int b = cb;
    const uint32_t cphase = cr;
    if (++cb == NS) {
      cb = 0;
      cr ^= 1u;
    }
    const int par = (int)(k & 1u);
    uint64_t* s_wcount = s_wcnt[par];
    uint64_t* s_wbase = s_wb[par];
    dev::mbar_wait(&full[b], cphase);
    const SmjDesc d = s_desc[b];
    if (WRITE && s_abort[b]) break;  // the speculation failed: the producer stopped
    const bool pre = s_pre[b];
    // the speculative fill alternates its lower bounds between loff and the
    // list region by tile parity, so a tile needs no barrier at its end
    uint32_t* const lw = WRITE && a.spec_fail && par ? list : loff;
    uint64_t tile_base = 0;
    if (WRITE && tid == 32) tile_base = a.spec_fail ? d.s_lo : a.tile_off[t];
    uint8_t* st = smem + (size_t)b * a.stage_bytes;
    const uint32_t nq = (uint32_t)(d.s_hi - d.s_lo);
    const uint64_t w = d.r_hi - d.r_lo;
    const bool win = w <= a.wmax;
    const K* sk = reinterpret_cast<const K*>(st + a.off_sk) + (d.s_lo - dev::align_lo(d.s_lo, kb));
    const K* rk = reinterpret_cast<const K*>(st + a.off_rk) + (d.r_lo - dev::align_lo(d.r_lo, kb));
    // the count pass's tile total: every probe matched once (PK-FK tile whose
    // r window is staged; the count pass may take wider windows) -> the
    // output rows are the probe rows in order, their r rows are match_e; no
    // bounds, scan or compaction
    const uint64_t fcnt = WRITE && pre && win ? s_fcnt[b] : ~0ull;
    if (WRITE && fcnt == nq) {
      const uint16_t* me = reinterpret_cast<const uint16_t*>(st + a.off_e) +
                           (d.s_lo - dev::align_lo(d.s_lo, 2));
      smj_emit_rows<K>(a, d, st, sk, s_fbase[b], nq,
                       [&](uint32_t tt) { return ((uint32_t)me[tt] << 16) | tt; });
      release(b);
      continue;
    }

    // 1. bounds of this thread's four probes
    const uint32_t j0 = tid * kSmjPer;
    uint32_t tsum = 0;
    if (pre) {
      const uint16_t* me = reinterpret_cast<const uint16_t*>(st + a.off_e) +
                           (d.s_lo - dev::align_lo(d.s_lo, 2));
#pragma unroll
      for (uint32_t q = 0; q < kSmjPer; ++q) {
        const uint32_t jl = j0 + q;
        const uint32_t e = jl < nq ? me[jl] : 0xffffu;
        lw[jl] = e;
        mcnt[jl] = e != 0xffffu;
        tsum += e != 0xffffu;
      }
    } else if (win) {
      uint32_t lb = 0;
      uint16_t e16[kSmjPer];
      // a PK-FK window of consecutive keys (dense surrogate keys): key k sits
      // at k - rk[0]; no search.  Sorted + span w - 1 means gap-free only
      // when the keys are unique, so the shortcut is PK-FK only (a non-PK
      // window [5,5,7] has the span of [5,6,7]), and each hit is verified as
      // the lower bound (rk[i] == k, rk[i-1] < k) so a build mislabelled
      // unique falls back to the search and keeps merge_match.cpp:65-68's
      // lower-bound emission.
      const K rlo = w ? rk[0] : K(0);
      const bool dense = a.pk_fk && w > 0 && (uint64_t)(rk[w - 1] - rlo) == w - 1;
      bool searched = false;  // lb is a valid galloping start for later probes
#pragma unroll
      for (uint32_t q = 0; q < kSmjPer; ++q) {
        const uint32_t jl = j0 + q;
        e16[q] = 0xffffu;
        bool done = false;
        if (jl < nq && dense) {
          const K k = sk[jl];
          const bool inr = k >= rlo && (uint64_t)(k - rlo) < w;
          const uint32_t i = inr ? (uint32_t)(k - rlo) : 0u;
          const bool hit = inr && rk[i] == k && (i == 0 || rk[i - 1] < k);
          if (hit || !inr) {
            lb = k < rlo ? 0u : (hit ? i : (uint32_t)w);
            lw[jl] = lb;
            mcnt[jl] = hit;
            tsum += hit;
            e16[q] = hit ? (uint16_t)lb : (uint16_t)0xffffu;
            searched = true;
            done = true;
          }
        }
        if (jl < nq && !done) {
          const K k = sk[jl];
          if (!searched) {
            searched = true;
            // interpolate between the window's end keys (exact on dense
            // keys), then gallop to the lower bound from below
            uint32_t g = 0;
            const K r0 = w ? rk[0] : K(0), r1 = w ? rk[w - 1] : K(0);
            if (w > 1 && k > r0 && r1 > r0) {
              const float f = (float)(k - r0) / (float)(r1 - r0);
              g = (uint32_t)fminf((float)(w - 1), f * (float)(w - 1));
              // step back until rk[g] < k (or g = 0) so galloping stays monotone
              uint32_t back = 1;
              while (g > 0 && !(rk[g] < k)) {
                g = g > back ? g - back : 0;
                back <<= 1;
              }
            }
            lb = gallop<K, false>(rk, g, (uint32_t)w, k);
          } else {
            lb = gallop<K, false>(rk, lb, (uint32_t)w, k);
          }
          uint32_t m = 0;
          if (lb < w && rk[lb] == k) m = a.pk_fk ? 1u : gallop<K, true>(rk, lb, (uint32_t)w, k) - lb;
          lw[jl] = lb;
          mcnt[jl] = m;
          tsum += m;
          e16[q] = (uint16_t)(m ? lb : 0xffffu);
        }
      }
      if (!WRITE && a.match_e) {  // four u16 hand-off entries in one 8-byte store
        if (j0 + kSmjPer <= nq)
          *reinterpret_cast<uint2*>(a.match_e + d.s_lo + j0) =
              make_uint2(e16[0] | ((uint32_t)e16[1] << 16), e16[2] | ((uint32_t)e16[3] << 16));
        else
          for (uint32_t q = 0; q < kSmjPer && j0 + q < nq; ++q) a.match_e[d.s_lo + j0 + q] = e16[q];
      }
    } else {  // window beyond shared memory: global binary searches
#pragma unroll
      for (uint32_t q = 0; q < kSmjPer; ++q) {
        const uint32_t jl = j0 + q;
        if (jl < nq) {
          const K k = sk[jl];
          const uint64_t g = g_lower_bound<K>(rg, d.r_lo, d.r_hi, k);
          uint64_t m = 0;
          if (g < d.r_hi && rg[g] == k) m = a.pk_fk ? 1 : g_upper_bound<K>(rg, g, d.r_hi, k) - g;
          lw[jl] = (uint32_t)(g - d.r_lo);
          mcnt[jl] = (uint32_t)m;
          tsum += (uint32_t)m;
        }
      }
    }
    if (!WRITE && a.match_e && tid == 0) a.tile_pre[t] = (a.pk_fk && win) ? 1 : 0;
    if (WRITE && a.spec_fail) {
      // speculation: unique build keys match a probe at most once, so the tile
      // holds iff no thread saw a miss among its probes — one OR-barrier, no
      // count or scan; the output rows are then the probe rows in order
      uint32_t mine = 0;
#pragma unroll
      for (uint32_t q = 0; q < kSmjPer; ++q) mine += j0 + q < nq ? 1u : 0u;
      if (dev::named_bar_or(1, kTmaThreads, tsum != mine)) {
        if (tid == 0) atomicExch(a.spec_fail, 1u);
        release(b);
        continue;  // loff / mcnt are not read again
      }
      if (tid == 0) atomicAdd(a.spec_rows, nq);
      if (win) {
        smj_emit_rows<K>(a, d, st, sk, d.s_lo, nq, [&](uint32_t tt) { return (lw[tt] << 16) | tt; });
        release(b);
        continue;
      }
      // a window beyond shared memory: the general emission below, at d.s_lo
    }
    const uint32_t tinc = dev::warp_inclusive_sum(tsum);
    if (lane == 31) s_wcount[warp] = tinc;
    consumers_sync();
    if (!WRITE) release(b);  // the count pass reads the stage no further
    if (warp == 1) {
      const uint64_t v = lane < kTmaWarps ? s_wcount[lane] : 0;
      const uint64_t inc = dev::warp_inclusive_sum(v);
      const uint64_t base = __shfl_sync(0xffffffffu, tile_base, 0);
      if (lane < kTmaWarps) s_wbase[lane] = base + inc - v;
      if (!WRITE && lane == kTmaWarps - 1) a.tile_counts[t] = inc;
    }
    if (!WRITE) continue;
    consumers_sync();
    const uint32_t ssh4 = (uint32_t)(d.s_lo & 3), ssh8 = (uint32_t)(d.s_lo & 1);
    const uint32_t rsh4 = (uint32_t)(d.r_lo & 3), rsh8 = (uint32_t)(d.r_lo & 1);
    const uint64_t tbase = s_wbase[0];
    const uint64_t tcount = s_wbase[kTmaWarps - 1] + s_wcount[kTmaWarps - 1] - tbase;
    if (win && tcount <= kSmjList) {
      // every probe matched exactly once (PK-FK, match ratio 1): output row t
      // is probe t, its r row loff[t]; no compaction needed
      const bool ident = a.pk_fk && tcount == nq;
      if (!ident) {
        // 2a. compact in (probe, r) order
        uint32_t o = (uint32_t)(s_wbase[warp] - tbase) + tinc - tsum;
        for (uint32_t q = 0; q < kSmjPer; ++q) {
          const uint32_t jl = j0 + q;
          if (jl < nq) {
            const uint32_t m = mcnt[jl], l0 = lw[jl];
            for (uint32_t i = 0; i < m; ++i) list[o++] = ((l0 + i) << 16) | jl;
          }
        }
        consumers_sync();
      }
      // 2b. column by column, consecutive threads on consecutive output rows
      const uint32_t* lst = list;
      const uint32_t* lof = lw;
      if (ident)
        smj_emit_rows<K>(a, d, st, sk, tbase, (uint32_t)tcount,
                         [&](uint32_t tt) { return (lof[tt] << 16) | tt; });
      else
        smj_emit_rows<K>(a, d, st, sk, tbase, (uint32_t)tcount, [&](uint32_t tt) { return lst[tt]; });
      release(b);
      consumers_sync();  // loff / mcnt / list are rewritten by the next tile
      continue;
    }
    // general: per probe, its whole r run, in rounds of 32 probe rows over the
    // same probes whose matches s_wbase[warp] counted (the warp's 32 * kSmjPer
    // rows; a partial last tile must not redistribute them)
    const uint32_t r0 = (uint32_t)warp * kSmjPer, r1 = r0 + kSmjPer;
    uint64_t o = s_wbase[warp];
    for (uint32_t rr = r0; rr < r1; ++rr) {
      const uint32_t jl = rr * 32 + lane;
      const uint32_t m = jl < nq ? mcnt[jl] : 0;
      const uint32_t inc = dev::warp_inclusive_sum(m);
      uint64_t oo = o + inc - m;
      if (m) {
        const uint64_t j = d.s_lo + jl;
        const K k = sk[jl];
        const uint32_t l0 = lw[jl];
        for (uint32_t q = 0; q < m; ++q, ++oo) {
          if (oo >= a.capacity) continue;
          const uint32_t li = l0 + q;
          const uint64_t i = d.r_lo + li;
          if (a.key_out) static_cast<K*>(a.key_out)[oo] = k;
          if (a.ids_r) a.ids_r[oo] = a.carried_r ? a.carried_r[i] : (uint32_t)i;
          if (a.ids_s) a.ids_s[oo] = a.carried_s ? a.carried_s[j] : (uint32_t)j;
          for (int c = 0; c < a.nr_cols; ++c) {
            if (a.r_bytes[c] == 4)
              static_cast<uint32_t*>(a.r_dst[c])[oo] =
                  win ? reinterpret_cast<const uint32_t*>(st + a.off_r[c])[rsh4 + li]
                      : static_cast<const uint32_t*>(a.r_src[c])[i];
            else
              static_cast<uint64_t*>(a.r_dst[c])[oo] =
                  win ? reinterpret_cast<const uint64_t*>(st + a.off_r[c])[rsh8 + li]
                      : static_cast<const uint64_t*>(a.r_src[c])[i];
          }
          for (int c = 0; c < a.ns_cols; ++c) {
            if (a.s_bytes[c] == 4)
              static_cast<uint32_t*>(a.s_dst[c])[oo] =
                  reinterpret_cast<const uint32_t*>(st + a.off_s[c])[ssh4 + jl];
            else
              static_cast<uint64_t*>(a.s_dst[c])[oo] =
                  reinterpret_cast<const uint64_t*>(st + a.off_s[c])[ssh8 + jl];
          }
        }
      }
      o += __shfl_sync(0xffffffffu, inc, 31);
    }
    release(b);
    consumers_sync();
  }
}

template <class K>
size_t smj_layout_w(SmjArgs& a, bool write, uint32_t wmax) {
  auto up = [](size_t x) { return (x + 127) & ~size_t(127); };
  const uint32_t kb = sizeof(K);
  const uint32_t kWinMax = wmax;
  a.wmax = wmax;
  size_t off = 0;
  a.off_rk = (uint32_t)off;
  off = up(off + (size_t)(kWinMax + 8) * kb);
  if (write)
    for (int c = 0; c < a.nr_cols; ++c) {
      a.off_r[c] = (uint32_t)off;
      off = up(off + (size_t)(kWinMax + 8) * a.r_bytes[c]);
    }
  a.off_sk = (uint32_t)off;
  off = up(off + (size_t)(kTileS + 8) * kb);
  if (write)
    for (int c = 0; c < a.ns_cols; ++c) {
      a.off_s[c] = (uint32_t)off;
      off = up(off + (size_t)(kTileS + 8) * a.s_bytes[c]);
    }
  if (write && a.match_e) {
    a.off_e = (uint32_t)off;
    off = up(off + (size_t)(kTileS + 8) * 2);
  }
  a.stage_bytes = (uint32_t)off;
  // loff + mcnt [kTileS] each, list [kSmjList] (fill)
  return (size_t)a.nstages * off + 2 * sizeof(uint32_t) * kTileS +
         (write ? sizeof(uint32_t) * kSmjList : 0);
}

// Largest r window (shared-memory keys + R payloads) whose two stages fit.
template <class K>
size_t smj_layout(SmjArgs& a, bool write, int stages = 2) {
  // fill: `stages` (3 keeps two tiles in flight behind the one being emitted
  // but caps the staged r window at 2048 keys); count: two (two CTAs per SM);
  // fewer when the rows are too wide
  const char* e = std::getenv("CJ_SMJ_STAGES");
  const int want = e ? std::max(2, std::min(kSmjMaxStages, std::atoi(e))) : (write ? stages : 2);
  size_t smem = 0;
  for (a.nstages = want; a.nstages >= 2; --a.nstages) {
    for (uint32_t w : {4096u, 2048u, 1024u, 512u}) {
      smem = smj_layout_w<K>(a, write, w);
      if (smem <= 200 * 1024) return smem;
    }
  }
  a.nstages = 2;
  return smj_layout_w<K>(a, write, 512);
}

template <class K>
uint64_t run(cj_ctx* ctx, SmjArgs a);

template <class K>
uint64_t run_tma(cj_ctx* ctx, SmjArgs a) {
  if (a.write) {
    // rows too wide for two staged 2048-row probe tiles (many payload
    // columns): the general kernel, which reads the columns in place
    SmjArgs t = a;
    t.match_e = reinterpret_cast<uint16_t*>(16);  // the widest layout (with the hand-off)
    t.nstages = 2;
    if (smj_layout_w<K>(t, true, 512) > 220 * 1024) return run<K>(ctx, a);
  }
  a.tiles = (a.ns + kTileS - 1) / kTileS;
  Scratch tot(ctx, 8);
  CJ_CUDA(cudaMemsetAsync(tot.p, 0, 8, ctx->stream));
  if (a.tiles == 0 || a.nr == 0) return 0;
  Scratch desc(ctx, a.tiles * sizeof(SmjDesc)), counts(ctx, a.tiles * 8), offs(ctx, a.tiles * 8);
  a.desc = desc.p;
  // PK-FK: the count pass hands every probe's window index to the fill pass
  const char* he = std::getenv("CJ_FIND_HANDOFF");
  const bool handoff = a.write && a.pk_fk && a.padded && !(he && std::strcmp(he, "0") == 0);
  Scratch me(ctx, handoff ? a.ns * 2 + kPad : 0), pre(ctx, handoff ? a.tiles + 16 : 0);
  if (handoff) {
    a.match_e = me.as<uint16_t>();
    a.tile_pre = pre.as<uint8_t>();
  }
  ctx->kbegin("smj_bounds", a.tiles * (2 * sizeof(K) + 32));
  // tiles whose r window needs the 4096-key stages (skewed or sparse probes):
  // the fill takes three stages only when they are rare
  uint32_t* wide = ctx->ticket(4);
  uint32_t* miss = ctx->ticket(8);
  k_smj_bounds<K><<<grid_for(a.tiles, 128, 4096), 128, 0, ctx->stream>>>(
      static_cast<const K*>(a.r), a.nr, static_cast<const K*>(a.s), a.ns, a.tiles,
      desc.as<SmjDesc>(), 2048, a.write ? wide : nullptr, a.write && a.pk_fk ? miss : nullptr);
  ctx->kend();
  int fill_stages = 2;
  bool boundary_miss = true;
  if (a.write) {
    CJ_CUDA(cudaMemcpyAsync(ctx->host_pinned, wide, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CJ_CUDA(cudaMemcpyAsync(ctx->host_pinned + 1, miss, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    fill_stages = (uint64_t)ctx->host_pinned[0] * 64 <= a.tiles ? 3 : 2;
    boundary_miss = ctx->host_pinned[1] != 0;
  }
  // PK-FK speculation: one fill pass, each tile at its first probe row; a miss
  // anywhere falls back to count + fill below (CJ_SPECULATE=0: off)
  const char* se = std::getenv("CJ_SPECULATE");
  if (a.write && a.pk_fk && !boundary_miss && a.capacity >= a.ns &&
      !(se && std::strcmp(se, "0") == 0)) {
    SmjArgs as = a;
    as.match_e = nullptr;
    as.tile_pre = nullptr;
    as.tile_counts = nullptr;
    as.tile_off = nullptr;
    as.spec_fail = ctx->ticket(6);
    as.spec_rows = ctx->ticket(7);
    const size_t smem_s = smj_layout<K>(as, true, fill_stages);
    if (smem_s <= 220 * 1024) {
      CJ_CUDA(cudaFuncSetAttribute(k_smj_tma<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_s));
      const unsigned grid_s = (unsigned)std::min<uint64_t>((uint64_t)ctx->num_sms, a.tiles);
      ctx->kbegin("smj_find", 0);
      k_smj_tma<K, true><<<grid_s, kTmaThreads + 32, smem_s, ctx->stream>>>(as);
      ctx->kend();
      CJ_CUDA(cudaGetLastError());
      uint32_t* h = ctx->host_pinned;
      CJ_CUDA(cudaMemcpyAsync(h, as.spec_fail, 4, cudaMemcpyDeviceToHost, ctx->stream));
      CJ_CUDA(cudaMemcpyAsync(h + 1, as.spec_rows, 4, cudaMemcpyDeviceToHost, ctx->stream));
      CJ_CUDA(cudaMemcpyAsync(h + 2, ctx->err_word, 4, cudaMemcpyDeviceToHost, ctx->stream));
      CJ_CUDA(cudaStreamSynchronize(ctx->stream));
      if (h[0] == 0 && h[1] == a.ns) {
        ctx->err_known_clean = h[2] == 0;
        return a.ns;
      }
    }
  }
  SmjArgs ac = a;
  ac.tile_counts = counts.as<uint64_t>();
  const size_t smem_c = smj_layout<K>(ac, false);
  const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)ctx->num_sms, a.tiles);
  CJ_CUDA(cudaFuncSetAttribute(k_smj_tma<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem_c));
  int per_sm = 1;
  CJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_smj_tma<K, false>, kTmaThreads + 32,
                                                        smem_c));
  const unsigned grid_c = (unsigned)std::min<uint64_t>(
      (uint64_t)ctx->num_sms * std::max(1, std::min(per_sm, 2)), a.tiles);
  ctx->kbegin("smj_count", sizeof(K) * (a.nr + a.ns));
  k_smj_tma<K, false><<<grid_c, kTmaThreads + 32, smem_c, ctx->stream>>>(ac);
  ctx->kend();
  scan_counts(ctx, counts.as<uint64_t>(), a.tiles, offs.as<uint64_t>(), tot.as<uint64_t>());
  CJ_CUDA(cudaGetLastError());
  if (a.write) {
    // launched without waiting for the total: writes are bounded by the
    // capacity on the device; an overflow is reported after the one sync below
    a.tile_off = offs.as<uint64_t>();
    const char* ff = std::getenv("CJ_FIND_FAST");
    a.tile_counts = handoff && !(ff && std::strcmp(ff, "0") == 0) ? counts.as<uint64_t>() : nullptr;
    const size_t smem = smj_layout<K>(a, true, fill_stages);
    if (smem > 220 * 1024) fail(CJ_ERR_UNSUPPORTED, "merge join stage exceeds shared memory");
    CJ_CUDA(cudaFuncSetAttribute(k_smj_tma<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    ctx->kbegin("smj_find", 0);
    k_smj_tma<K, true><<<grid, kTmaThreads + 32, smem, ctx->stream>>>(a);
    ctx->kend();
    CJ_CUDA(cudaGetLastError());
  }
  uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  CJ_CUDA(cudaMemcpyAsync(h, tot.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  const uint64_t total = h[0];
  if (a.write && total > a.capacity) {
    const uint32_t v = kErrOverflow;
    CJ_CUDA(cudaMemcpyAsync(ctx->err_word, &v, 4, cudaMemcpyHostToDevice, ctx->stream));
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return total;
}

template <class K>
__global__ void k_check_sorted(const K* __restrict__ v, uint64_t n, int strict,
                               uint32_t* err, uint32_t code) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const K a = v[i - 1], b = v[i];
    if (strict ? !(a < b) : (a > b)) {
      atomicOr(err, code);
      return;
    }
  }
}

template <class K>
uint64_t run(cj_ctx* ctx, SmjArgs a) {
  a.tiles = (a.ns + kTileS - 1) / kTileS;
  Scratch tot(ctx, sizeof(uint64_t));
  CJ_CUDA(cudaMemsetAsync(tot.p, 0, sizeof(uint64_t), ctx->stream));
  a.total_out = tot.as<uint64_t>();
  if (a.tiles > 0 && a.nr > 0) {
    a.status = ctx->status_buffer(a.tiles);
    a.epoch = ctx->next_epoch();
    a.ticket = ctx->ticket(2);
    a.err = ctx->err_word;
    a.wmax = 8192;
    const size_t smem = (size_t)a.wmax * sizeof(K) + 2 * sizeof(uint32_t) * kTileS;
    CJ_CUDA(cudaFuncSetAttribute(k_smj_find<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    int per_sm = 0;
    CJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_smj_find<K>, kThreads, smem));
    per_sm = std::max(per_sm, 1);
    const uint64_t grid = std::min<uint64_t>((uint64_t)ctx->num_sms * per_sm, a.tiles);
    ctx->kbegin(a.write ? "smj_find" : "smj_count", 0);
    k_smj_find<K><<<(unsigned)grid, kThreads, smem, ctx->stream>>>(a);
    ctx->kend();
    CJ_CUDA(cudaGetLastError());
  }
  uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  CJ_CUDA(cudaMemcpyAsync(h, tot.p, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  return h[0];
}

SmjArgs base(const void* rkeys, uint64_t nr, const void* skeys, uint64_t ns, bool pk_fk) {
  SmjArgs a{};
  a.r = rkeys;
  a.nr = nr;
  a.s = skeys;
  a.ns = ns;
  a.pk_fk = pk_fk ? 1 : 0;
  return a;
}

}  // namespace

uint64_t smj_find(cj_ctx* ctx, const void* rkeys, uint64_t nr, const void* skeys, uint64_t ns,
                  int key_bytes, bool pk_fk, const OutSpec& out, uint64_t capacity) {
  SmjArgs a = base(rkeys, nr, skeys, ns, pk_fk);
  a.write = 1;
  a.capacity = capacity;
  a.key_out = out.key;
  a.ids_r = out.ids_r;
  a.ids_s = out.ids_s;
  a.carried_r = out.carried_r;
  a.carried_s = out.carried_s;
  a.nr_cols = out.nr;
  a.ns_cols = out.ns;
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
  a.padded = out.padded ? 1 : 0;
  const char* mode = std::getenv("CJ_FIND");
  const bool tma = a.padded && !(mode && std::strcmp(mode, "ldg") == 0);
  uint64_t t;
  if (tma) t = key_bytes == 4 ? run_tma<uint32_t>(ctx, a) : run_tma<uint64_t>(ctx, a);
  else t = key_bytes == 4 ? run<uint32_t>(ctx, a) : run<uint64_t>(ctx, a);
  raise_device_errors(ctx);
  return t;
}

uint64_t smj_count(cj_ctx* ctx, const void* rkeys, uint64_t nr, const void* skeys, uint64_t ns,
                   int key_bytes, bool pk_fk) {
  SmjArgs a = base(rkeys, nr, skeys, ns, pk_fk);
  a.write = 0;
  return key_bytes == 4 ? run<uint32_t>(ctx, a) : run<uint64_t>(ctx, a);
}

void check_sorted(cj_ctx* ctx, const void* keys, uint64_t n, int key_bytes, bool strict,
                  int err_code, const char* what) {
  if (n < 2) return;
  const uint32_t code = err_code == CJ_ERR_NOT_SORTED ? kErrNotSorted : kErrDupKeys;
  const unsigned grid = grid_for(n, 256 * 8, ctx->num_sms * 8);
  ctx->kbegin("check_sorted", n * key_bytes);
  if (key_bytes == 4)
    k_check_sorted<uint32_t><<<grid, 256, 0, ctx->stream>>>(static_cast<const uint32_t*>(keys), n,
                                                           strict, ctx->err_word, code);
  else
    k_check_sorted<uint64_t><<<grid, 256, 0, ctx->stream>>>(static_cast<const uint64_t*>(keys), n,
                                                           strict, ctx->err_word, code);
  ctx->kend();
  CJ_CUDA(cudaGetLastError());
  (void)what;
  raise_device_errors(ctx);
}

}  // namespace cj
