// Radix histogram, stable onesweep partition pass, LSD driver and layout
// offsets — the transform phase of both PHJ and SMJ.
//
// Reference semantics (paths relative to the reference's proj/):
//   histogram_kernel / digit_totals   primitives.cpp:33-46, 169-205
//   scatter_starts / scatter_pairs    primitives.cpp:51-97   (stable cursors)
//   radix_pass / lsd_passes           primitives.cpp:117-139, 217-256
//   wide_offsets / finish_layout      hash_match.cpp:30-62
//
// Design (B200): one read of the keys computes the digit counts of every pass
// (K1).  Each pass (K3) is a single onesweep kernel: a CTA takes the next tile
// ticket, ranks its keys stably with warp match-any (input order is kept within
// a digit across lanes, item rounds and warps), publishes its per-digit counts
// and resolves its global cursors by decoupled look-back over earlier tiles
// (K2), stages keys and then every carried column in shared memory in digit
// order, and writes each digit run contiguously.  Output equals the reference's
// stable counting sort bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <vector>

#include "cj_device.cuh"
#include "cj_internal.cuh"

namespace cj {
namespace {

using dev::kFlagAgg;
using dev::kFlagIncl;
using dev::kValMask;

constexpr int kHistThreads = 512;
constexpr int kHistWarps = kHistThreads / 32;
constexpr int kHistSub = 4;  // CTAs per static block in the counting kernel

// Per-block digit counts of every pass in one read of the keys.  Block b owns
// the contiguous tile range [b*tiles/nblocks, (b+1)*tiles/nblocks) — the same
// static ranges the scatter kernel walks — so the counts double as the
// scatter's cross-block cursors (no look-back).  cnt[b][p][d].
struct HistArgs {
  uint64_t n, tile, tiles;
  uint32_t nblocks, hparts;
  uint32_t lowbits;  // shard mode: digit = shard << lowbits | low key bits
  uint32_t shift[8], mask[8];
  unsigned long long* key_or;  // optional: OR of every key (the join's dense-key test)
  // optional: the last CTA to finish also writes the digit totals and
  // exclusive bases of every pass (digit_bases_block; no launch of its own)
  uint32_t* done;              // zeroed CTA ticket
  uint32_t* totals;
  uint64_t* base;
};

// Totals and exclusive digit bases per pass from the per-block counts
// cnt[b][p][d], by one CTA (blockDim.x >= radix): thread (d, q) sums the
// blocks b = q (mod split) of digit d for every pass at once (split =
// blockDim / radix independent load streams, NP loads per block in flight),
// then threads q = 0 scan the digits pass by pass.  part: blockDim words,
// warp_tot: radix / 32 words of shared memory.
template <int NP>
__device__ __forceinline__ void digit_bases_block(const uint32_t* __restrict__ cnt, uint32_t nblocks,
                                                  uint32_t radix, uint32_t* __restrict__ totals,
                                                  uint64_t* __restrict__ base, uint32_t* part,
                                                  uint64_t* warp_tot) {
  const uint32_t split = blockDim.x / radix;
  const uint32_t d = threadIdx.x % radix, q = threadIdx.x / radix;
  uint32_t cq[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) cq[p] = 0;
  if (q < split) {
#pragma unroll 4
    for (uint32_t b = q; b < nblocks; b += split) {
#pragma unroll
      for (int p = 0; p < NP; ++p) cq[p] += __ldcg(cnt + ((uint64_t)b * NP + p) * radix + d);
    }
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    part[threadIdx.x] = cq[p];
    __syncthreads();
    uint64_t c = 0, inc = 0;
    if (q == 0) {
      for (uint32_t i = 0; i < split; ++i) c += part[i * radix + d];
      totals[p * radix + d] = (uint32_t)c;
      inc = dev::warp_inclusive_sum(c);
      if ((d & 31) == 31) warp_tot[d >> 5] = inc;
    }
    __syncthreads();
    if (q == 0) {
      uint64_t off = 0;
      for (uint32_t w = 0; w < (d >> 5); ++w) off += warp_tot[w];
      base[p * radix + d] = off + inc - c;
    }
    __syncthreads();
  }
}

// Digit width: 8 bits (256 digits) everywhere, or 9 bits (512) for the
// full-width sorts where it saves a pass (see lsd_partition).
template <int RB> struct Radix {
  static constexpr int kR = 1 << RB;
};

// Histogram copies per CTA: one per warp while the copies fit 64 KB, else 4.
template <int NP, int RB>
constexpr int hist_copies() {
  return NP * (1 << RB) * kHistWarps * 4 <= 64 * 1024 ? kHistWarps : 4;
}

template <class K, int NP, bool SHARD, int RB>
__global__ void __launch_bounds__(kHistThreads)
k_block_hist(const K* __restrict__ keys, const __grid_constant__ HistArgs a,
             uint32_t* __restrict__ cnt) {
  extern __shared__ uint32_t sh[];  // [copy][NP * R]
  constexpr int kR = Radix<RB>::kR;
  constexpr int kWidth = NP * kR;
  constexpr int kCopies = hist_copies<NP, RB>();
  for (int i = threadIdx.x; i < kCopies * kWidth; i += kHistThreads) sh[i] = 0;
  __syncthreads();
  uint32_t* mine = sh + ((threadIdx.x >> 5) % kCopies) * kWidth;
  // gridDim.x = nblocks * kHistSub: sub-CTA s of block b counts a quarter of
  // the block's tiles and adds into cnt[b] (zeroed by the caller)
  const uint64_t b = blockIdx.x / kHistSub, sub = blockIdx.x % kHistSub;
  const uint64_t t0 = b * a.tiles / a.nblocks, t1 = (b + 1) * a.tiles / a.nblocks;
  const uint64_t lo = dev::umin64(a.n, (t0 + sub * (t1 - t0) / kHistSub) * a.tile);
  const uint64_t hi = dev::umin64(a.n, (t0 + (sub + 1) * (t1 - t0) / kHistSub) * a.tile);
  uint32_t shf[NP], msk[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    shf[p] = a.shift[p];
    msk[p] = a.mask[p];
  }
  K kor = 0;
  auto count = [&](K k) {
    kor |= k;
    if (SHARD) {
      atomicAdd(&mine[dev::shard_digit((uint64_t)k, a.hparts, a.lowbits)], 1u);
    } else {
#pragma unroll
      for (int p = 0; p < NP; ++p) atomicAdd(&mine[p * kR + ((uint32_t)(k >> shf[p]) & msk[p])], 1u);
    }
  };
  constexpr int kVec = 16 / sizeof(K);
  uint64_t i = lo;
  if ((reinterpret_cast<uintptr_t>(keys + lo) & 15u) == 0) {
    const uint4* kv = reinterpret_cast<const uint4*>(keys + lo);
    const uint64_t nvec = (hi - lo) / kVec;
    uint64_t v = threadIdx.x;
    for (; v + 3 * kHistThreads < nvec; v += 4 * kHistThreads) {  // 4 loads in flight
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = __ldcs(kv + v + u * kHistThreads);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        K e[kVec];
        memcpy(e, &q[u], 16);
#pragma unroll
        for (int j = 0; j < kVec; ++j) count(e[j]);
      }
    }
    for (; v < nvec; v += kHistThreads) {
      uint4 q = __ldcs(kv + v);
      K e[kVec];
      memcpy(e, &q, 16);
#pragma unroll
      for (int j = 0; j < kVec; ++j) count(e[j]);
    }
    i = lo + nvec * kVec;
  }
  for (uint64_t j = i + threadIdx.x; j < hi; j += kHistThreads) count(keys[j]);
  if (a.key_or) {
    uint64_t o = (uint64_t)kor;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) o |= __shfl_xor_sync(0xffffffffu, o, s);
    if ((threadIdx.x & 31) == 0 && o) atomicOr(a.key_or, (unsigned long long)o);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kWidth; d += kHistThreads) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kCopies; ++w) t += sh[w * kWidth + d];
    if (t) atomicAdd(&cnt[b * kWidth + d], t);
  }
  if (a.done) {  // the last CTA turns the counts into digit totals and bases
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      // (the histogram copies are dead: their >= 4 KB hold part and warp_tot)
      digit_bases_block<NP>(cnt, a.nblocks, (uint32_t)kR, a.totals, a.base, sh,
                            reinterpret_cast<uint64_t*>(sh + kHistThreads));
    }
  }
}

template <class K, int NP, bool SHARD, int RB>
void launch_hist(cj_ctx* ctx, const K* keys, const HistArgs& a, uint32_t* cnt) {
  const size_t smem = sizeof(uint32_t) * (1 << RB) * NP * hist_copies<NP, RB>();
  CJ_CUDA(cudaFuncSetAttribute(k_block_hist<K, NP, SHARD, RB>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_block_hist<K, NP, SHARD, RB><<<a.nblocks * kHistSub, kHistThreads, smem, ctx->stream>>>(keys, a,
                                                                                           cnt);
}

template <class K, int RB>
void launch_hist_np(cj_ctx* ctx, const K* keys, const HistArgs& a, int np, uint32_t* cnt) {
  if (a.hparts) return launch_hist<K, 1, true, RB>(ctx, keys, a, cnt);
  switch (np) {
    case 1: return launch_hist<K, 1, false, RB>(ctx, keys, a, cnt);
    case 2: return launch_hist<K, 2, false, RB>(ctx, keys, a, cnt);
    case 3: return launch_hist<K, 3, false, RB>(ctx, keys, a, cnt);
    case 4: return launch_hist<K, 4, false, RB>(ctx, keys, a, cnt);
    case 5: return launch_hist<K, 5, false, RB>(ctx, keys, a, cnt);
    case 6: return launch_hist<K, 6, false, RB>(ctx, keys, a, cnt);
    case 7: return launch_hist<K, 7, false, RB>(ctx, keys, a, cnt);
    default: return launch_hist<K, 8, false, RB>(ctx, keys, a, cnt);
  }
}

// ---- onesweep scatter pass ------------------------------------------------

constexpr int kPassThreads = 256;  // == kRadix: thread d owns digit d in scans
constexpr int kPassWarps = kPassThreads / 32;

template <class K> struct PassShape;
template <> struct PassShape<uint32_t> { static constexpr int kItems = 16; };
template <> struct PassShape<uint64_t> { static constexpr int kItems = 12; };

struct PassArgs {
  const void* keys_in;
  void* keys_out;
  uint64_t n;
  uint32_t shift, mask;
  const uint64_t* base;   // [256] exclusive digit base of this pass
  uint64_t* status;       // [tiles * 256]
  uint32_t* ticket;
  uint32_t* err;
  uint64_t epoch;
  int nvals;
  int gen_ids;
  const void* vin[CJ_MAX_COLS + 1];
  void* vout[CJ_MAX_COLS + 1];
  uint32_t vbytes[CJ_MAX_COLS + 1];
};

template <class K>
__global__ void __launch_bounds__(kPassThreads)
k_scatter_pass(const __grid_constant__ PassArgs a) {
  constexpr int kItems = PassShape<K>::kItems;
  constexpr int kTile = kPassThreads * kItems;
  __shared__ uint32_t s_tile;
  __shared__ uint16_t whist[kPassWarps][kRadix];  // per-warp counts -> warp prefix
  __shared__ uint32_t dstart[kRadix];             // tile-local digit start
  __shared__ uint64_t goff[kRadix];               // global position - local position
  __shared__ uint32_t wsum[kPassWarps];
  __shared__ uint8_t sdig[kTile];
  __shared__ __align__(16) uint64_t sbuf[kTile];  // staging (keys, then each column)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kPassWarps * kRadix; i += kPassThreads) (&whist[0][0])[i] = 0;
  if (tid == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t tbase = tile * kTile;
  const K* __restrict__ kin = static_cast<const K*>(a.keys_in);

  // 1. load keys: warp-striped, warp w owns a contiguous segment of the tile
  K key[kItems];
  uint32_t dig[kItems];
  const uint64_t wbase = tbase + (uint64_t)warp * 32 * kItems;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t idx = wbase + (uint64_t)i * 32 + lane;
    if (idx < a.n) {
      key[i] = __ldcs(kin + idx);
      dig[i] = (uint32_t)(key[i] >> a.shift) & a.mask;
    } else {
      key[i] = 0;
      dig[i] = kRadix;  // padding: ranked but never stored
    }
  }

  // 2. stable rank within the warp segment (item rounds in input order)
  uint32_t rank[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint32_t peers = __match_any_sync(0xffffffffu, dig[i]);
    const uint32_t before = __popc(peers & dev::lanemask_lt());
    const bool valid = dig[i] < kRadix;
    uint32_t prev = valid ? whist[warp][dig[i]] : 0;
    rank[i] = prev + before;
    __syncwarp();
    if (valid && before == 0) whist[warp][dig[i]] = (uint16_t)(prev + __popc(peers));
    __syncwarp();
  }
  __syncthreads();

  // 3. per digit: exclusive prefix over warps, tile total; publish aggregate
  const int d = tid;
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < kPassWarps; ++w) {
    const uint32_t c = whist[w][d];
    whist[w][d] = (uint16_t)run;
    run += c;
  }
  const uint32_t tile_count = run;
  uint64_t* my_status = a.status + tile * kRadix;
  if (tile == 0)
    dev::st_relaxed(my_status + d, dev::pack_status(a.epoch, kFlagIncl, tile_count));
  else
    dev::st_relaxed(my_status + d, dev::pack_status(a.epoch, kFlagAgg, tile_count));

  // 4. tile-local digit starts (exclusive scan over digits)
  {
    const uint32_t inc = dev::warp_inclusive_sum(tile_count);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t off = 0;
#pragma unroll
    for (int w = 0; w < kPassWarps; ++w) off += w < warp ? wsum[w] : 0;
    dstart[d] = off + inc - tile_count;
  }
  __syncthreads();

  // 5. place keys in digit order in shared memory
  uint32_t lpos[kItems];
  K* skey = reinterpret_cast<K*>(sbuf);
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    if (dig[i] < kRadix) {
      lpos[i] = dstart[dig[i]] + whist[warp][dig[i]] + rank[i];
      skey[lpos[i]] = key[i];
      sdig[lpos[i]] = (uint8_t)dig[i];
    } else {
      lpos[i] = 0xffffffffu;
    }
  }

  // 6. decoupled look-back: exclusive count of digit d over earlier tiles
  {
    uint64_t excl = 0;
    if (tile > 0) {
      int64_t t = (int64_t)tile - 1;
      while (t >= 0) {
        uint64_t w, f;
        uint32_t spins = 0;
        do {
          w = dev::ld_relaxed(a.status + (uint64_t)t * kRadix + d);
          f = dev::st_flag(w, a.epoch);
          if (f == 0 && ++spins > dev::kSpinLimit) {
            atomicOr(a.err, dev::kErrStall);
            f = kFlagIncl;
            w = 0;
          }
        } while (f == 0);
        excl += w & kValMask;
        if (f == kFlagIncl) break;
        --t;
      }
      dev::st_relaxed(my_status + d,
                      dev::pack_status(a.epoch, kFlagIncl, excl + tile_count));
    }
    goff[d] = a.base[d] + excl - dstart[d];
  }
  __syncthreads();

  const uint32_t tile_n = (uint32_t)dev::umin64(kTile, a.n > tbase ? a.n - tbase : 0);
  K* __restrict__ kout = static_cast<K*>(a.keys_out);
  for (uint32_t j = tid; j < tile_n; j += kPassThreads) kout[goff[sdig[j]] + j] = skey[j];

  // 7. every carried column through the same permutation
  for (int c = 0; c < a.nvals; ++c) {
    const bool gen = a.gen_ids && c == 0;
    const uint32_t vb = a.vbytes[c];
    __syncthreads();
    if (vb == 4) {
      uint32_t v[kItems];
      const uint32_t* __restrict__ vin = static_cast<const uint32_t*>(a.vin[c]);
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = wbase + (uint64_t)i * 32 + lane;
        v[i] = gen ? (uint32_t)idx : (idx < a.n ? __ldcs(vin + idx) : 0u);
      }
      uint32_t* s = reinterpret_cast<uint32_t*>(sbuf);
#pragma unroll
      for (int i = 0; i < kItems; ++i)
        if (lpos[i] != 0xffffffffu) s[lpos[i]] = v[i];
      __syncthreads();
      uint32_t* __restrict__ vout = static_cast<uint32_t*>(a.vout[c]);
      for (uint32_t j = tid; j < tile_n; j += kPassThreads) vout[goff[sdig[j]] + j] = s[j];
    } else {
      uint64_t v[kItems];
      const uint64_t* __restrict__ vin = static_cast<const uint64_t*>(a.vin[c]);
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = wbase + (uint64_t)i * 32 + lane;
        v[i] = gen ? idx : (idx < a.n ? __ldcs(vin + idx) : 0ull);
      }
#pragma unroll
      for (int i = 0; i < kItems; ++i)
        if (lpos[i] != 0xffffffffu) sbuf[lpos[i]] = v[i];
      __syncthreads();
      uint64_t* __restrict__ vout = static_cast<uint64_t*>(a.vout[c]);
      for (uint32_t j = tid; j < tile_n; j += kPassThreads) vout[goff[sdig[j]] + j] = sbuf[j];
    }
  }
}

// ---- blocked scatter pass: shared types ----------------------------------------
//
// Persistent CTAs of 512 threads, one per SM; CTA b walks its static range of
// consecutive tiles in order and carries the per-digit write cursors in shared
// memory, so no CTA ever waits for another (the cross-block starting cursors
// come from the per-block counts of k_block_hist).

constexpr int kTmaThreads = 512;
constexpr int kTmaWarps = kTmaThreads / 32;

struct BlockPassArgs {
  const void* keys_in;
  void* keys_out;
  uint64_t n, tiles;
  uint32_t nblocks;
  uint32_t shift, mask, bits;
  uint32_t hparts;          // > 0: digit = shard of the key << lowbits | its low lowbits bits
  uint32_t lowbits;
  int runs;                 // input grouped by an earlier pass: test rounds for one digit
  int warp_slots;           // phase 4: warp-contiguous slots instead of CTA-strided
  const uint64_t* base;     // [256] exclusive digit base of this pass
  const uint32_t* cnt;      // per-block counts of this pass: cnt[b * cnt_stride + d]
  uint32_t cnt_stride;
  uint32_t stage_bytes, pbytes;
  int nvals, gen_ids;
  int stages;               // 2: prefetch the next tile while this one runs
  unsigned long long* cta_ns;  // CJ_CTA_TIMES: [start, end] globaltimer per CTA (diagnostics)
  const void* vin[CJ_MAX_COLS + 1];
  void* vout[CJ_MAX_COLS + 1];
  uint32_t vbytes[CJ_MAX_COLS + 1];
  uint32_t voff[CJ_MAX_COLS + 1];
};

// offsets[p] = first index whose low-`bits` digit is >= p (keys sorted by it)
template <class K>
__global__ void k_offsets(const K* __restrict__ keys, uint64_t n, uint32_t bits,
                          uint64_t* __restrict__ off) {
  const uint64_t fanout = 1ull << bits;
  const K mask = (K)(fanout - 1);
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= fanout;
       p += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if ((uint64_t)(keys[mid] & mask) < p) lo = mid + 1; else hi = mid;
    }
    off[p] = p == fanout ? n : lo;
  }
}

// The same offsets by one pass over the keys: row i, the first row of its
// digit, writes off[p] = i for every digit p between the previous row's digit
// (exclusive) and its own; the last row fills the digits above it with n.
// Reads n keys instead of (fanout + 1) binary searches of log2(n) dependent
// loads: the faster one for small inputs (partition_offsets picks).
template <class K>
__global__ void k_offsets_scan(const K* __restrict__ keys, uint64_t n, uint32_t bits,
                               uint64_t* __restrict__ off) {
  const uint64_t fanout = 1ull << bits;
  const K mask = (K)(fanout - 1);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = (uint64_t)(keys[i] & mask);
    const uint64_t prev = i ? (uint64_t)(keys[i - 1] & mask) + 1 : 0;  // first digit to set
    for (uint64_t p = prev; p <= d; ++p) off[p] = i;
    if (i == n - 1)
      for (uint64_t p = d + 1; p <= fanout; ++p) off[p] = n;
  }
}

// ---- blocked scatter pass v2: source-index staging ---------------------------
//
// A tile costs four block barriers regardless of the number of carried columns:
//   1. rank: each warp ranks its contiguous 32*ITEMS segment (input order =
//      (warp, item, lane)); the stable in-warp peers of a digit come from
//      RANK: 0 = shared atomic-OR peer masks (default), 1 = bit ballots;
//      the lowest peer bumps the warp's per-digit count (no atomics);
//   2. scan: per digit, exclusive prefix over warps and over digits;
//   3. place: slot of every row in the digit-sorted tile; only the SOURCE
//      INDEX (u16) is written to shared memory;
//   4. write: slot j reads src = sidx[j], the key at src (its digit gives the
//      run's global offset) and every carried column at src straight from the
//      TMA stage, and stores them at goff[d] + j.  Consecutive slots of a digit
//      run are consecutive output rows (coalesced runs), and no column needs a
//      re-staging barrier.
// Global row indices are u32 (kMaxRows = 2^31 - 1, column.hpp:21).

// mm: the warp's peer-mask row of (1 << RB) + 32 words (the 32 spare words
// are unused: kept so the table layout does not depend on the rank mode).
template <int RANK, int RB>
__device__ __forceinline__ uint32_t peers_of(uint32_t d, bool valid, uint32_t* mm, uint32_t bits) {
  const uint32_t lane = threadIdx.x & 31u;
  if (RANK == 0) {
    // a truly predicated shared reduction: lanes that take no part issue
    // nothing (an if-converted atomicOr(.., 0) from every lane costs ~18
    // wavefronts in a skewed round: profiles/r02_scatter_skew_atoms.txt)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
        "@p red.shared.or.b32 [%0], %1;\n\t}" ::"r"(dev::smem_addr(&mm[d])),
        "r"(1u << lane), "r"((uint32_t)valid)
        : "memory");
    __syncwarp();
    const uint32_t p = valid ? mm[d] : 0u;
    __syncwarp();
    return p;
  }
  return dev::digit_peers(d, bits, __ballot_sync(0xffffffffu, valid)) & (valid ? ~0u : 0u);
}

#ifdef CJ_PHASE_CLOCKS
// Debug builds only (tools/ubench_phases): cycles per scatter phase, CTA 0 thread 0.
__device__ unsigned long long g_phase_clk[16];
#define CJ_CLK(i) CJ_CLKT(i, 0)
#define CJ_CLKT(i, th)                                              \
  do {                                                              \
    if (blockIdx.x == 0 && threadIdx.x == (th)) {                   \
      const long long now = clock64();                              \
      g_phase_clk[i] += (unsigned long long)(now - clk_prev);       \
      clk_prev = now;                                               \
    }                                                               \
  } while (0)
#else
#define CJ_CLK(i) \
  do {            \
  } while (0)
#define CJ_CLKT(i, th) \
  do {                 \
  } while (0)
#endif

// Digit of key k in pass (shift, mask) or, in shard mode, its shard.
template <bool SHARD, class K>
__device__ __forceinline__ uint32_t digit_of(K k, const BlockPassArgs& a) {
  if (SHARD) return dev::shard_digit((uint64_t)k, a.hparts, a.lowbits);
  return (uint32_t)(k >> a.shift) & a.mask;
}

// One tile of k_scatter_v2 (phases 1-4).  FULL: tile_n == kTile, no guards.
// HOT (skewed keys): the pass has one dominant digit `hot` (>= 1/8 of the
// rows).  Its lanes take their peer masks from a ballot instead of an atomic
// OR on a shared word that much of the warp would hit.
template <class K, int ITEMS, int RANK, bool SHARD, bool FULL, int RB, int HOT, bool UNI, int NT>
__device__ __forceinline__ void scatter_tile(const BlockPassArgs& a, const uint8_t* st,
                                             uint16_t* sidx, uint16_t (*whist)[1 << RB],
                                             uint32_t* mm, uint32_t* dstart, uint32_t* run,
                                             uint32_t* goff, uint32_t* wsum, uint32_t tbase,
                                             uint32_t tile_n, uint32_t hot) {
  constexpr uint32_t kTile = ITEMS * NT;
  constexpr int kR = 1 << RB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const K* skey = reinterpret_cast<const K*>(st);
#ifdef CJ_PHASE_CLOCKS
  long long clk_prev = clock64();
#endif

  // 1. stable in-warp ranking; pk = (rank within warp << 8) | digit, or ~0u
  const uint32_t wseg = warp * 32 * ITEMS;
  uint32_t pk[ITEMS];
  uint16_t* wh = &whist[warp][0];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t li = wseg + i * 32 + lane;
    const bool valid = FULL || li < tile_n;
    const uint32_t d = digit_of<SHARD>(skey[li], a);
    uint32_t peers;
    // After a first pass over skewed keys the rows arrive grouped by its
    // digit, so a frequent key's rows are contiguous and most lanes of a round
    // share one digit: they would serialise on one shared word.  UNI: the
    // lanes holding lane 0's digit take their peer mask from one ballot, the
    // others the atomic-OR masks (a second leader measured slower; per-CTA
    // times: profiles/r02_skew_summary.md).
    if constexpr (UNI) {
      const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
      const bool m0 = valid && d == d0;
      const uint32_t b0 = __ballot_sync(0xffffffffu, m0);
      if (b0 == 0xffffffffu) {
        peers = b0;
      } else {
        peers = peers_of<RANK, RB>(d, valid && !m0, mm, a.bits);
        if (m0) peers = b0;
      }
    } else if constexpr (HOT) {
      // a dominant digit (>= 1/8 of the rows): its lanes take one ballot, the
      // others the atomic-OR masks
      const bool h = valid && d == hot;
      const uint32_t hb = __ballot_sync(0xffffffffu, h);
      peers = peers_of<RANK, RB>(d, valid && !h, mm, a.bits);
      if (h) peers = hb;
    } else {
      peers = peers_of<RANK, RB>(d, valid, mm, a.bits);
    }
    const uint32_t lt = peers & dev::lanemask_lt();
    uint32_t old = 0;
    if (valid && lt == 0) {
      old = wh[d];
      wh[d] = (uint16_t)(old + __popc(peers));
      if (RANK == 0) mm[d] = 0;
    }
    old = __shfl_sync(0xffffffffu, old, __ffs(peers | (1u << lane)) - 1);
    pk[i] = valid ? ((old + __popc(lt)) << RB) | d : 0xffffffffu;
    if (RANK == 0) __syncwarp();
  }
  __syncthreads();
  CJ_CLK(0);

  // 2. per digit: tile total, exclusive digit start, then whist[w][d] = slot
  //    of warp w's first row of digit d (digit start + earlier warps' counts)
  if constexpr (kR == 64) {  // (128 digits: 4 per lane measured slower than 4 warps + a barrier)
    // one warp, kD adjacent digits per lane (kD / 2 32-bit words of every
    // warp's row): the digit scan needs no second barrier
    constexpr int kD = kR / 32, kW = kD / 2;
    if (warp == 0) {
      uint32_t c[(NT / 32)][kW], r[kD] = {};
#pragma unroll
      for (int w = 0; w < (NT / 32); ++w) {
        const uint32_t* row = reinterpret_cast<const uint32_t*>(&whist[w][0]) + lane * kW;
#pragma unroll
        for (int j = 0; j < kW; ++j) {
          c[w][j] = row[j];
          r[2 * j] += c[w][j] & 0xffffu;
          r[2 * j + 1] += c[w][j] >> 16;
        }
      }
      uint32_t tot = 0;
#pragma unroll
      for (int j = 0; j < kD; ++j) tot += r[j];
      uint32_t ds[kD];
      ds[0] = dev::warp_inclusive_sum(tot) - tot;
#pragma unroll
      for (int j = 1; j < kD; ++j) ds[j] = ds[j - 1] + r[j - 1];
      uint32_t p[kD];
#pragma unroll
      for (int j = 0; j < kD; ++j) p[j] = ds[j];
#pragma unroll
      for (int w = 0; w < (NT / 32); ++w) {
        uint32_t* row = reinterpret_cast<uint32_t*>(&whist[w][0]) + lane * kW;
#pragma unroll
        for (int j = 0; j < kW; ++j) {
          row[j] = p[2 * j] | (p[2 * j + 1] << 16);
          p[2 * j] += c[w][j] & 0xffffu;
          p[2 * j + 1] += c[w][j] >> 16;
        }
      }
#pragma unroll
      for (int j = 0; j < kD; ++j) {
        const uint32_t d = lane * kD + j;
        goff[d] = run[d] - ds[j];
        run[d] += r[j];
      }
    }
    __syncthreads();
  } else {
    uint32_t c[(NT / 32)], r = 0, inc = 0;
    if (tid < kR) {
#pragma unroll
      for (int w = 0; w < (NT / 32); ++w) {
        c[w] = whist[w][tid];
        r += c[w];
      }
      inc = dev::warp_inclusive_sum(r);
      if (lane == 31) wsum[warp] = inc;
    }
    __syncthreads();
    CJ_CLK(2);
    if (tid < kR) {
      uint32_t off = 0;
#pragma unroll
      for (int w = 0; w < kR / 32; ++w) off += w < warp ? wsum[w] : 0;
      const uint32_t ds = off + inc - r;
      uint32_t p = ds;
#pragma unroll
      for (int w = 0; w < (NT / 32); ++w) {
        whist[w][tid] = (uint16_t)p;
        p += c[w];
      }
      goff[tid] = run[tid] - ds;
      run[tid] += r;
    }
    __syncthreads();
    CJ_CLK(3);
  }

  // 3. slot of every row; record its source index
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (FULL || pk[i] != 0xffffffffu) {
      sidx[wh[pk[i] & (kR - 1)] + (pk[i] >> RB)] = (uint16_t)(wseg + i * 32 + lane);
    }
  }
  __syncthreads();
  CJ_CLK(1);

  // 4. write key + carried columns of each slot (loads batched for ILP)
  // slot of item k: warp-contiguous (a warp writes 32*ITEMS consecutive slots,
  // a.warp_slots) or CTA-strided (slot tid + k*NT)
  const uint32_t jb = a.warp_slots ? (uint32_t)warp * 32 * ITEMS + lane : (uint32_t)tid;
  const uint32_t js = a.warp_slots ? 32u : (uint32_t)NT;
  uint32_t src[ITEMS], g[ITEMS];
  K key[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t j = jb + k * js;
    src[k] = (FULL || j < tile_n) ? sidx[j] : 0u;
  }
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) key[k] = skey[src[k]];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) g[k] = goff[digit_of<SHARD>(key[k], a)] + jb + k * js;
  K* __restrict__ kout = static_cast<K*>(a.keys_out);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k)
    if (FULL || jb + k * js < tile_n) kout[g[k]] = key[k];
  for (int c = 0; c < a.nvals; ++c) {
    if (a.gen_ids && c == 0) {
      uint32_t* __restrict__ vout = static_cast<uint32_t*>(a.vout[c]);
#pragma unroll
      for (int k = 0; k < ITEMS; ++k)
        if (FULL || jb + k * js < tile_n) vout[g[k]] = tbase + src[k];
    } else if (a.vbytes[c] == 4) {
      const uint32_t* sv = reinterpret_cast<const uint32_t*>(st + a.voff[c]);
      uint32_t* __restrict__ vout = static_cast<uint32_t*>(a.vout[c]);
      uint32_t v[ITEMS];
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) v[k] = sv[src[k]];
#pragma unroll
      for (int k = 0; k < ITEMS; ++k)
        if (FULL || jb + k * js < tile_n) vout[g[k]] = v[k];
    } else {
      const uint64_t* sv = reinterpret_cast<const uint64_t*>(st + a.voff[c]);
      uint64_t* __restrict__ vout = static_cast<uint64_t*>(a.vout[c]);
      uint64_t v[ITEMS];
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) v[k] = sv[src[k]];
#pragma unroll
      for (int k = 0; k < ITEMS; ++k)
        if (FULL || jb + k * js < tile_n) vout[g[k]] = v[k];
    }
  }
  CJ_CLK(7);
  (void)kTile;
}

template <class K, int ITEMS, int RANK, bool SHARD, int MINB, int RB, int NT>
__global__ void __launch_bounds__(NT, MINB)
k_scatter_v2(const __grid_constant__ BlockPassArgs a) {
  constexpr uint32_t kTile = ITEMS * NT;
  constexpr int kR = 1 << RB;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* const stage0 = smem;
  uint16_t* const sidx = reinterpret_cast<uint16_t*>(smem + (size_t)a.stages * a.stage_bytes);
  // per-warp peer masks (rank mode 0) after the source indices, 16-byte aligned
  uint32_t (*match_word)[kR + 32] = reinterpret_cast<uint32_t (*)[kR + 32]>(
      smem + (((size_t)a.stages * a.stage_bytes + (size_t)kTile * 2 + 15) & ~size_t(15)));
  __shared__ uint16_t whist[(NT / 32)][kR];
  __shared__ uint32_t dstart[kR];
  __shared__ uint32_t run[kR];   // next global row of each digit in this block
  __shared__ uint32_t goff[kR];  // global row of tile slot 0 of each digit's run (mod 2^32)
  __shared__ uint32_t wsum[kR / 32];
  __shared__ __align__(8) uint64_t mbar[2];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const K* __restrict__ kin = static_cast<const K*>(a.keys_in);
  const uint64_t blk = blockIdx.x;
  const uint64_t t_begin = blk * a.tiles / a.nblocks, t_end = (blk + 1) * a.tiles / a.nblocks;

  auto issue = [&](int b, uint64_t t) {  // thread 0: bulk-copy tile t into stage b
    const uint64_t tb = t * kTile;
    uint8_t* st = stage0 + (size_t)b * a.stage_bytes;
    uint32_t total = kTile * sizeof(K);
    for (int c = 0; c < a.nvals; ++c)
      if (!(a.gen_ids && c == 0)) total += kTile * a.vbytes[c];
    dev::mbar_expect_tx(&mbar[b], total);
    dev::tma_load_1d(st, kin + tb, kTile * sizeof(K), &mbar[b]);
    for (int c = 0; c < a.nvals; ++c)
      if (!(a.gen_ids && c == 0))
        dev::tma_load_1d(st + a.voff[c], static_cast<const uint8_t*>(a.vin[c]) + tb * a.vbytes[c],
                         kTile * a.vbytes[c], &mbar[b]);
  };
  auto full_tile = [&](uint64_t t) { return (t + 1) * kTile <= a.n; };

  if (tid == 0) {
    dev::mbar_init(&mbar[0], 1);
    dev::mbar_init(&mbar[1], 1);
    dev::fence_mbar_init();
    if (t_begin < t_end && full_tile(t_begin)) issue(0, t_begin);
  }
  if (RANK == 0)
    for (int i = tid; i < (NT / 32) * (kR + 32); i += NT) (&match_word[0][0])[i] = 0;
  __shared__ uint64_t s_dmax[kR / 32];
  if (tid < kR) {
    uint64_t c = a.base[tid];
    for (uint64_t b2 = 0; b2 < blk; ++b2) c += a.cnt[b2 * a.cnt_stride + tid];
    run[tid] = (uint32_t)c;
    // the pass's most frequent digit (totals = differences of the bases)
    const uint64_t tot = (tid + 1 < kR ? a.base[tid + 1] : a.n) - a.base[tid];
    uint64_t v = (tot << 16) | (uint64_t)tid;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) s_dmax[warp] = v;
  }
  __syncthreads();
  uint64_t vmax = 0;
#pragma unroll
  for (int w = 0; w < kR / 32; ++w) vmax = max(vmax, s_dmax[w]);
  // >= 1/8 of the rows: a warp round holds 4+ lanes of that digit on average
  const uint32_t hot = !SHARD && RANK == 0 && (vmax >> 16) * 8 >= a.n ? (uint32_t)(vmax & 0xffffu)
                                                                         : 0xffffffffu;
  // skewed digits after an earlier pass (the top digit at least twice its
  // uniform share): frequent keys arrive in runs, test rounds for one digit
  const bool uni = !SHARD && RANK == 0 && a.runs && ((vmax >> 16) << a.bits) >= 2 * a.n;

  uint64_t t_start = 0;
  if (a.cta_ns && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  uint32_t ph0 = 0, ph1 = 0;
  int b = 0;
  uint32_t* mm = &match_word[RANK == 0 ? warp : 0][0];
  for (uint64_t t = t_begin; t < t_end; ++t, b = b + 1 == a.stages ? 0 : b + 1) {
    if (a.stages == 2 && tid == 0 && t + 1 < t_end && full_tile(t + 1)) {
      dev::fence_proxy_async();
      issue(b ^ 1, t + 1);
    }
    // each warp zeroes its own histogram row (only it touches the row until
    // the barrier after ranking)
    {
      uint32_t* wrow = reinterpret_cast<uint32_t*>(&whist[warp][0]);
#pragma unroll
      for (int i = 0; i < kR / 2 / 32; ++i) wrow[lane + 32 * i] = 0;
      __syncwarp();
    }
    const uint64_t tbase = t * kTile;
    const uint32_t tile_n = (uint32_t)dev::umin64(kTile, a.n - tbase);
    uint8_t* st = stage0 + (size_t)b * a.stage_bytes;
    if (full_tile(t)) {
      dev::mbar_wait(&mbar[b], b ? ph1 : ph0);
      if (b) ph1 ^= 1; else ph0 ^= 1;
#define CJ_TILE(H, U)                                                                      \
  scatter_tile<K, ITEMS, RANK, SHARD, true, RB, H, U, NT>(a, st, sidx, whist, mm, dstart, run, goff, \
                                                          wsum, (uint32_t)tbase, tile_n, hot)
      switch ((hot != 0xffffffffu ? 1 : 0) | (uni ? 2 : 0)) {
        case 0: CJ_TILE(0, false); break;
        case 1: CJ_TILE(1, false); break;
        case 2: CJ_TILE(0, true); break;
        default: CJ_TILE(1, true); break;
      }
#undef CJ_TILE
    } else {  // last, partial tile: plain loads
      K* wk = reinterpret_cast<K*>(st);
      for (uint32_t j = tid; j < kTile; j += NT) wk[j] = j < tile_n ? kin[tbase + j] : K(0);
      for (int c = 0; c < a.nvals; ++c) {
        if (a.gen_ids && c == 0) continue;
        if (a.vbytes[c] == 4) {
          const uint32_t* src = static_cast<const uint32_t*>(a.vin[c]) + tbase;
          uint32_t* dst = reinterpret_cast<uint32_t*>(st + a.voff[c]);
          for (uint32_t j = tid; j < tile_n; j += NT) dst[j] = src[j];
        } else {
          const uint64_t* src = static_cast<const uint64_t*>(a.vin[c]) + tbase;
          uint64_t* dst = reinterpret_cast<uint64_t*>(st + a.voff[c]);
          for (uint32_t j = tid; j < tile_n; j += NT) dst[j] = src[j];
        }
      }
      __syncthreads();
      scatter_tile<K, ITEMS, RANK, SHARD, false, RB, 0, false, NT>(a, st, sidx, whist, mm, dstart, run, goff,
                                                            wsum, (uint32_t)tbase, tile_n, hot);
    }
    __syncthreads();
    if (a.stages == 1 && tid == 0 && t + 1 < t_end && full_tile(t + 1)) {
      dev::fence_proxy_async();
      issue(0, t + 1);
    }
  }
  if (a.cta_ns && tid == 0) {
    uint64_t t_end_ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end_ns));
    a.cta_ns[2 * blockIdx.x] = t_start;
    a.cta_ns[2 * blockIdx.x + 1] = t_end_ns;
  }
}

template <class K, int ITEMS, int RANK, int MINB, int RB>
void launch_v2(cj_ctx* ctx, const BlockPassArgs& a, size_t smem, int threads) {
  auto go = [&](auto kern, int nt) {
    CJ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<a.nblocks, nt, smem, ctx->stream>>>(a);
  };
  if (threads == 256) {  // two CTAs per SM
    if (a.hparts) go(k_scatter_v2<K, ITEMS, RANK, true, 2, RB, 256>, 256);
    else go(k_scatter_v2<K, ITEMS, RANK, false, 2, RB, 256>, 256);
  } else {
    if (a.hparts) go(k_scatter_v2<K, ITEMS, RANK, true, MINB, RB, 512>, 512);
    else go(k_scatter_v2<K, ITEMS, RANK, false, MINB, RB, 512>, 512);
  }
}

template <class K, int RANK>
void launch_v2_items(cj_ctx* ctx, const BlockPassArgs& a, size_t smem, int items, int rb,
                     int threads) {
  if (rb == 6) {  // passes of <= 6 bits: 64-digit tables, room for 8192-row tiles
    switch (items) {
      case 16: launch_v2<K, 16, RANK, 1, 6>(ctx, a, smem, threads); break;
      case 12: launch_v2<K, 12, RANK, 1, 6>(ctx, a, smem, threads); break;
      case 8: launch_v2<K, 8, RANK, 1, 6>(ctx, a, smem, threads); break;
      default: launch_v2<K, 4, RANK, 1, 6>(ctx, a, smem, threads); break;
    }
    return;
  }
  if (rb == 7) {  // 7-bit passes (27-bit sort keys: 7+7+7+6)
    switch (items) {
      case 16: launch_v2<K, 16, RANK, 1, 7>(ctx, a, smem, threads); break;
      case 12: launch_v2<K, 12, RANK, 1, 7>(ctx, a, smem, threads); break;
      case 8: launch_v2<K, 8, RANK, 1, 7>(ctx, a, smem, threads); break;
      default: launch_v2<K, 4, RANK, 1, 7>(ctx, a, smem, threads); break;
    }
    return;
  }
  if (rb != 8) fail(CJ_ERR_UNSUPPORTED, "scatter pass digits wider than 8 bits");
  switch (items) {
    case 16: launch_v2<K, 16, RANK, 1, 8>(ctx, a, smem, threads); break;
    case 12: launch_v2<K, 12, RANK, 1, 8>(ctx, a, smem, threads); break;
    case 8: launch_v2<K, 8, RANK, 1, 8>(ctx, a, smem, threads); break;
    default: launch_v2<K, 4, RANK, 1, 8>(ctx, a, smem, threads); break;
  }
}


template <class T>
__global__ void k_iota(T* out, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (T)i;
}

}  // namespace

namespace {

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

ScatterGeom scatter_geom(cj_ctx* ctx, uint64_t n, int key_bytes, const ValCols& vals,
                         const void* keys_in, int rb) {
  ScatterGeom g;
  g.rb = rb;
  uint64_t row = key_bytes;
  uint32_t maxw = key_bytes;
  bool al = aligned16(keys_in);
  for (int c = 0; c < vals.n; ++c) {
    const bool gen = vals.gen_ids && c == 0;
    if (!gen) {
      row += vals.bytes[c];
      al = al && aligned16(vals.in[c]);
    }
    maxw = std::max(maxw, vals.bytes[c]);
  }
  const char* mode = std::getenv("CJ_SCATTER");
  g.tma = al && !(mode && std::strcmp(mode, "ldg") == 0);
  // tuning knobs (defaults chosen from the sweeps recorded in profiles/)
  const char* e_items = std::getenv("CJ_SCATTER_ITEMS");
  const char* e_stages = std::getenv("CJ_SCATTER_STAGES");
  const char* e_rank = std::getenv("CJ_RANK");
  g.rank = e_rank ? std::atoi(e_rank) : 0;
  // CJ_SCATTER_THREADS=256: two 256-thread CTAs per SM, each with half the
  // shared memory (experiment knob; default one 512-thread CTA per SM)
  const char* e_thr = std::getenv("CJ_SCATTER_THREADS");
  g.threads = e_thr && std::atoi(e_thr) == 256 ? 256 : 512;
  g.ctas_per_sm = g.threads == 256 ? 2 : 1;
  g.stages = e_stages ? std::min(2, std::max(1, std::atoi(e_stages))) : 2;
  const int want_items = e_items ? std::atoi(e_items) : 16;
  // 227 KB per CTA minus the static arrays (per-warp digit counts 8 KB and
  // ~4 KB of cursors, twice that for 9-bit digits) and the dynamic peer masks
  // of rank mode 0 (16 KB / 32 KB)
  const size_t budget = (227 / g.ctas_per_sm - (((size_t)12 << rb) >> 8)) * 1024;
  const size_t match = g.rank == 0 ? (size_t)(g.threads / 32) * 4 * ((1u << rb) + 32) : 0;
  for (int items : {16, 12, 8, 4}) {
    if (items > want_items && items > 4) continue;
    if (rb == 9 && items > 12) continue;
    g.items = items;
    g.tile = (uint64_t)g.threads * items;
    g.stage_bytes = (uint32_t)(g.tile * row);
    g.pbytes = 0;
    g.smem = (((size_t)g.stages * g.stage_bytes + g.tile * 2 + 15) & ~size_t(15)) + match;
    if (g.smem <= budget) break;
  }
  if (g.smem > budget) g.tma = false;  // rows too wide: the look-back onesweep path
  uint32_t off = (uint32_t)(g.tile * key_bytes);
  for (int c = 0; c < vals.n; ++c) {
    g.voff[c] = off;
    if (!(vals.gen_ids && c == 0)) off += (uint32_t)(g.tile * vals.bytes[c]);
  }
  g.tiles = std::max<uint64_t>((n + g.tile - 1) / g.tile, 1);
  g.nblocks = (uint32_t)std::min<uint64_t>(g.tiles, (uint64_t)ctx->num_sms * g.ctas_per_sm);
  return g;
}

void block_hist(cj_ctx* ctx, const void* keys, uint64_t n, int key_bytes, const PassPlan& plan,
                const ScatterGeom& g, uint32_t* cnt_dev, uint32_t hparts, uint32_t lowbits,
                unsigned long long* key_or, uint32_t* totals_dev, uint64_t* base_dev) {
  const int np = plan.npasses;
  if (np < 1 || np > 8) fail(CJ_ERR_UNSUPPORTED, "histogram of 1..8 passes");
  HistArgs a{};
  a.n = n;
  a.tile = g.tile;
  a.tiles = g.tiles;
  a.nblocks = g.nblocks;
  a.hparts = hparts;
  a.lowbits = lowbits;
  a.key_or = key_or;
  if (totals_dev && base_dev) {
    a.done = ctx->ticket(9);
    a.totals = totals_dev;
    a.base = base_dev;
  }
  for (int p = 0; p < np; ++p) {
    a.shift[p] = plan.lo[p];
    a.mask[p] = (1u << (plan.hi[p] - plan.lo[p])) - 1u;
  }
  const uint32_t R = 1u << g.rb;
  CJ_CUDA(cudaMemsetAsync(cnt_dev, 0, sizeof(uint32_t) * R * np * g.nblocks, ctx->stream));
  ctx->kbegin("histogram", n * key_bytes);
  if (g.rb < 6 || g.rb > 8) fail(CJ_ERR_UNSUPPORTED, "histogram digits wider than 8 bits");
  if (key_bytes == 4) {
    const uint32_t* k = static_cast<const uint32_t*>(keys);
    if (g.rb == 6) launch_hist_np<uint32_t, 6>(ctx, k, a, np, cnt_dev);
    else if (g.rb == 7) launch_hist_np<uint32_t, 7>(ctx, k, a, np, cnt_dev);
    else launch_hist_np<uint32_t, 8>(ctx, k, a, np, cnt_dev);
  } else {
    const uint64_t* k = static_cast<const uint64_t*>(keys);
    if (g.rb == 6) launch_hist_np<uint64_t, 6>(ctx, k, a, np, cnt_dev);
    else if (g.rb == 7) launch_hist_np<uint64_t, 7>(ctx, k, a, np, cnt_dev);
    else launch_hist_np<uint64_t, 8>(ctx, k, a, np, cnt_dev);
  }
  ctx->kend();
  CJ_CUDA(cudaGetLastError());
}

void histogram_passes(cj_ctx* ctx, const void* keys, uint64_t n, int key_bytes,
                      const PassPlan& plan, const ScatterGeom& g, uint32_t* cnt_dev,
                      uint32_t* totals_dev, uint64_t* base_dev,
                      std::vector<uint32_t>* totals_host, uint32_t hparts, uint32_t lowbits,
                      unsigned long long* key_or) {
  const int np = plan.npasses;
  if (np > 8) fail(CJ_ERR_UNSUPPORTED, "histogram of more than 8 passes");
  // (the histogram's last CTA writes the totals and bases)
  block_hist(ctx, keys, n, key_bytes, plan, g, cnt_dev, hparts, lowbits, key_or, totals_dev,
             base_dev);
  const uint32_t R = 1u << g.rb;
  if (totals_host) {
    totals_host->resize((size_t)R * np);
    CJ_CUDA(cudaMemcpyAsync(ctx->host_pinned, totals_dev, sizeof(uint32_t) * R * np,
                            cudaMemcpyDeviceToHost, ctx->stream));
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(totals_host->data(), ctx->host_pinned, sizeof(uint32_t) * R * np);
  }
}

void scatter_pass(cj_ctx* ctx, const void* keys_in, void* keys_out, uint64_t n, int key_bytes,
                  uint32_t lo, uint32_t hi, const uint64_t* base_dev, const uint32_t* cnt,
                  uint32_t cnt_stride, const ScatterGeom& g, const ValCols& vals, uint32_t hparts,
                  uint32_t lowbits, int runs) {
  if (n == 0) return;
  if (hparts && !g.tma)
    fail(CJ_ERR_UNSUPPORTED, "shard partition needs 16-byte aligned columns");
  if (hparts && !cnt) fail(CJ_ERR_UNSUPPORTED, "shard partition needs per-block counts");
  uint64_t row = key_bytes, wrow = key_bytes;
  for (int c = 0; c < vals.n; ++c) {
    row += vals.bytes[c] - ((vals.gen_ids && c == 0) ? 4 : 0);
    wrow += vals.bytes[c];
  }
  if (g.tma && cnt) {
    BlockPassArgs a{};
    a.keys_in = keys_in;
    a.keys_out = keys_out;
    a.n = n;
    a.tiles = g.tiles;
    a.nblocks = g.nblocks;
    a.shift = lo;
    a.bits = hi - lo;
    a.mask = (1u << (hi - lo)) - 1u;
    a.hparts = hparts;
    a.lowbits = lowbits;
    a.runs = runs;
    // phase-4 slot order: warp-contiguous for 64-digit passes (longer runs per
    // warp: C2 PHJ scatter 6.17 -> 6.04 ms), CTA-strided for wider digits
    // (SMJ 7-bit passes 9.01 -> 9.17 ms the other way); CJ_SLOTS=warp|cta forces
    static const int slots_env = [] {
      const char* e = std::getenv("CJ_SLOTS");
      return e ? (std::strcmp(e, "warp") == 0 ? 1 : 0) : -1;
    }();
    a.warp_slots = slots_env >= 0 ? slots_env : (g.rb <= 6 ? 1 : 0);
    if (hparts) {  // digit = shard << lowbits | low bits: ceil(log2 parts) + lowbits bits
      uint32_t sb = 0;
      while ((1u << sb) < hparts) ++sb;
      a.bits = sb + lowbits;
    }
    a.base = base_dev;
    a.cnt = cnt;
    a.cnt_stride = cnt_stride;
    a.stage_bytes = g.stage_bytes;
    a.pbytes = g.pbytes;
    a.stages = g.stages;
    a.nvals = vals.n;
    a.gen_ids = vals.gen_ids;
    for (int c = 0; c < vals.n; ++c) {
      a.vin[c] = vals.in[c];
      a.vout[c] = vals.out[c];
      a.vbytes[c] = vals.bytes[c];
      a.voff[c] = g.voff[c];
    }
    static const bool cta_times = std::getenv("CJ_CTA_TIMES") != nullptr;
    Scratch cta_buf(ctx, cta_times ? 16ull * g.nblocks : 0);
    a.cta_ns = cta_times ? cta_buf.as<unsigned long long>() : nullptr;
    ctx->kbegin("scatter_pass", n * (row + wrow));
    if (key_bytes == 4) {
      if (g.rank == 1) launch_v2_items<uint32_t, 1>(ctx, a, g.smem, g.items, g.rb, g.threads);
      else launch_v2_items<uint32_t, 0>(ctx, a, g.smem, g.items, g.rb, g.threads);
    } else {
      if (g.rank == 1) launch_v2_items<uint64_t, 1>(ctx, a, g.smem, g.items, g.rb, g.threads);
      else launch_v2_items<uint64_t, 0>(ctx, a, g.smem, g.items, g.rb, g.threads);
    }
    ctx->kend();
    CJ_CUDA(cudaGetLastError());
    if (cta_times) {  // diagnostics: per-CTA durations of this pass (stderr)
      std::vector<unsigned long long> h(2ull * g.nblocks);
      CJ_CUDA(cudaMemcpyAsync(h.data(), cta_buf.p, 16ull * g.nblocks, cudaMemcpyDeviceToHost,
                              ctx->stream));
      CJ_CUDA(cudaStreamSynchronize(ctx->stream));
      unsigned long long t0 = ~0ull, t1 = 0;
      std::vector<double> d(g.nblocks);
      for (uint32_t i = 0; i < g.nblocks; ++i) {
        t0 = std::min(t0, h[2 * i]);
        t1 = std::max(t1, h[2 * i + 1]);
        d[i] = (h[2 * i + 1] - h[2 * i]) / 1e3;
      }
      std::vector<double> sd = d;
      std::sort(sd.begin(), sd.end());
      std::fprintf(stderr, "cta_times n=%llu bits=%u..%u: span %.1f us, per-CTA min %.1f med %.1f max %.1f us; first 16:",
                   (unsigned long long)n, lo, hi, (t1 - t0) / 1e3, sd.front(), sd[sd.size() / 2],
                   sd.back());
      for (uint32_t i = 0; i < g.nblocks; i += std::max(1u, g.nblocks / 16)) std::fprintf(stderr, " %.0f", d[i]);
      std::fprintf(stderr, "\n");
    }
    return;
  }
  // fallback for unaligned columns: register-staged onesweep with look-back
  const int items = key_bytes == 4 ? PassShape<uint32_t>::kItems : PassShape<uint64_t>::kItems;
  const uint64_t tile = (uint64_t)kPassThreads * items;
  const uint64_t tiles = (n + tile - 1) / tile;
  PassArgs a{};
  a.keys_in = keys_in;
  a.keys_out = keys_out;
  a.n = n;
  a.shift = lo;
  a.mask = (1u << (hi - lo)) - 1u;
  a.base = base_dev;
  a.status = ctx->status_buffer(tiles * kRadix);
  a.ticket = ctx->ticket(0);
  a.err = ctx->err_word;
  a.epoch = ctx->next_epoch();
  a.nvals = vals.n;
  a.gen_ids = vals.gen_ids;
  for (int c = 0; c < vals.n; ++c) {
    a.vin[c] = vals.in[c];
    a.vout[c] = vals.out[c];
    a.vbytes[c] = vals.bytes[c];
  }
  ctx->kbegin("scatter_pass_ldg", n * (row + wrow));
  if (key_bytes == 4)
    k_scatter_pass<uint32_t><<<(unsigned)tiles, kPassThreads, 0, ctx->stream>>>(a);
  else
    k_scatter_pass<uint64_t><<<(unsigned)tiles, kPassThreads, 0, ctx->stream>>>(a);
  ctx->kend();
  CJ_CUDA(cudaGetLastError());
}

void copy_columns(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int key_bytes,
                  const ValCols& vals) {
  if (n == 0) return;
  if (keys_out != keys)
    CJ_CUDA(cudaMemcpyAsync(keys_out, keys, n * key_bytes, cudaMemcpyDeviceToDevice,
                            ctx->stream));
  for (int c = 0; c < vals.n; ++c) {
    if (vals.gen_ids && c == 0) {
      ctx->kbegin("iota", n * 4);
      k_iota<uint32_t><<<grid_for(n, 256 * 8, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
          static_cast<uint32_t*>(vals.out[0]), n);
      ctx->kend();
    } else if (vals.out[c] != vals.in[c]) {
      CJ_CUDA(cudaMemcpyAsync(vals.out[c], vals.in[c], n * vals.bytes[c],
                              cudaMemcpyDeviceToDevice, ctx->stream));
    }
  }
}

namespace {
void lsd_partition_group(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int key_bytes,
                         const PassPlan& plan, const ValCols& vals,
                         std::vector<uint32_t>* counts_out, unsigned long long* key_or);
}  // namespace

// Wide rows are partitioned in column groups of at most 32 payload bytes: each
// group runs the same stable LSD plan with the key, so every group sees the same
// permutation (the reference re-partitions each GFTR payload column with the key
// the same way, join_engine.cpp:180-213).
void lsd_partition(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int key_bytes,
                   const PassPlan& plan, const ValCols& vals, std::vector<uint32_t>* counts_out,
                   unsigned long long* key_or) {
  // payload bytes per column group (CJ_GROUP_BYTES: experiments)
  static const uint32_t kGroupBytes = [] {
    const char* e = std::getenv("CJ_GROUP_BYTES");
    return e ? (uint32_t)std::max(4, std::atoi(e)) : 32u;
  }();
  uint32_t total = 0;
  for (int c = 0; c < vals.n; ++c) total += vals.bytes[c];
  if (total <= kGroupBytes)
    return lsd_partition_group(ctx, keys, keys_out, n, key_bytes, plan, vals, counts_out, key_or);
  int c = 0;
  bool first = true;
  while (c < vals.n) {
    ValCols g;
    uint32_t bytes = 0;
    while (c < vals.n && (g.n == 0 || bytes + vals.bytes[c] <= kGroupBytes)) {
      g.in[g.n] = vals.in[c];
      g.out[g.n] = vals.out[c];
      g.bytes[g.n] = vals.bytes[c];
      bytes += vals.bytes[c];
      ++g.n;
      ++c;
    }
    g.gen_ids = first ? vals.gen_ids : 0;
    lsd_partition_group(ctx, keys, keys_out, n, key_bytes, plan, g, first ? counts_out : nullptr,
                        first ? key_or : nullptr);
    first = false;
  }
}

namespace {
void lsd_partition_group(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int key_bytes,
                         const PassPlan& plan, const ValCols& vals,
                         std::vector<uint32_t>* counts_out, unsigned long long* key_or) {
  if (plan.npasses > 8) fail(CJ_ERR_UNSUPPORTED, "LSD segment longer than 8 passes");
  const int np = plan.npasses;
  // digit tables sized to the widest pass: 64 digits for passes of <= 6 bits
  // (smaller shared-memory tables leave room for longer tiles), else 256
  int rb = 6;
  for (int p = 0; p < np; ++p) rb = std::max(rb, (int)(plan.hi[p] - plan.lo[p]));
  if (plan.npasses > 0 && std::getenv("CJ_RB8")) rb = 8;
  ScatterGeom g0 = scatter_geom(ctx, n, key_bytes, vals, keys, rb);
  if (rb != 8 && !g0.tma) {  // the look-back onesweep fallback has 256-digit tables
    rb = 8;
    g0 = scatter_geom(ctx, n, key_bytes, vals, keys, rb);
  }
  const uint32_t kRadix = 1u << rb;
  std::vector<uint32_t> totals;
  Scratch cnt(ctx, sizeof(uint32_t) * kRadix * std::max(np, 1) * g0.nblocks);
  Scratch tot(ctx, sizeof(uint32_t) * kRadix * std::max(np, 1));
  Scratch base(ctx, sizeof(uint64_t) * kRadix * std::max(np, 1));
  // Constant-digit passes are skipped (primitives.cpp:224-226) after one host
  // round trip for the digit totals; callers that know their passes are live
  // (ctx->assume_live_passes) run every pass instead and save the sync.
  const bool skip_check = ctx->assume_live_passes && !counts_out;
  // Four or more live passes (SMJ's 7-bit digits): counting every pass's
  // digits in one read costs ~2x a read (four shared atomics per key), and the
  // later passes re-read their keys for per-block counts anyway; so the first
  // read counts only the first pass and each later pass takes its digit bases
  // from its own re-read (the re-read's last CTA computes them).
  int first_live = -1, nlive = 0;
  for (int p = 0; p < np; ++p)
    if (plan.hi[p] != plan.lo[p] && p >= plan.done) {
      if (first_live < 0) first_live = p;
      ++nlive;
    }
  const bool per_pass_bases = skip_check && nlive >= 4 && g0.tma;
  if (per_pass_bases) {
    PassPlan one;
    one.npasses = 1;
    one.lo[0] = plan.lo[first_live];
    one.hi[0] = plan.hi[first_live];
    histogram_passes(ctx, keys, n, key_bytes, one, g0, cnt.as<uint32_t>(),
                     tot.as<uint32_t>() + (size_t)first_live * kRadix,
                     base.as<uint64_t>() + (size_t)first_live * kRadix, nullptr, 0, 0, key_or);
  } else {
    histogram_passes(ctx, keys, n, key_bytes, plan, g0, cnt.as<uint32_t>(), tot.as<uint32_t>(),
                     base.as<uint64_t>(), skip_check ? nullptr : &totals, 0, 0, key_or);
  }
  if (counts_out) *counts_out = totals;
  std::vector<int> live;
  for (int p = 0; p < np; ++p) {
    if (plan.hi[p] == plan.lo[p] || p < plan.done) continue;
    bool constant = n == 0;
    for (uint32_t d = 0; d < kRadix && !constant && !skip_check; ++d)
      if (totals[(size_t)p * kRadix + d] == n) constant = true;
    if (!constant) live.push_back(p);
  }
  if (live.empty()) {
    copy_columns(ctx, keys, keys_out, n, key_bytes, vals);
    return;
  }
  // ping-pong scratch; the first target is chosen so the last pass lands in
  // the caller's buffers (primitives.cpp:236-255)
  const int nv = vals.n;
  Scratch sk(ctx, live.size() > 1 ? n * key_bytes + kPad : 0);
  uint64_t vbytes_total = 0;
  auto col_span = [&](int c) { return (n * vals.bytes[c] + kPad + 255) & ~uint64_t(255); };
  for (int c = 0; c < nv; ++c) vbytes_total += col_span(c);
  Scratch svals(ctx, live.size() > 1 ? vbytes_total : 0);
  void* scratch_cols[CJ_MAX_COLS + 1] = {};
  {
    uint64_t off = 0;  // 256-byte aligned column starts
    for (int c = 0; c < nv; ++c) {
      scratch_cols[c] = static_cast<char*>(svals.p) + off;
      off += col_span(c);
    }
  }
  // later passes may tile differently (the first pass generates GFUR ids
  // instead of staging them): size for the most blocks any geometry uses
  const uint64_t max_blocks = (uint64_t)ctx->num_sms * 2;
  Scratch cnt2(ctx, live.size() > 1 ? sizeof(uint32_t) * kRadix * max_blocks + 4096 : 0);
  const void* cur_k = keys;
  ValCols cur = vals;
  bool to_out = (live.size() % 2) == 1;
  for (size_t li = 0; li < live.size(); ++li) {
    const int p = live[li];
    ValCols step = cur;
    void* tk = to_out ? keys_out : sk.p;
    for (int c = 0; c < nv; ++c) step.out[c] = to_out ? vals.out[c] : scratch_cols[c];
    step.gen_ids = li == 0 ? vals.gen_ids : 0;
    const uint64_t* pbase = base.as<uint64_t>() + (size_t)p * kRadix;
    // after an earlier pass (or a presorted first digit) the rows arrive in runs
    const int runs = li > 0 || plan.done > 0;
    if (li == 0) {
      // (per_pass_bases: the first read counted this pass alone)
      scatter_pass(ctx, cur_k, tk, n, key_bytes, plan.lo[p], plan.hi[p], pbase,
                   g0.tma ? cnt.as<uint32_t>() + (per_pass_bases ? 0 : (size_t)p * kRadix) : nullptr,
                   (uint32_t)(kRadix * (per_pass_bases ? 1 : np)), g0, step, 0, 0, runs);
    } else {
      const ScatterGeom g = scatter_geom(ctx, n, key_bytes, step, cur_k, rb);
      const uint32_t* pc = nullptr;
      if (g.tma || per_pass_bases) {
        PassPlan one;
        one.npasses = 1;
        one.lo[0] = plan.lo[p];
        one.hi[0] = plan.hi[p];
        // (a pass without the TMA geometry counts in the first pass's tiling:
        // only its digit totals are used)
        const ScatterGeom& gh = g.tma ? g : g0;
        if ((uint64_t)gh.nblocks > max_blocks) fail(CJ_ERR_CUDA, "block count scratch too small");
        // (per_pass_bases: its last CTA writes this pass's totals and bases)
        block_hist(ctx, cur_k, n, key_bytes, one, gh, cnt2.as<uint32_t>(), 0, 0, nullptr,
                   per_pass_bases ? tot.as<uint32_t>() + (size_t)p * kRadix : nullptr,
                   per_pass_bases ? base.as<uint64_t>() + (size_t)p * kRadix : nullptr);
        if (g.tma) pc = cnt2.as<uint32_t>();
      }
      scatter_pass(ctx, cur_k, tk, n, key_bytes, plan.lo[p], plan.hi[p], pbase, pc, kRadix, g,
                   step, 0, 0, runs);
    }
    cur_k = tk;
    for (int c = 0; c < nv; ++c) cur.in[c] = step.out[c];
    cur.gen_ids = 0;
    to_out = !to_out;
  }
}

}  // namespace

// Stable partition by (shard, low `lowbits` key bits): the send layout of the
// multi-GPU shuffle, grouped by destination and, inside a destination, by the
// receiver's first LSD digit.  Rows wider than the TMA stage allows are
// partitioned in column groups (each group with the key: the digits are the
// same, so every group gets the same stable permutation).
void shard_partition(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int key_bytes,
                     uint32_t parts, uint32_t lowbits, const ValCols& vals, uint64_t* counts_host) {
  if (parts == 0 || parts > 256) fail(CJ_ERR_SPEC_INVALID, "shard count must be in [1, 256]");
  if (lowbits > 8 || ((uint64_t)parts << lowbits) > 256)
    fail(CJ_ERR_FANOUT_TOO_LARGE, "shards x 2^first_bits must not exceed 256 digits");
  const uint32_t digits = parts << lowbits;
  PassPlan plan;
  plan.npasses = 1;
  plan.lo[0] = 0;
  plan.hi[0] = 8;
  constexpr uint32_t kGroupBytes = 32;
  std::vector<ValCols> groups;
  {
    ValCols cur;
    uint32_t bytes = 0;
    for (int c = 0; c < vals.n; ++c) {
      if (cur.n > 0 && bytes + vals.bytes[c] > kGroupBytes) {
        groups.push_back(cur);
        cur = ValCols();
        bytes = 0;
      }
      cur.in[cur.n] = vals.in[c];
      cur.out[cur.n] = vals.out[c];
      cur.bytes[cur.n] = vals.bytes[c];
      ++cur.n;
      bytes += vals.bytes[c];
    }
    groups.push_back(cur);
  }
  std::vector<uint32_t> totals;
  // up to 64 digits: 64-entry digit tables (longer tiles fit), else 256
  const int rb = digits <= 64 ? 6 : 8;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    const ScatterGeom g = scatter_geom(ctx, n, key_bytes, groups[gi], keys, rb);
    if (!g.tma) fail(CJ_ERR_UNSUPPORTED, "shard partition needs 16-byte aligned columns");
    Scratch cnt(ctx, sizeof(uint32_t) * kRadix * g.nblocks), tot(ctx, sizeof(uint32_t) * kRadix),
        base(ctx, sizeof(uint64_t) * kRadix);
    histogram_passes(ctx, keys, n, key_bytes, plan, g, cnt.as<uint32_t>(), tot.as<uint32_t>(),
                     base.as<uint64_t>(), gi == 0 ? &totals : nullptr, parts, lowbits);
    if (n > 0)
      scatter_pass(ctx, keys, keys_out, n, key_bytes, 0, 8, base.as<uint64_t>(),
                   cnt.as<uint32_t>(), 1u << g.rb, g, groups[gi], parts, lowbits);
  }
  for (uint32_t d = 0; d < digits; ++d) counts_host[d] = n ? totals[d] : 0;
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
}

namespace {
template <class K>
__global__ void k_key_or(const K* __restrict__ keys, uint64_t n, unsigned long long* out) {
  K acc = 0;
  constexpr int kVec = 16 / sizeof(K);
  const uint4* kv = reinterpret_cast<const uint4*>(keys);
  const uint64_t nvec = n / kVec;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 q = __ldcs(kv + v);
    K e[kVec];
    memcpy(e, &q, 16);
#pragma unroll
    for (int j = 0; j < kVec; ++j) acc |= e[j];
  }
  for (uint64_t i = nvec * kVec + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc |= keys[i];
  uint64_t a64 = (uint64_t)acc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a64 |= __shfl_xor_sync(0xffffffffu, a64, o);
  if ((threadIdx.x & 31) == 0 && a64) atomicOr(out, (unsigned long long)a64);
}
}  // namespace

// Stable full-width sort plan (sort_pairs, primitives.cpp:358-362): LSD digits
// over the significant bits of the keys only (higher bits are zero for every
// key, so those passes would be constant and skipped anyway), ceil(bits / 8)
// passes of balanced width — e.g. 27-bit keys: 7+7+7+6 bits, which scatter
// faster than 8+8+8+3 (fewer digits per pass: longer runs per tile).  9-bit
// digits (3 passes) measured slower than four narrow passes (r01d).  The stable
// result is the same for every split.
PassPlan sort_plan(cj_ctx* ctx, const void* keys, uint64_t n, int key_bytes, const ValCols& vals) {
  uint32_t bits = (uint32_t)key_bytes * 8;
  if (n > 0 && (reinterpret_cast<uintptr_t>(keys) & 15u) == 0) {
    Scratch acc(ctx, 8);
    CJ_CUDA(cudaMemsetAsync(acc.p, 0, 8, ctx->stream));
    ctx->kbegin("key_bits", n * key_bytes);
    if (key_bytes == 4)
      k_key_or<uint32_t><<<grid_for(n / 4, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
          static_cast<const uint32_t*>(keys), n, acc.as<unsigned long long>());
    else
      k_key_or<uint64_t><<<grid_for(n / 2, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
          static_cast<const uint64_t*>(keys), n, acc.as<unsigned long long>());
    ctx->kend();
    uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
    CJ_CUDA(cudaMemcpyAsync(h, acc.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    bits = h[0] ? 64u - (uint32_t)__builtin_clzll(h[0]) : 1u;
  }
  const uint32_t np = (bits + 7) / 8;
  PassPlan plan;
  plan.npasses = (int)np;
  uint32_t lo = 0;
  for (uint32_t p = 0; p < np; ++p) {  // balanced widths, each <= 8 (or 9)
    const uint32_t w = (bits - lo + (np - p) - 1) / (np - p);
    plan.lo[p] = lo;
    plan.hi[p] = lo + w;
    lo += w;
  }
  return plan;
}

void partition_offsets(cj_ctx* ctx, const void* keys_sorted, uint64_t n, int key_bytes,
                       uint32_t bits, uint64_t* offsets_dev) {
  const uint64_t fanout = 1ull << bits;
  // small inputs: one pass over the keys beats (fanout + 1) chains of
  // log2(n) dependent loads (C1: 2^22 keys, 13 -> ~5 us)
  if (n > 0 && n <= (1ull << 23)) {
    ctx->kbegin("offsets", (uint64_t)key_bytes * n + 8 * (fanout + 1));
    const unsigned g2 = grid_for(n, 256, ctx->num_sms * 8);
    if (key_bytes == 4)
      k_offsets_scan<uint32_t><<<g2, 256, 0, ctx->stream>>>(
          static_cast<const uint32_t*>(keys_sorted), n, bits, offsets_dev);
    else
      k_offsets_scan<uint64_t><<<g2, 256, 0, ctx->stream>>>(
          static_cast<const uint64_t*>(keys_sorted), n, bits, offsets_dev);
    ctx->kend();
    CJ_CUDA(cudaGetLastError());
    return;
  }
  const unsigned grid = grid_for(fanout + 1, 256, 4096);
  ctx->kbegin("offsets", 8 * (fanout + 1));
  if (key_bytes == 4)
    k_offsets<uint32_t><<<grid, 256, 0, ctx->stream>>>(
        static_cast<const uint32_t*>(keys_sorted), n, bits, offsets_dev);
  else
    k_offsets<uint64_t><<<grid, 256, 0, ctx->stream>>>(
        static_cast<const uint64_t*>(keys_sorted), n, bits, offsets_dev);
  ctx->kend();
  CJ_CUDA(cudaGetLastError());
}

}  // namespace cj

#ifdef CJ_PHASE_CLOCKS
extern "C" void cj_debug_phase_clocks(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, cj::g_phase_clk, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(cj::g_phase_clk, z, sizeof(z));
  }
}
#endif
