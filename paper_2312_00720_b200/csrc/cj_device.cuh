// Device-side helpers: memory-order primitives for decoupled look-back,
// warp scans, and the 64-bit status word format.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cj {
namespace dev {

// Look-back status word: [63:48] epoch, [47:46] flag, [45:0] value.
// A word whose epoch differs from the launch's is "not yet written", so the
// status buffer never needs clearing between launches.
constexpr uint64_t kFlagAgg = 1ull, kFlagIncl = 2ull;
constexpr uint64_t kValMask = (1ull << 46) - 1;

__device__ __forceinline__ uint64_t pack_status(uint64_t epoch, uint64_t flag, uint64_t v) {
  return (epoch << 48) | (flag << 46) | (v & kValMask);
}
__device__ __forceinline__ uint64_t st_flag(uint64_t w, uint64_t epoch) {
  return (w >> 48) == epoch ? ((w >> 46) & 3ull) : 0ull;
}

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <class T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= (unsigned)o) v += n;
  }
  return v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Spin bound of every look-back wait: a predecessor that never publishes (a
// bug, never a legal schedule) raises kErrStall instead of hanging the GPU.
constexpr uint32_t kSpinLimit = 1u << 26;
constexpr uint32_t kErrStall = 16u;

// Warp-cooperative decoupled look-back over a single-value chain.
// Returns the exclusive prefix of `idx` (sum of values of all earlier ids),
// having published `agg` for idx.  Called by one full warp.
__device__ __forceinline__ uint64_t warp_lookback(uint64_t* status, uint64_t idx, uint64_t agg,
                                                  uint64_t epoch, uint32_t* err) {
  const unsigned lane = lane_id();
  if (idx == 0) {
    if (lane == 0) st_relaxed(status, pack_status(epoch, kFlagIncl, agg));
    return 0;
  }
  if (lane == 0) st_relaxed(status + idx, pack_status(epoch, kFlagAgg, agg));
  uint64_t excl = 0;
  int64_t hi = (int64_t)idx - 1;  // window [hi-31, hi]
  while (true) {
    const int64_t my = hi - (int64_t)lane;
    uint64_t w = 0, f = 2;  // out-of-range lanes count as "inclusive 0"
    if (my >= 0) {
      uint32_t spins = 0;
      do {
        w = ld_relaxed(status + my);
        f = st_flag(w, epoch);
        if (f == 0 && ++spins > kSpinLimit) {
          atomicOr(err, kErrStall);
          f = kFlagIncl;
          w = 0;
        }
      } while (f == 0);
    }
    const uint64_t v = my >= 0 ? (w & kValMask) : 0;
    const uint32_t incl = __ballot_sync(0xffffffffu, f == kFlagIncl);
    // lanes up to and including the first (lowest lane) inclusive contribute
    const int stop = incl ? __ffs(incl) - 1 : 31;
    uint64_t contrib = (int)lane <= stop ? v : 0;
    excl += warp_sum(contrib);
    if (incl) break;
    hi -= 32;
  }
  if (lane == 0) st_relaxed(status + idx, pack_status(epoch, kFlagIncl, excl + agg));
  return excl;
}

// SplitMix64 finaliser (the reference's rng.hpp:8-12), used as the shard hash.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Shard digit of a key: shard = floor(mix64(key) * hparts / 2^64) —
// uncorrelated with the low key bits that pick partitions and hash slots —
// followed by the key's low `lowbits` bits (the receiver's first LSD digit).
__device__ __forceinline__ uint32_t shard_digit(uint64_t k, uint32_t hparts, uint32_t lowbits) {
  const uint32_t s = (uint32_t)__umul64hi(mix64(k), (uint64_t)hparts);
  return (s << lowbits) | ((uint32_t)k & ((1u << lowbits) - 1u));
}

// ---- TMA bulk copies (cp.async.bulk) + mbarrier ----------------------------

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// order earlier generic-proxy shared accesses before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// Named barrier among `count` threads (a multiple of 32) of the CTA; id 1..15.
__device__ __forceinline__ void named_bar(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// Named-barrier OR reduction among `count` threads (a multiple of 32).
__device__ __forceinline__ bool named_bar_or(uint32_t id, uint32_t count, bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "barrier.red.or.pred q, %2, %3, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id), "r"(count)
      : "memory");
  return r != 0;
}
// 1-D bulk copy global -> shared; 16-byte aligned addresses, size % 16 == 0.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// Stable in-warp peers of a 9-bit (or narrower) digit by bit ballots: the
// lanes holding the same digit, restricted to `valid` lanes.
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, uint32_t bits, uint32_t valid) {
  uint32_t peers = valid;
#pragma unroll
  for (uint32_t b = 0; b < 9; ++b) {
    if (b < bits) {
      const bool set = (d >> b) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, set);
      peers &= set ? bal : ~bal;
    }
  }
  return peers;
}

// Exclusive scan of n u64 counts in three small launches (block scans, a scan
// of the block totals, fix-up); no inter-block waiting.
constexpr int kScanThreads = 512, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

template <int = 0>
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const uint64_t* __restrict__ in,
                                                             uint64_t n, uint64_t* __restrict__ out,
                                                             uint64_t* __restrict__ tile_tot) {
  __shared__ uint64_t wsum[kScanThreads / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint64_t v[kScanItems], local = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    local += v[i];
  }
  const uint64_t inc = warp_inclusive_sum(local);
  if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = inc;
  __syncthreads();
  uint64_t off = 0;
  for (unsigned w = 0; w < (threadIdx.x >> 5); ++w) off += wsum[w];
  uint64_t run = off + inc - local;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (threadIdx.x == kScanThreads - 1) tile_tot[blockIdx.x] = run;
}

template <int = 0>
__global__ void __launch_bounds__(1024) k_scan_top(uint64_t* __restrict__ tot, uint64_t ntiles,
                                                    uint64_t* __restrict__ total) {
  __shared__ uint64_t wsum[32];
  const uint64_t per = (ntiles + blockDim.x - 1) / blockDim.x;
  const uint64_t i0 = umin64(ntiles, threadIdx.x * per), i1 = umin64(ntiles, i0 + per);
  uint64_t local = 0;
  for (uint64_t i = i0; i < i1; ++i) local += tot[i];
  const uint64_t inc = warp_inclusive_sum(local);
  if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = inc;
  __syncthreads();
  uint64_t off = 0;
  for (unsigned w = 0; w < (threadIdx.x >> 5); ++w) off += wsum[w];
  uint64_t run = off + inc - local;
  for (uint64_t i = i0; i < i1; ++i) {
    const uint64_t t = tot[i];
    tot[i] = run;
    run += t;
  }
  if (threadIdx.x == blockDim.x - 1) *total = run;
}

template <int = 0>
__global__ void k_scan_fix(uint64_t* __restrict__ out, uint64_t n,
                           const uint64_t* __restrict__ tile_off) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += tile_off[i / kScanTile];
}

// 16-byte aligned superset of an element range, for bulk copies of w-byte elements
// (w is a power of two <= 16: 16 / w as a shift, not a division — these run
// ~15 times per staged unit on the producer thread)
__device__ __forceinline__ uint64_t elems16(uint32_t w) { return 16u >> (__ffs((int)w) - 1); }
__device__ __forceinline__ uint64_t align_lo(uint64_t i, uint32_t w) { return i & ~(elems16(w) - 1); }
__device__ __forceinline__ uint64_t align_hi(uint64_t i, uint32_t w) {
  return (i + elems16(w) - 1) & ~(elems16(w) - 1);
}

}  // namespace dev
}  // namespace cj
