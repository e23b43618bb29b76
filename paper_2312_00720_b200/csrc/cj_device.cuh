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

}  // namespace dev
}  // namespace cj
