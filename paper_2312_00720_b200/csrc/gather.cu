// Gather / materialise (K6): out[c][i] = in[c][map[i]] for several columns
// sharing one map (primitives.cpp:369-396, join_engine.cpp:161-176).
//
// The map is read once per launch for all columns; each thread keeps
// kUnroll independent loads in flight so random (GFUR) maps stay
// sector-throughput bound rather than latency bound.  Out-of-range map
// entries set the ctx error word (IndexOutOfBounds after the phase).
#include <algorithm>

#include "cj_device.cuh"
#include "cj_internal.cuh"

namespace cj {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 8;

struct GatherArgs {
  const void* in[CJ_MAX_COLS * 2];
  void* out[CJ_MAX_COLS * 2];
  uint32_t bytes[CJ_MAX_COLS * 2];
  int ncols;
  const uint32_t* map;
  uint64_t m, n_in;
  uint32_t* err;
};

__global__ void __launch_bounds__(kThreads) k_gather(const __grid_constant__ GatherArgs a) {
  const uint64_t chunk = (uint64_t)kThreads * kUnroll;
  for (uint64_t base = (uint64_t)blockIdx.x * chunk; base < a.m; base += (uint64_t)gridDim.x * chunk) {
    uint32_t idx[kUnroll];
    bool ok[kUnroll];
    bool bad = false;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t i = base + (uint64_t)u * kThreads + threadIdx.x;
      ok[u] = i < a.m;
      idx[u] = ok[u] ? __ldcs(a.map + i) : 0u;
      if (ok[u] && idx[u] >= a.n_in) {
        bad = true;
        ok[u] = false;
      }
    }
    if (bad) atomicOr(a.err, kErrOOB);
    for (int c = 0; c < a.ncols; ++c) {
      if (a.bytes[c] == 4) {
        const uint32_t* __restrict__ in = static_cast<const uint32_t*>(a.in[c]);
        uint32_t* __restrict__ out = static_cast<uint32_t*>(a.out[c]);
        uint32_t v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = ok[u] ? __ldg(in + idx[u]) : 0u;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (ok[u]) __stcs(out + base + (uint64_t)u * kThreads + threadIdx.x, v[u]);
      } else {
        const unsigned long long* __restrict__ in = static_cast<const unsigned long long*>(a.in[c]);
        unsigned long long* __restrict__ out = static_cast<unsigned long long*>(a.out[c]);
        unsigned long long v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = ok[u] ? __ldg(in + idx[u]) : 0ull;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (ok[u]) __stcs(out + base + (uint64_t)u * kThreads + threadIdx.x, v[u]);
      }
    }
  }
}

}  // namespace

void gather_cols(cj_ctx* ctx, const void* const* in, uint64_t n_in, const uint32_t* map,
                 uint64_t m, void* const* out, const uint32_t* bytes, int ncols) {
  if (m == 0 || ncols == 0) return;
  for (int c0 = 0; c0 < ncols; c0 += CJ_MAX_COLS * 2) {
    GatherArgs a{};
    a.ncols = std::min(ncols - c0, CJ_MAX_COLS * 2);
    for (int c = 0; c < a.ncols; ++c) {
      a.in[c] = in[c0 + c];
      a.out[c] = out[c0 + c];
      a.bytes[c] = bytes[c0 + c];
    }
    a.map = map;
    a.m = m;
    a.n_in = n_in;
    a.err = ctx->err_word;
    const unsigned grid = grid_for(m, kThreads * kUnroll, ctx->num_sms * 8);
    uint64_t alg = (uint64_t)m * 4;
    for (int c = 0; c < a.ncols; ++c) alg += 2ull * m * a.bytes[c];
    ctx->kbegin("gather", alg);
    k_gather<<<grid, kThreads, 0, ctx->stream>>>(a);
    ctx->kend();
    CJ_CUDA(cudaGetLastError());
  }
}

}  // namespace cj
