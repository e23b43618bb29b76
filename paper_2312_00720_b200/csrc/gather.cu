// Gather / materialise (K6): out[c][i] = in[c][map[i]] for several columns
// sharing one map (primitives.cpp:369-396, join_engine.cpp:161-176).
//
// The map is read once per launch for all columns; each thread keeps
// U * G independent loads in flight (U map entries x a group of G columns) so
// random (GFUR) maps stay sector-throughput bound rather than latency bound.  Out-of-range map
// entries set the ctx error word (IndexOutOfBounds after the phase).
#include <algorithm>
#include <cstdlib>

#include "cj_device.cuh"
#include "cj_internal.cuh"

namespace cj {
namespace {

constexpr int kThreads = 256;

struct GatherArgs {
  const void* in[CJ_MAX_COLS * 2];
  void* out[CJ_MAX_COLS * 2];
  uint32_t bytes[CJ_MAX_COLS * 2];
  int ncols;
  const uint32_t* map;
  uint64_t m, n_in;
  uint32_t* err;
};

// U map entries per thread; columns in groups of G whose loads are all issued
// before the group's stores (U * G independent loads in flight per thread).
template <int U, int G>
__global__ void __launch_bounds__(kThreads) k_gather(const __grid_constant__ GatherArgs a) {
  const uint64_t chunk = (uint64_t)kThreads * U;
  for (uint64_t base = (uint64_t)blockIdx.x * chunk; base < a.m; base += (uint64_t)gridDim.x * chunk) {
    uint32_t idx[U];
    bool ok[U];
    bool bad = false;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + (uint64_t)u * kThreads + threadIdx.x;
      ok[u] = i < a.m;
      idx[u] = ok[u] ? __ldcs(a.map + i) : 0u;
      if (ok[u] && idx[u] >= a.n_in) {
        bad = true;
        ok[u] = false;
      }
    }
    if (bad) atomicOr(a.err, kErrOOB);
    for (int c0 = 0; c0 < a.ncols; c0 += G) {
      unsigned long long v[G][U];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int c = c0 + g;
        if (c >= a.ncols) break;
        if (a.bytes[c] == 4) {
          const uint32_t* __restrict__ in = static_cast<const uint32_t*>(a.in[c]);
#pragma unroll
          for (int u = 0; u < U; ++u) v[g][u] = ok[u] ? __ldg(in + idx[u]) : 0u;
        } else {
          const unsigned long long* __restrict__ in = static_cast<const unsigned long long*>(a.in[c]);
#pragma unroll
          for (int u = 0; u < U; ++u) v[g][u] = ok[u] ? __ldg(in + idx[u]) : 0ull;
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int c = c0 + g;
        if (c >= a.ncols) break;
        if (a.bytes[c] == 4) {
          uint32_t* __restrict__ out = static_cast<uint32_t*>(a.out[c]);
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (ok[u]) __stcs(out + base + (uint64_t)u * kThreads + threadIdx.x, (uint32_t)v[g][u]);
        } else {
          unsigned long long* __restrict__ out = static_cast<unsigned long long*>(a.out[c]);
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (ok[u]) __stcs(out + base + (uint64_t)u * kThreads + threadIdx.x, v[g][u]);
        }
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
    // 16 map entries x 2 columns in flight per thread (C2 GFUR gathers
    // 20.7 -> 18.3 ms against 8 x 1; 8 x 4 and 4 x 4 lose occupancy);
    // CJ_GATHER selects the others for measurement
    static const int mode = [] {
      const char* e = std::getenv("CJ_GATHER");
      return e ? std::atoi(e) : 4;
    }();
    uint64_t alg = (uint64_t)m * 4;
    for (int c = 0; c < a.ncols; ++c) alg += 2ull * m * a.bytes[c];
    ctx->kbegin("gather", alg);
    auto launch = [&](auto kern, int u) {
      kern<<<grid_for(m, kThreads * u, ctx->num_sms * 8), kThreads, 0, ctx->stream>>>(a);
    };
    switch (mode) {
      case 1: launch(k_gather<8, 1>, 8); break;
      case 2: launch(k_gather<16, 1>, 16); break;
      case 3: launch(k_gather<8, 4>, 8); break;
      default: launch(k_gather<16, 2>, 16); break;
    }
    ctx->kend();
    CJ_CUDA(cudaGetLastError());
  }
}

}  // namespace cj
