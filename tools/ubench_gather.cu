// Microbenchmark (tooling, not product): the random-gather ceiling of one B200
// for GFUR's materialisation shape — out[c][i] = in[c][map[i]] with a uniformly
// random map over a table far larger than L2 — as a function of the loads in
// flight per thread and of the column count, next to the same map sorted
// (sequential) for scale.  K6 k_gather (csrc/gather.cu) is judged against the
// best random figure here, not against the streaming HBM peak.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

template <int U, int C>
__global__ void __launch_bounds__(256) k_rg(const uint32_t* __restrict__ map,
                                            const uint32_t* const* __restrict__ in,
                                            uint32_t* const* __restrict__ out, size_t m) {
  const size_t chunk = 256 * (size_t)U;
  for (size_t base = blockIdx.x * chunk; base < m; base += (size_t)gridDim.x * chunk) {
    uint32_t idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + u * 256 + threadIdx.x;
      idx[u] = i < m ? __ldcs(map + i) : 0u;
    }
    uint32_t v[C][U];
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int u = 0; u < U; ++u) v[c][u] = __ldg(in[c] + idx[u]);
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t i = base + u * 256 + threadIdx.x;
        if (i < m) __stcs(out[c] + i, v[c][u]);
      }
  }
}

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static uint64_t next_u64() {
  rng_state ^= rng_state << 13;
  rng_state ^= rng_state >> 7;
  rng_state ^= rng_state << 17;
  return rng_state;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t m = 1ull << 28;  // C2: 2^28 output rows (gathers per column)
  const size_t n_max = 1ull << 28;
  std::vector<uint32_t> h(m);
  uint32_t *map, *map_sorted, *in_b, *out_b;
  CK(cudaMalloc(&map, m * 4));
  CK(cudaMalloc(&map_sorted, m * 4));
  CK(cudaMalloc(&in_b, 4 * n_max * 4));
  CK(cudaMalloc(&out_b, 4 * m * 4));
  CK(cudaMemset(in_b, 1, 4 * n_max * 4));
  uint32_t **din, **dout;
  CK(cudaMalloc(&din, 4 * sizeof(uint32_t*)));
  CK(cudaMalloc(&dout, 4 * sizeof(uint32_t*)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, auto kern, int u, int c, int per_sm, const uint32_t* mp) {
    const size_t chunk = 256ull * u;
    const size_t need = (m + chunk - 1) / chunk;
    const int grid = (int)std::min<size_t>(need, (size_t)sms * per_sm);
    for (int w = 0; w < 2; ++w) kern<<<grid, 256>>>(mp, din, dout, m);
    CK(cudaEventRecord(e0));
    const int reps = 5;
    for (int r = 0; r < reps; ++r) kern<<<grid, 256>>>(mp, din, dout, m);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    const double g = (double)m * c / (ms * 1e-3);  // gathers per second
    printf("%-8s U=%2d cols=%d ctas/SM=%2d: %7.3f ms  %6.2f Ggather/s  useful %6.0f GB/s\n", name, u,
           c, per_sm, ms, g * 1e-9, (m * 4.0 + 2.0 * 4 * m * c) / (ms * 1e6));
  };
  // table rows: C2's R side (2^27) and S side (2^28); 4-byte columns
  for (size_t n_in : {1ull << 27, 1ull << 28}) {
    for (size_t i = 0; i < m; ++i) h[i] = (uint32_t)(next_u64() % n_in);
    CK(cudaMemcpy(map, h.data(), m * 4, cudaMemcpyHostToDevice));
    std::sort(h.begin(), h.end());
    CK(cudaMemcpy(map_sorted, h.data(), m * 4, cudaMemcpyHostToDevice));
    uint32_t* hin[4];
    uint32_t* hout[4];
    for (int c = 0; c < 4; ++c) {
      hin[c] = in_b + c * n_in;
      hout[c] = out_b + c * m;
    }
    CK(cudaMemcpy(din, hin, sizeof(hin), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dout, hout, sizeof(hout), cudaMemcpyHostToDevice));
    printf("== %zu-row tables (%zu MB per column), uniform random map of %zu entries\n", n_in,
           n_in * 4 >> 20, m);
    for (int per_sm : {4, 8, 16}) {
      run("random", k_rg<8, 1>, 8, 1, per_sm, map);
      run("random", k_rg<16, 1>, 16, 1, per_sm, map);
      run("random", k_rg<32, 1>, 32, 1, per_sm, map);
      run("random", k_rg<16, 2>, 16, 2, per_sm, map);
      run("random", k_rg<8, 4>, 8, 4, per_sm, map);
    }
    run("sorted", k_rg<16, 2>, 16, 2, 8, map_sorted);
  }
  // cudaLimitMaxL2FetchGranularity (32 / 64 / 128) was measured to change
  // none of these figures (profiles/r02d_gather_ceiling.md)
  return 0;
}
