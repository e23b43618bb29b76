// Per-phase cycle counts of the scatter pass (tooling, not product).  Built by
// tools/Makefile with radix.cu compiled -DCJ_PHASE_CLOCKS.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include "cj_api.h"
extern "C" void cj_debug_phase_clocks(unsigned long long* out, int reset);

__global__ void k_fill(uint32_t* p, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull + seed;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    p[i] = (uint32_t)(x ^ (x >> 31));
  }
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 28);
  cj_ctx* ctx;
  cj_ctx_create(0, nullptr, &ctx);
  uint32_t *k, *ko, *v[2], *vo[2];
  cudaMalloc(&k, n * 4 + 64); cudaMalloc(&ko, n * 4 + 64);
  for (int c = 0; c < 2; ++c) { cudaMalloc(&v[c], n * 4 + 64); cudaMalloc(&vo[c], n * 4 + 64); }
  k_fill<<<1184, 256>>>(k, n, 1); k_fill<<<1184, 256>>>(v[0], n, 2); k_fill<<<1184, 256>>>(v[1], n, 3);
  cudaDeviceSynchronize();
  const uint32_t lo[2] = {0, 8}, hi[2] = {8, 16}, vb[2] = {4, 4};
  const void* vin[2] = {v[0], v[1]};
  void* vout[2] = {vo[0], vo[1]};
  unsigned long long clk[16];
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    cj_debug_phase_clocks(clk, 1);
    cudaEventRecord(e0);
    int st = cj_radix_partition_passes(ctx, k, ko, n, 4, lo, hi, 2, vin, vout, vb, 2, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cj_debug_phase_clocks(clk, 0);
    unsigned long long tot = 0;
    for (int i = 0; i < 8; ++i) tot += clk[i];
    printf("it %d status %d  %.3f ms  CTA0 cycles: rank %llu scan1 %llu scan2 %llu place %llu write %llu  (sum %llu)\n",
           it, st, ms, clk[0], clk[2], clk[3], clk[1], clk[7], tot);
    printf("   ws rankers: wait_full %llu rank %llu wait_wd %llu bar %llu scan+place %llu | writers: wait_rd %llu write %llu bar %llu\n",
           clk[8], clk[9], clk[10], clk[11], clk[12], clk[13], clk[14], clk[15]);
  }
  return 0;
}
