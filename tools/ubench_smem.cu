// Shared-memory op throughput with random 8-bit digits (tooling, not product):
// cycles per warp-instruction per SM with 16 warps (1 CTA of 512 threads / SM).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t lanemask_lt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
__device__ __forceinline__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; return x ^ (x >> 16); }

template <int OP>
__global__ void __launch_bounds__(512, 1) k(uint32_t* out, int iters) {
  __shared__ uint32_t tab[16][256];
  __shared__ uint16_t t16[16][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 16 * 256; i += 512) { (&tab[0][0])[i] = 0; (&t16[0][0])[i] = 0; }
  __syncthreads();
  uint32_t acc = 0, seed = hash(threadIdx.x * 7919 + blockIdx.x);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t d = ((seed + it * 0x9E3779B1u) * 0x85EBCA77u) >> 24;
    if (OP == 0) acc += tab[warp][d];                               // LDS random
    if (OP == 1) { tab[warp][d] = acc + it; acc ^= it; }              // STS random
    if (OP == 2) atomicOr(&tab[warp][d], 1u << lane);                // ATOMS.OR
    if (OP == 3) acc += atomicAdd(&tab[warp][d], 1u);                // ATOMS.ADD with return
    if (OP == 4) {                                                   // 8 ballots peers
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) { const bool s = (d >> b) & 1; const uint32_t bal = __ballot_sync(0xffffffffu, s); peers &= s ? bal : ~bal; }
      acc += __popc(peers & lanemask_lt());
    }
    if (OP == 5) acc += __popc(__match_any_sync(0xffffffffu, d) & lanemask_lt());
    if (OP == 6) acc += t16[warp][d];                                // LDS.U16 random
    if (OP == 7) {                                                   // rank0 full item
      atomicOr(&tab[warp][d], 1u << lane); __syncwarp();
      const uint32_t p = tab[warp][d]; __syncwarp();
      const uint32_t lt = p & lanemask_lt(); uint32_t old = 0;
      if (lt == 0) { old = t16[warp][d]; t16[warp][d] = (uint16_t)(old + __popc(p)); tab[warp][d] = 0; }
      old = __shfl_sync(0xffffffffu, old, __ffs(p) - 1);
      acc += old + __popc(lt); __syncwarp();
    }
    if (OP == 8) {                                                   // digit only (baseline)
      acc += d;
    }
    if (OP == 9) {                                                   // rank0 w/o clear via leader atomicAdd
      atomicOr(&tab[warp][d], 1u << lane); __syncwarp();
      const uint32_t p = tab[warp][d]; __syncwarp();
      const uint32_t lt = p & lanemask_lt(); uint32_t old = 0;
      if (lt == 0) { old = atomicAdd((uint32_t*)&t16[0][0] + warp * 128 + (d & 127), __popc(p)); tab[warp][d] = 0; }
      old = __shfl_sync(0xffffffffu, old, __ffs(p) - 1);
      acc += old + __popc(lt); __syncwarp();
    }
    if (OP == 10) {                                                  // peers only (atomicOr + LDS + clear)
      atomicOr(&tab[warp][d], 1u << lane); __syncwarp();
      const uint32_t p = tab[warp][d]; __syncwarp();
      if ((p & lanemask_lt()) == 0) tab[warp][d] = 0;
      acc += p; __syncwarp();
    }
  }
  long long t1 = clock64();
  if (acc == 0x12345678) out[1] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (uint32_t)(t1 - t0);
}

int main() {
  uint32_t* out; cudaMalloc(&out, 8);
  const int iters = 4096;
  const char* names[] = {"LDS random", "STS random", "ATOMS.OR", "ATOMS.ADD ret", "8 ballots", "match.any", "LDS.U16 random", "rank0 item", "digit only", "rank0 atomicAdd", "peers only"};
  void (*ks[])(uint32_t*, int) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>, k<10>};
  for (int o = 0; o < 11; ++o) {
    ks[o]<<<148, 512>>>(out, iters);
    ks[o]<<<148, 512>>>(out, iters);
    cudaDeviceSynchronize();
    uint32_t c; cudaMemcpy(&c, out, 4, cudaMemcpyDeviceToHost);
    // 16 warps each issue `iters` ops: cycles per warp-op per SM
    printf("%-16s %7.2f cycles per warp-op per SM (%s)\n", names[o], (double)c / (iters * 16.0), cudaGetErrorString(cudaGetLastError()));
  }
}
