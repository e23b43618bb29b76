// Microbenchmark (tooling, not product): what does the 1-CTA/SM TMA -> smem -> STG
// structure of the scatter pass sustain on B200, vs plain copies?
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include "../paper_2312_00720_b200/csrc/cj_device.cuh"
using namespace cj;

__global__ void k_copy_vec(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = __ldcs(a + i);
}
// 3 columns, scalar 4-byte, persistent
__global__ void k_copy3_scalar(const uint32_t* a0, const uint32_t* a1, const uint32_t* a2, uint32_t* b0,
                               uint32_t* b1, uint32_t* b2, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    b0[i] = a0[i]; b1[i] = a1[i]; b2[i] = a2[i];
  }
}
// TMA double-buffered tiles of T rows x 3 columns; LDS + STG.32 (or STG.128)
template <int T, int VEC, int NT>
__global__ void __launch_bounds__(NT, 1) k_tma3(const uint32_t* a0, const uint32_t* a1, const uint32_t* a2,
                                                uint32_t* b0, uint32_t* b1, uint32_t* b2, size_t n) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[2];
  const uint32_t* src[3] = {a0, a1, a2};
  uint32_t* dst[3] = {b0, b1, b2};
  const size_t tiles = n / T;
  const size_t t0 = blockIdx.x * tiles / gridDim.x, t1 = (blockIdx.x + 1) * tiles / gridDim.x;
  auto issue = [&](int b, size_t t) {
    uint8_t* st = smem + (size_t)b * 3 * T * 4;
    dev::mbar_expect_tx(&mbar[b], 3 * T * 4);
    for (int c = 0; c < 3; ++c) dev::tma_load_1d(st + c * T * 4, src[c] + t * T, T * 4, &mbar[b]);
  };
  if (threadIdx.x == 0) {
    dev::mbar_init(&mbar[0], 1); dev::mbar_init(&mbar[1], 1); dev::fence_mbar_init();
    if (t0 < t1) issue(0, t0);
  }
  __syncthreads();
  uint32_t ph[2] = {0, 0};
  int b = 0;
  for (size_t t = t0; t < t1; ++t, b ^= 1) {
    if (threadIdx.x == 0 && t + 1 < t1) { dev::fence_proxy_async(); issue(b ^ 1, t + 1); }
    dev::mbar_wait(&mbar[b], ph[b]); ph[b] ^= 1;
    const uint32_t* st = reinterpret_cast<const uint32_t*>(smem + (size_t)b * 3 * T * 4);
    for (int c = 0; c < 3; ++c) {
      if (VEC == 4) {
        const uint4* s4 = reinterpret_cast<const uint4*>(st + c * T);
        uint4* d4 = reinterpret_cast<uint4*>(dst[c] + t * T);
#pragma unroll 4
        for (int j = threadIdx.x; j < T / 4; j += NT) d4[j] = s4[j];
      } else {
        const uint32_t* s1 = st + c * T;
        uint32_t* d1 = dst[c] + t * T;
#pragma unroll 8
        for (int j = threadIdx.x; j < T; j += NT) d1[j] = s1[j];
      }
    }
    __syncthreads();
  }
}

int main() {
  const size_t n = 1ull << 28;
  uint32_t *a[3], *b[3];
  for (int c = 0; c < 3; ++c) { cudaMalloc(&a[c], n * 4); cudaMalloc(&b[c], n * 4); cudaMemset(a[c], 1, n * 4); }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto time = [&](const char* name, auto f) {
    for (int i = 0; i < 2; ++i) f();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) f();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-40s %8.3f ms  %7.0f GB/s  (%s)\n", name, ms, 3.0 * 2 * n * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  time("copy_vec uint4 x3 arrays", [&] { for (int c = 0; c < 3; ++c) k_copy_vec<<<sms * 8, 512>>>((const uint4*)a[c], (uint4*)b[c], n / 4); });
  time("copy3 scalar persistent 4x512", [&] { k_copy3_scalar<<<sms * 4, 512>>>(a[0], a[1], a[2], b[0], b[1], b[2], n); });
  time("copy3 scalar 1x512", [&] { k_copy3_scalar<<<sms, 512>>>(a[0], a[1], a[2], b[0], b[1], b[2], n); });
#define TMA(T, V, NT) { auto k = k_tma3<T, V, NT>; size_t sm = 2 * 3 * T * 4; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    time("tma3 T=" #T " vec=" #V " nt=" #NT, [&] { k<<<sms, NT, sm>>>(a[0], a[1], a[2], b[0], b[1], b[2], n); }); }
  TMA(4096, 1, 512) TMA(6144, 1, 512) TMA(8192, 1, 512) TMA(8192, 1, 1024) TMA(8192, 4, 512) TMA(4096, 4, 512) TMA(4096, 1, 1024)
  return 0;
}
