// Workload generation bit-identical to the reference's workloads::gen_pk_fk
// (workloads.cpp:89-133) and its counter RNG (rng.hpp:8-37).
//
// The Fisher-Yates permutation (workloads.cpp:26-34) and the Zipf CDF
// (workloads.cpp:60-70, a sequential double accumulation) are sequential by
// definition and run on the host; every per-draw quantity (uniform / Zipf
// foreign keys, key displacement, payload streams) is a pure function of
// (stream, index) and is generated on the device.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "cj_device.cuh"
#include "cj_internal.cuh"

namespace cj {
namespace {

constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;

using dev::mix64;
__host__ __device__ __forceinline__ uint64_t stream_of(uint64_t seed, uint64_t tag) {
  return mix64(seed ^ mix64(tag + kGold));
}
__host__ __device__ __forceinline__ uint64_t rng_at(uint64_t seed, uint64_t i) {
  return mix64(seed + (i + 1) * kGold);
}
__host__ __device__ __forceinline__ double rng_u01(uint64_t seed, uint64_t i) {
  return static_cast<double>(rng_at(seed, i) >> 11) * 0x1.0p-53;
}
__host__ __forceinline__ uint64_t rng_below(uint64_t seed, uint64_t i, uint64_t bound) {
  return static_cast<uint64_t>((static_cast<unsigned __int128>(rng_at(seed, i)) * bound) >> 64);
}

std::vector<uint32_t> permutation(uint64_t n, uint64_t seed) {
  std::vector<uint32_t> p(n);
  for (uint64_t i = 0; i < n; ++i) p[i] = static_cast<uint32_t>(i);
  for (uint64_t i = n; i > 1; --i) {
    const uint64_t j = rng_below(seed, i, i);
    std::swap(p[i - 1], p[j]);
  }
  return p;
}

template <class K>
__global__ void k_rkeys(const uint32_t* __restrict__ perm, uint64_t n, uint64_t keep, K* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v = perm[i];
    if (v >= keep) v += n;  // workloads.cpp:113-120
    out[i] = (K)v;
  }
}

template <class K>
__global__ void k_skeys_uniform(uint64_t seed, uint64_t n_r, uint64_t n_s, K* out) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_s;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const double u = rng_u01(seed, j);
    uint64_t r = static_cast<uint64_t>(__dmul_rn(u, static_cast<double>(n_r)));
    if (r >= n_r) r = n_r - 1;
    out[j] = (K)r;
  }
}

template <class K>
__global__ void k_skeys_zipf(uint64_t seed, const double* __restrict__ cdf,
                             const uint32_t* __restrict__ rank_to_key, uint64_t n_r, uint64_t n_s,
                             K* out) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_s;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const double u = rng_u01(seed, j);
    uint64_t lo = 0, hi = n_r;  // upper_bound: first cdf > u
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (cdf[mid] > u) hi = mid; else lo = mid + 1;
    }
    const uint64_t rank = lo == n_r ? n_r - 1 : lo;
    out[j] = (K)rank_to_key[rank];
  }
}

template <class T>
__global__ void k_payload(uint64_t seed, uint64_t n, T* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (T)rng_at(seed, i);
}

// workloads.cpp:141-145: fact FK i = stream.below(i, dim_rows)
template <class K>
__global__ void k_star_fk(uint64_t seed, uint64_t n, uint64_t bound, K* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (K)__umul64hi(rng_at(seed, i), bound);
}

__global__ void k_iota32(uint32_t* out, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)i;
}

template <class K>
__global__ void k_perm_keys(const uint32_t* __restrict__ perm, uint64_t n, K* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (K)perm[i];
}

// Bijection of [0, 2^m): rounds of (odd multiply, add, xor-shift), all mod 2^m.
__device__ __forceinline__ uint64_t scramble(uint64_t x, uint32_t m, uint64_t seed) {
  const uint64_t mask = m >= 64 ? ~0ull : ((1ull << m) - 1);
  const uint32_t sh = m > 1 ? (m + 1) / 2 : 1;
  uint64_t k = seed;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    k = mix64(k + kGold);
    x = (x * (k | 1ull) + (k >> 7)) & mask;
    x ^= x >> sh;
  }
  return x;
}

__global__ void k_shard(uint64_t r_total, uint32_t m, uint64_t s_total, uint64_t r_lo, uint64_t r_n,
                        uint64_t s_lo, uint64_t s_n, uint64_t seed, uint32_t* __restrict__ rk,
                        uint32_t* __restrict__ sk) {
  const uint64_t pseed = stream_of(seed, 0x52100000ull), fseed = stream_of(seed, 0x53100000ull);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < r_n; i += stride)
    rk[i] = (uint32_t)scramble(r_lo + i, m, pseed);
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < s_n; j += stride)
    sk[j] = (uint32_t)__umul64hi(rng_at(fseed, s_lo + j), r_total);
}

template <class T>
__global__ void k_payload_at(uint64_t seed, uint64_t first, uint64_t n, T* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (T)rng_at(seed, first + i);
}

}  // namespace

void gen_shard(cj_ctx* ctx, uint64_t r_total, uint64_t s_total, uint32_t rank, uint32_t ranks,
               uint32_t r_pay, uint32_t s_pay, uint64_t seed, void* r_key, void* const* r_pays,
               void* s_key, void* const* s_pays) {
  if (ranks == 0 || rank >= ranks) fail(CJ_ERR_SPEC_INVALID, "rank out of range");
  if (r_total == 0 || (r_total & (r_total - 1)) || r_total % ranks || s_total % ranks)
    fail(CJ_ERR_SPEC_INVALID, "shard generator needs |R| a power of two and |R|,|S| divisible by ranks");
  if (r_total > (1ull << 32)) fail(CJ_ERR_UNSUPPORTED, "shard generator keys are 4 bytes");
  uint32_t m = 0;
  while ((1ull << m) < r_total) ++m;
  const uint64_t rn = r_total / ranks, sn = s_total / ranks, r_lo = rn * rank, s_lo = sn * rank;
  const unsigned grid = ctx->num_sms * 8;
  ctx->kbegin("gen_shard", 4 * (rn + sn));
  k_shard<<<grid, 256, 0, ctx->stream>>>(r_total, m, s_total, r_lo, rn, s_lo, sn, seed,
                                         static_cast<uint32_t*>(r_key), static_cast<uint32_t*>(s_key));
  ctx->kend();
  for (uint32_t c = 0; c < r_pay; ++c) {
    ctx->kbegin("gen_payload", rn * 4);
    k_payload_at<uint32_t><<<grid, 256, 0, ctx->stream>>>(stream_of(seed, 0x7000ull + c), r_lo, rn,
                                                          static_cast<uint32_t*>(r_pays[c]));
    ctx->kend();
  }
  for (uint32_t c = 0; c < s_pay; ++c) {
    ctx->kbegin("gen_payload", sn * 4);
    k_payload_at<uint32_t><<<grid, 256, 0, ctx->stream>>>(stream_of(seed, 0x8000ull + c), s_lo, sn,
                                                          static_cast<uint32_t*>(s_pays[c]));
    ctx->kend();
  }
  CJ_CUDA(cudaGetLastError());
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
}

void gen_pk_fk(cj_ctx* ctx, uint64_t r_rows, uint64_t s_rows, uint32_t r_pay, uint32_t s_pay,
               uint32_t key_bytes, uint32_t pay_bytes, double match_ratio, double zipf,
               uint64_t seed, void* r_key, void* const* r_pays, void* s_key,
               void* const* s_pays) {
  if (match_ratio < 0.0 || match_ratio > 1.0) fail(CJ_ERR_SPEC_INVALID, "match ratio must lie in [0, 1]");
  if (zipf < 0.0) fail(CJ_ERR_SPEC_INVALID, "zipf factor must be >= 0");
  if (r_rows > 0x7fffffffull || s_rows > 0x7fffffffull)
    fail(CJ_ERR_SPEC_INVALID, "row count exceeds the 2^31-1 cap");
  if ((key_bytes != 4 && key_bytes != 8) || (pay_bytes != 4 && pay_bytes != 8))
    fail(CJ_ERR_KIND, "key/payload widths must be 4 or 8 bytes");
  const unsigned grid = ctx->num_sms * 8;
  // R keys: shuffled dense domain [0, |R|), non-kept keys displaced by |R|
  const std::vector<uint32_t> perm = permutation(r_rows, stream_of(seed, 0x52000001ull));
  const uint64_t keep = static_cast<uint64_t>(std::llround(match_ratio * static_cast<double>(r_rows)));
  {
    Scratch dperm(ctx, r_rows * 4);
    if (r_rows) {
      CJ_CUDA(cudaMemcpyAsync(dperm.p, perm.data(), r_rows * 4, cudaMemcpyHostToDevice, ctx->stream));
      ctx->kbegin("gen_rkeys", r_rows * (4 + key_bytes));
      if (key_bytes == 4)
        k_rkeys<uint32_t><<<grid, 256, 0, ctx->stream>>>(dperm.as<uint32_t>(), r_rows, keep,
                                                         static_cast<uint32_t*>(r_key));
      else
        k_rkeys<uint64_t><<<grid, 256, 0, ctx->stream>>>(dperm.as<uint32_t>(), r_rows, keep,
                                                         static_cast<uint64_t*>(r_key));
      ctx->kend();
    }
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));  // perm host buffer lifetime
  }
  // S keys (workloads.cpp:55-81, 98-111)
  const uint64_t zseed = stream_of(seed, 0x5a1bf001ull);
  if (r_rows > 0 && s_rows > 0) {
    if (zipf == 0.0) {
      ctx->kbegin("gen_skeys", s_rows * key_bytes);
      if (key_bytes == 4)
        k_skeys_uniform<uint32_t><<<grid, 256, 0, ctx->stream>>>(zseed, r_rows, s_rows,
                                                                 static_cast<uint32_t*>(s_key));
      else
        k_skeys_uniform<uint64_t><<<grid, 256, 0, ctx->stream>>>(zseed, r_rows, s_rows,
                                                                 static_cast<uint64_t*>(s_key));
      ctx->kend();
    } else {
      std::vector<double> cdf(r_rows);
      double acc = 0.0;
      for (uint64_t k = 0; k < r_rows; ++k) {
        acc += std::pow(static_cast<double>(k + 1), -zipf);
        cdf[k] = acc;
      }
      const double norm = 1.0 / acc;
      for (auto& v : cdf) v *= norm;
      cdf.back() = 1.0;
      const std::vector<uint32_t> r2k = permutation(r_rows, stream_of(seed, 0x53000001ull));
      Scratch dcdf(ctx, r_rows * 8), dr2k(ctx, r_rows * 4);
      CJ_CUDA(cudaMemcpyAsync(dcdf.p, cdf.data(), r_rows * 8, cudaMemcpyHostToDevice, ctx->stream));
      CJ_CUDA(cudaMemcpyAsync(dr2k.p, r2k.data(), r_rows * 4, cudaMemcpyHostToDevice, ctx->stream));
      ctx->kbegin("gen_skeys_zipf", s_rows * key_bytes);
      if (key_bytes == 4)
        k_skeys_zipf<uint32_t><<<grid, 256, 0, ctx->stream>>>(zseed, dcdf.as<double>(),
                                                              dr2k.as<uint32_t>(), r_rows, s_rows,
                                                              static_cast<uint32_t*>(s_key));
      else
        k_skeys_zipf<uint64_t><<<grid, 256, 0, ctx->stream>>>(zseed, dcdf.as<double>(),
                                                              dr2k.as<uint32_t>(), r_rows, s_rows,
                                                              static_cast<uint64_t*>(s_key));
      ctx->kend();
      CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  } else if (s_rows > 0) {
    CJ_CUDA(cudaMemsetAsync(s_key, 0, s_rows * key_bytes, ctx->stream));
  }
  // payload streams 0x7000+c (R) / 0x8000+c (S), truncated to the width
  auto pay = [&](void* dst, uint64_t n, uint64_t tag) {
    if (n == 0) return;
    const uint64_t sd = stream_of(seed, tag);
    ctx->kbegin("gen_payload", n * pay_bytes);
    if (pay_bytes == 4)
      k_payload<uint32_t><<<grid, 256, 0, ctx->stream>>>(sd, n, static_cast<uint32_t*>(dst));
    else
      k_payload<uint64_t><<<grid, 256, 0, ctx->stream>>>(sd, n, static_cast<uint64_t*>(dst));
    ctx->kend();
  };
  for (uint32_t c = 0; c < r_pay; ++c) pay(r_pays[c], r_rows, 0x7000ull + c);
  for (uint32_t c = 0; c < s_pay; ++c) pay(s_pays[c], s_rows, 0x8000ull + c);
  CJ_CUDA(cudaGetLastError());
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
}

// workloads::gen_star (workloads.cpp:135-160): fact key = physical tuple ids
// (u32 iota), FK_d = stream(0x46b00000 + d).below(i, dim_rows); dimension d =
// Fisher-Yates permutation of [0, dim_rows) (stream 0xd1a00000 + d, host) as
// keys + one payload column (stream 0xd1a08000 + d).
void gen_star(cj_ctx* ctx, uint64_t fact_rows, uint32_t dims, uint64_t dim_rows, uint64_t seed,
              uint32_t key_bytes, uint32_t pay_bytes, void* fact_ids, void* const* fks,
              void* const* dim_keys, void* const* dim_pays) {
  if (dims < 1) fail(CJ_ERR_SPEC_INVALID, "star schema needs at least one dimension");
  if (dim_rows == 0) fail(CJ_ERR_SPEC_INVALID, "dimension tables cannot be empty");
  if (fact_rows > 0x7fffffffull || dim_rows > 0x7fffffffull)
    fail(CJ_ERR_SPEC_INVALID, "row count exceeds the 2^31-1 cap");
  if ((key_bytes != 4 && key_bytes != 8) || (pay_bytes != 4 && pay_bytes != 8))
    fail(CJ_ERR_KIND, "key/payload widths must be 4 or 8 bytes");
  const unsigned grid = ctx->num_sms * 8;
  if (fact_rows) {
    ctx->kbegin("gen_star_ids", fact_rows * 4);
    k_iota32<<<grid, 256, 0, ctx->stream>>>(static_cast<uint32_t*>(fact_ids), fact_rows);
    ctx->kend();
  }
  for (uint32_t d = 0; d < dims; ++d) {
    if (fact_rows) {
      const uint64_t fs = stream_of(seed, 0x46b00000ull + d);
      ctx->kbegin("gen_star_fk", fact_rows * key_bytes);
      if (key_bytes == 4)
        k_star_fk<uint32_t><<<grid, 256, 0, ctx->stream>>>(fs, fact_rows, dim_rows,
                                                           static_cast<uint32_t*>(fks[d]));
      else
        k_star_fk<uint64_t><<<grid, 256, 0, ctx->stream>>>(fs, fact_rows, dim_rows,
                                                           static_cast<uint64_t*>(fks[d]));
      ctx->kend();
    }
    const std::vector<uint32_t> perm = permutation(dim_rows, stream_of(seed, 0xd1a00000ull + d));
    {
      Scratch dperm(ctx, dim_rows * 4);
      CJ_CUDA(cudaMemcpyAsync(dperm.p, perm.data(), dim_rows * 4, cudaMemcpyHostToDevice, ctx->stream));
      ctx->kbegin("gen_star_dim", dim_rows * (4 + key_bytes));
      if (key_bytes == 4)
        k_perm_keys<uint32_t><<<grid, 256, 0, ctx->stream>>>(dperm.as<uint32_t>(), dim_rows,
                                                             static_cast<uint32_t*>(dim_keys[d]));
      else
        k_perm_keys<uint64_t><<<grid, 256, 0, ctx->stream>>>(dperm.as<uint32_t>(), dim_rows,
                                                             static_cast<uint64_t*>(dim_keys[d]));
      ctx->kend();
      CJ_CUDA(cudaStreamSynchronize(ctx->stream));  // perm host buffer lifetime
    }
    const uint64_t ps = stream_of(seed, 0xd1a08000ull + d);
    ctx->kbegin("gen_payload", dim_rows * pay_bytes);
    if (pay_bytes == 4)
      k_payload<uint32_t><<<grid, 256, 0, ctx->stream>>>(ps, dim_rows, static_cast<uint32_t*>(dim_pays[d]));
    else
      k_payload<uint64_t><<<grid, 256, 0, ctx->stream>>>(ps, dim_rows, static_cast<uint64_t*>(dim_pays[d]));
    ctx->kend();
  }
  CJ_CUDA(cudaGetLastError());
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace cj
