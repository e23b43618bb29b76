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
#include <cstring>

#include "cj_device.cuh"
#include "cj_internal.cuh"

namespace cj {
namespace {

using dev::kFlagAgg;
using dev::kFlagIncl;
using dev::kValMask;

constexpr int kHistThreads = 512;

template <class K>
__global__ void __launch_bounds__(kHistThreads)
k_histogram(const K* __restrict__ keys, uint64_t n, int npasses, uint4 shifts_lo, uint4 shifts_hi,
            uint4 masks_lo, uint4 masks_hi, uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t sh[];  // npasses * 256
  const uint32_t sh_arr[8] = {shifts_lo.x, shifts_lo.y, shifts_lo.z, shifts_lo.w,
                              shifts_hi.x, shifts_hi.y, shifts_hi.z, shifts_hi.w};
  const uint32_t mk_arr[8] = {masks_lo.x, masks_lo.y, masks_lo.z, masks_lo.w,
                              masks_hi.x, masks_hi.y, masks_hi.z, masks_hi.w};
  for (int i = threadIdx.x; i < npasses * kRadix; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  auto count = [&](K k) {
#pragma unroll
    for (int p = 0; p < 8; ++p)
      if (p < npasses) atomicAdd(&sh[p * kRadix + (uint32_t)((k >> sh_arr[p]) & mk_arr[p])], 1u);
  };
  constexpr int kVec = 16 / sizeof(K);
  const bool aligned = (reinterpret_cast<uintptr_t>(keys) & 15u) == 0;
  uint64_t start = 0;
  if (aligned) {
    const uint64_t nvec = n / kVec;
    const uint4* kv = reinterpret_cast<const uint4*>(keys);
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
      uint4 q = __ldcs(kv + v);
      K e[kVec];
      memcpy(e, &q, 16);
#pragma unroll
      for (int j = 0; j < kVec; ++j) count(e[j]);
    }
    start = nvec * kVec;
  }
  for (uint64_t i = start + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    count(keys[i]);
  __syncthreads();
  for (int i = threadIdx.x; i < npasses * kRadix; i += blockDim.x)
    if (sh[i]) atomicAdd(&counts[i], sh[i]);
}

// Exclusive digit bases per pass (digit order), 1 block of 256 threads.
__global__ void k_digit_bases(const uint32_t* __restrict__ counts, int npasses,
                              uint64_t* __restrict__ base) {
  __shared__ uint64_t warp_tot[kRadix / 32];
  const int d = threadIdx.x;
  for (int p = 0; p < npasses; ++p) {
    const uint64_t c = counts[p * kRadix + d];
    const uint64_t inc = dev::warp_inclusive_sum(c);
    if ((d & 31) == 31) warp_tot[d >> 5] = inc;
    __syncthreads();
    uint64_t off = 0;
    for (int w = 0; w < (d >> 5); ++w) off += warp_tot[w];
    base[p * kRadix + d] = off + inc - c;
    __syncthreads();
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

template <class T>
__global__ void k_iota(T* out, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (T)i;
}

}  // namespace

void histogram_passes(cj_ctx* ctx, const void* keys, uint64_t n, int key_bytes,
                      const PassPlan& plan, uint32_t* counts_dev, uint64_t* base_dev,
                      std::vector<uint32_t>* counts_host) {
  const int np = plan.npasses;
  CJ_CUDA(cudaMemsetAsync(counts_dev, 0, sizeof(uint32_t) * kRadix * np, ctx->stream));
  uint32_t sh[8] = {}, mk[8] = {};
  for (int p = 0; p < np; ++p) {
    sh[p] = plan.lo[p];
    mk[p] = (1u << (plan.hi[p] - plan.lo[p])) - 1u;
  }
  const uint4 s_lo{sh[0], sh[1], sh[2], sh[3]}, s_hi{sh[4], sh[5], sh[6], sh[7]};
  const uint4 m_lo{mk[0], mk[1], mk[2], mk[3]}, m_hi{mk[4], mk[5], mk[6], mk[7]};
  if (n > 0) {
    const unsigned grid = grid_for(n, kHistThreads * 16, ctx->num_sms * 4);
    const size_t smem = sizeof(uint32_t) * kRadix * np;
    ctx->kbegin("histogram", n * key_bytes);
    if (key_bytes == 4)
      k_histogram<uint32_t><<<grid, kHistThreads, smem, ctx->stream>>>(
          static_cast<const uint32_t*>(keys), n, np, s_lo, s_hi, m_lo, m_hi, counts_dev);
    else
      k_histogram<uint64_t><<<grid, kHistThreads, smem, ctx->stream>>>(
          static_cast<const uint64_t*>(keys), n, np, s_lo, s_hi, m_lo, m_hi, counts_dev);
    ctx->kend();
  }
  ctx->kbegin("digit_bases", 12ull * kRadix * np);
  k_digit_bases<<<1, kRadix, 0, ctx->stream>>>(counts_dev, np, base_dev);
  ctx->kend();
  CJ_CUDA(cudaGetLastError());
  if (counts_host) {
    counts_host->resize((size_t)kRadix * np);
    CJ_CUDA(cudaMemcpyAsync(ctx->host_pinned, counts_dev, sizeof(uint32_t) * kRadix * np,
                            cudaMemcpyDeviceToHost, ctx->stream));
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(counts_host->data(), ctx->host_pinned, sizeof(uint32_t) * kRadix * np);
  }
}

void scatter_pass(cj_ctx* ctx, const void* keys_in, void* keys_out, uint64_t n, int key_bytes,
                  uint32_t lo, uint32_t hi, const uint64_t* base_dev, const ValCols& vals) {
  if (n == 0) return;
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
  uint64_t row = key_bytes;
  for (int c = 0; c < vals.n; ++c) row += vals.bytes[c] - ((vals.gen_ids && c == 0) ? 4 : 0);
  uint64_t wrow = key_bytes;
  for (int c = 0; c < vals.n; ++c) wrow += vals.bytes[c];
  ctx->kbegin("scatter_pass", n * (row + wrow));
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

void lsd_partition(cj_ctx* ctx, const void* keys, void* keys_out, uint64_t n, int key_bytes,
                   const PassPlan& plan, const ValCols& vals, std::vector<uint32_t>* counts_out) {
  std::vector<uint32_t> counts;
  Scratch cnt(ctx, sizeof(uint32_t) * kRadix * CJ_MAX_PASSES);
  Scratch base(ctx, sizeof(uint64_t) * kRadix * CJ_MAX_PASSES);
  histogram_passes(ctx, keys, n, key_bytes, plan, cnt.as<uint32_t>(), base.as<uint64_t>(),
                   &counts);
  if (counts_out) *counts_out = counts;
  std::vector<int> live;
  for (int p = 0; p < plan.npasses; ++p) {
    if (plan.hi[p] == plan.lo[p]) continue;
    bool constant = n == 0;
    for (int d = 0; d < kRadix && !constant; ++d)
      if (counts[(size_t)p * kRadix + d] == n) constant = true;
    if (!constant) live.push_back(p);
  }
  if (live.empty()) {
    copy_columns(ctx, keys, keys_out, n, key_bytes, vals);
    return;
  }
  // ping-pong scratch; the first target is chosen so the last pass lands in
  // the caller's buffers (primitives.cpp:236-255)
  const int nv = vals.n;
  Scratch sk(ctx, live.size() > 1 ? n * key_bytes : 0);
  std::vector<Scratch*> sv;
  uint64_t vbytes_total = 0;
  auto col_span = [&](int c) { return (n * vals.bytes[c] + 255) & ~uint64_t(255); };
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
  const void* cur_k = keys;
  ValCols cur = vals;
  bool to_out = (live.size() % 2) == 1;
  for (size_t li = 0; li < live.size(); ++li) {
    const int p = live[li];
    ValCols step = cur;
    void* tk = to_out ? keys_out : sk.p;
    for (int c = 0; c < nv; ++c) step.out[c] = to_out ? vals.out[c] : scratch_cols[c];
    step.gen_ids = li == 0 ? vals.gen_ids : 0;
    scatter_pass(ctx, cur_k, tk, n, key_bytes, plan.lo[p], plan.hi[p],
                 base.as<uint64_t>() + (size_t)p * kRadix, step);
    cur_k = tk;
    for (int c = 0; c < nv; ++c) cur.in[c] = step.out[c];
    cur.gen_ids = 0;
    to_out = !to_out;
  }
}

void partition_offsets(cj_ctx* ctx, const void* keys_sorted, uint64_t n, int key_bytes,
                       uint32_t bits, uint64_t* offsets_dev) {
  const uint64_t fanout = 1ull << bits;
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
