// Non-partitioned hash join (K7): one global open-addressing table over the
// build relation in HBM, probed in probe order.  The reference has no NPHJ
// (the paper uses cuDF's as a baseline); parity is by the
// canonical row multiset, and the emission order is defined here as (probe
// position, ascending build row).
//
// Unique build keys (PK): slots are rows of 32-bit words [row+1][key (1|2
// words)][payload words...]. GFTR stores the build payload columns inside the
// slot (the hashed build relation IS the transformed relation), so
// materialising a match reads the key's own sector; GFUR stores only (row,
// key) and gathers payloads later.  Non-unique builds: the build is sorted
// (stable, with row ids) and the table holds one slot per distinct key.
#include <cuda_runtime.h>

#include <algorithm>

#include "cj_device.cuh"
#include "cj_internal.cuh"

namespace cj {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kTile = 2048;

struct NphjArgs {
  const void* rkeys;
  uint64_t nr;
  const void* skeys;
  uint64_t ns;
  uint32_t* table;
  uint32_t log2cap, slot_words, key_words;
  int nr_cols;
  uint32_t r_word_off[CJ_MAX_COLS];
  const void* r_src[CJ_MAX_COLS];
  void* r_dst[CJ_MAX_COLS];
  uint32_t r_bytes[CJ_MAX_COLS];
  int ns_cols;
  const void* s_src[CJ_MAX_COLS];
  void* s_dst[CJ_MAX_COLS];
  uint32_t s_bytes[CJ_MAX_COLS];
  void* key_out;
  uint32_t* ids_r;
  uint32_t* ids_s;
  uint64_t tiles;
  uint64_t* status;
  uint64_t epoch;
  uint32_t* ticket;
  uint32_t* err;
  uint64_t capacity;
  int write;
  uint64_t* total_out;
  int unique;                // build keys unique (Relation::key_unique): one match per probe
  // non-unique builds: the build keys sorted (stable) with their row ids; the
  // table holds one slot per distinct key [run start + 1][key], a probe finds
  // its run's end by galloping over the sorted keys
  const void* sorted_keys;
  const uint32_t* sorted_ids;
};

template <class K>
__device__ __forceinline__ uint64_t nslot(K k, uint32_t log2cap) {
  return ((uint64_t)k * 0x9E3779B97F4A7C15ull) >> (64 - log2cap);
}

template <class K>
__device__ __forceinline__ K slot_key(const uint32_t* s) {
  if constexpr (sizeof(K) == 4) {
    return s[1];
  } else {
    return (uint64_t)s[1] | ((uint64_t)s[2] << 32);
  }
}

template <class K>
__global__ void __launch_bounds__(kThreads) k_nphj_build(const __grid_constant__ NphjArgs a) {
  const K* __restrict__ rk = static_cast<const K*>(a.rkeys);
  const uint64_t mask = (1ull << a.log2cap) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.nr;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const K k = rk[i];
    uint64_t h = nslot(k, a.log2cap);
    while (true) {
      uint32_t* s = a.table + h * a.slot_words;
      if (atomicCAS(s, 0u, (uint32_t)(i + 1)) == 0u) {
        if (a.slot_words == 4 && sizeof(K) == 4) {
          // one 16-byte store of the whole slot (word 0 rewritten with its own value)
          uint32_t w2 = 0, w3 = 0;
          if (a.nr_cols == 1 && a.r_bytes[0] == 8) {
            const uint64_t v = static_cast<const uint64_t*>(a.r_src[0])[i];
            w2 = (uint32_t)v;
            w3 = (uint32_t)(v >> 32);
          } else {
            if (a.nr_cols > 0) w2 = static_cast<const uint32_t*>(a.r_src[0])[i];
            if (a.nr_cols > 1) w3 = static_cast<const uint32_t*>(a.r_src[1])[i];
          }
          *reinterpret_cast<uint4*>(s) = make_uint4((uint32_t)(i + 1), (uint32_t)k, w2, w3);
        } else {
          s[1] = (uint32_t)k;
          if constexpr (sizeof(K) == 8) s[2] = (uint32_t)((uint64_t)k >> 32);
          for (int c = 0; c < a.nr_cols; ++c) {
            uint32_t* d = s + a.r_word_off[c];
            if (a.r_bytes[c] == 4) {
              d[0] = static_cast<const uint32_t*>(a.r_src[c])[i];
            } else {
              const uint64_t v = static_cast<const uint64_t*>(a.r_src[c])[i];
              d[0] = (uint32_t)v;
              d[1] = (uint32_t)(v >> 32);
            }
          }
        }
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

// Unique build keys (Relation::key_unique, as the reference's PK-FK merge
// trusts it, merge_match.cpp:65-68): a probe stops at its first match; a
// 4-word slot (4-byte key + <= 8 payload bytes) is read with one 16-byte load
// and its payload words are kept in shared memory for the write, so the table
// is touched once per probe step.
template <class K, bool VEC>
__global__ void __launch_bounds__(kThreads) k_nphj_probe_u(const __grid_constant__ NphjArgs a) {
  __shared__ uint32_t s_hit[kTile];      // 0: no match, else build row + 1
  __shared__ uint2 s_pay[VEC ? kTile : 1];  // slot words 2, 3 of the match
  __shared__ uint64_t s_t, s_base;
  __shared__ uint64_t s_wcount[kWarps], s_wbase[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const K* __restrict__ sk = static_cast<const K*>(a.skeys);
  const uint64_t mask = (1ull << a.log2cap) - 1;
  while (true) {
    if (tid == 0) s_t = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const uint64_t t = s_t;
    if (t >= a.tiles) break;
    const uint64_t j0 = t * kTile;
    const uint32_t nq = (uint32_t)dev::umin64(kTile, a.ns - j0);
    const uint32_t rounds = (nq + 31) / 32;
    const uint32_t r0 = rounds * warp / kWarps, r1 = rounds * (warp + 1) / kWarps;
    uint64_t wc = 0;
    for (uint32_t rr = r0; rr < r1; ++rr) {
      const uint32_t jl = rr * 32 + lane;
      uint32_t hit = 0;
      if (jl < nq) {
        const K k = __ldcs(sk + j0 + jl);
        uint64_t h = nslot(k, a.log2cap);
        while (true) {
          const uint32_t* s = a.table + h * a.slot_words;
          if (VEC) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(s));
            if (w.x == 0) break;
            if (w.y == (uint32_t)k) {
              hit = w.x;
              s_pay[jl] = make_uint2(w.z, w.w);
              break;
            }
          } else {
            const uint32_t row1 = s[0];
            if (row1 == 0) break;
            if (slot_key<K>(s) == k) {
              hit = row1;
              break;
            }
          }
          h = (h + 1) & mask;
        }
        s_hit[jl] = hit;
      }
      wc += __popc(__ballot_sync(0xffffffffu, hit != 0));
    }
    if (lane == 0) s_wcount[warp] = wc;
    __syncthreads();
    if (warp == 0) {
      const uint64_t v = lane < kWarps ? s_wcount[lane] : 0;
      const uint64_t inc = dev::warp_inclusive_sum(v);
      if (lane < kWarps) s_wbase[lane] = inc - v;
      const uint64_t tot = __shfl_sync(0xffffffffu, inc, kWarps - 1);
      const uint64_t base = dev::warp_lookback(a.status, t, tot, a.epoch, a.err);
      if (lane == 0) {
        s_base = base;
        if (t == a.tiles - 1) *a.total_out = base + tot;
        if (a.write && base + tot > a.capacity) atomicOr(a.err, kErrOverflow);
      }
    }
    __syncthreads();
    if (a.write) {
      uint64_t o = s_base + s_wbase[warp];
      for (uint32_t rr = r0; rr < r1; ++rr) {
        const uint32_t jl = rr * 32 + lane;
        const uint32_t hit = jl < nq ? s_hit[jl] : 0;
        const uint32_t bal = __ballot_sync(0xffffffffu, hit != 0);
        const uint64_t oo = o + __popc(bal & dev::lanemask_lt());
        o += __popc(bal);
        if (!hit || oo >= a.capacity) continue;
        const uint64_t j = j0 + jl;
        const uint32_t i = hit - 1;
        if (a.key_out) static_cast<K*>(a.key_out)[oo] = sk[j];
        if (a.ids_r) a.ids_r[oo] = i;
        if (a.ids_s) a.ids_s[oo] = (uint32_t)j;
        if (VEC) {
          const uint2 pw = s_pay[jl];
          if (a.nr_cols == 1 && a.r_bytes[0] == 8) {
            static_cast<uint64_t*>(a.r_dst[0])[oo] = (uint64_t)pw.x | ((uint64_t)pw.y << 32);
          } else {
            if (a.nr_cols > 0) static_cast<uint32_t*>(a.r_dst[0])[oo] = pw.x;
            if (a.nr_cols > 1) static_cast<uint32_t*>(a.r_dst[1])[oo] = pw.y;
          }
        } else {
          uint64_t h = nslot(sk[j], a.log2cap);  // rare layouts: find the slot again
          const uint32_t* s;
          while (true) {
            s = a.table + h * a.slot_words;
            if (s[0] == hit) break;
            h = (h + 1) & mask;
          }
          for (int c = 0; c < a.nr_cols; ++c) {
            const uint32_t* w = s + a.r_word_off[c];
            if (a.r_bytes[c] == 4)
              static_cast<uint32_t*>(a.r_dst[c])[oo] = w[0];
            else
              static_cast<uint64_t*>(a.r_dst[c])[oo] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
          }
        }
        for (int c = 0; c < a.ns_cols; ++c) {
          if (a.s_bytes[c] == 4)
            static_cast<uint32_t*>(a.s_dst[c])[oo] = static_cast<const uint32_t*>(a.s_src[c])[j];
          else
            static_cast<uint64_t*>(a.s_dst[c])[oo] = static_cast<const uint64_t*>(a.s_src[c])[j];
        }
      }
    }
    __syncthreads();
  }
}

// Non-unique builds: one slot per distinct key of the sorted build (its run
// start), so equal keys never form a probe chain (emission order unchanged:
// probe position, then ascending build row).
template <class K>
__global__ void __launch_bounds__(kThreads) k_nphj_build_runs(const __grid_constant__ NphjArgs a) {
  const K* __restrict__ sk = static_cast<const K*>(a.sorted_keys);
  const uint64_t mask = (1ull << a.log2cap) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.nr;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const K k = sk[i];
    if (i > 0 && sk[i - 1] == k) continue;
    uint64_t h = nslot(k, a.log2cap);
    while (true) {
      uint32_t* sl = a.table + h * a.slot_words;
      if (atomicCAS(sl, 0u, (uint32_t)(i + 1)) == 0u) {
        sl[1] = (uint32_t)k;
        if constexpr (sizeof(K) == 8) sl[2] = (uint32_t)((uint64_t)k >> 32);
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

// First index >= lo whose sorted key differs from k (galloping, then binary).
template <class K>
__device__ __forceinline__ uint64_t run_end(const K* __restrict__ sk, uint64_t n, uint64_t lo, K k) {
  uint64_t step = 1, prev = lo;
  uint64_t hi = lo + 1;
  while (hi < n && sk[hi] == k) {
    prev = hi;
    step <<= 1;
    hi = lo + step;
  }
  if (hi > n) hi = n;
  uint64_t l = prev + 1;  // sk[prev] == k; answer in [l, hi]
  while (l < hi) {
    const uint64_t mid = (l + hi) >> 1;
    if (sk[mid] == k) l = mid + 1; else hi = mid;
  }
  return l;
}

template <class K>
__global__ void __launch_bounds__(kThreads) k_nphj_probe_runs(const __grid_constant__ NphjArgs a) {
  __shared__ uint32_t s_m[kTile];
  __shared__ uint64_t s_first[kTile];
  __shared__ uint64_t s_t, s_base;
  __shared__ uint64_t s_wcount[kWarps], s_wbase[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const K* __restrict__ sk = static_cast<const K*>(a.skeys);
  const K* __restrict__ bk = static_cast<const K*>(a.sorted_keys);
  const uint64_t mask = (1ull << a.log2cap) - 1;
  while (true) {
    if (tid == 0) s_t = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const uint64_t t = s_t;
    if (t >= a.tiles) break;
    const uint64_t j0 = t * kTile;
    const uint32_t nq = (uint32_t)dev::umin64(kTile, a.ns - j0);
    const uint32_t rounds = (nq + 31) / 32;
    const uint32_t r0 = rounds * warp / kWarps, r1 = rounds * (warp + 1) / kWarps;
    uint64_t wc = 0;
    for (uint32_t rr = r0; rr < r1; ++rr) {
      const uint32_t jl = rr * 32 + lane;
      if (jl < nq) {
        const K k = sk[j0 + jl];
        uint64_t h = nslot(k, a.log2cap);
        uint32_t m = 0;
        uint64_t first = 0;
        while (true) {
          const uint32_t* sl = a.table + h * a.slot_words;
          const uint32_t row1 = sl[0];
          if (row1 == 0) break;
          if (slot_key<K>(sl) == k) {
            first = row1 - 1;
            m = (uint32_t)(run_end<K>(bk, a.nr, first, k) - first);
            break;
          }
          h = (h + 1) & mask;
        }
        s_m[jl] = m;
        s_first[jl] = first;
        wc += m;
      }
    }
    wc = dev::warp_sum(wc);
    if (lane == 0) s_wcount[warp] = wc;
    __syncthreads();
    if (warp == 0) {
      const uint64_t v = lane < kWarps ? s_wcount[lane] : 0;
      const uint64_t inc = dev::warp_inclusive_sum(v);
      if (lane < kWarps) s_wbase[lane] = inc - v;
      const uint64_t tot = __shfl_sync(0xffffffffu, inc, kWarps - 1);
      const uint64_t base = dev::warp_lookback(a.status, t, tot, a.epoch, a.err);
      if (lane == 0) {
        s_base = base;
        if (t == a.tiles - 1) *a.total_out = base + tot;
        if (a.write && base + tot > a.capacity) atomicOr(a.err, kErrOverflow);
      }
    }
    __syncthreads();
    if (a.write) {
      uint64_t o = s_base + s_wbase[warp];
      for (uint32_t rr = r0; rr < r1; ++rr) {
        const uint32_t jl = rr * 32 + lane;
        const uint32_t m = jl < nq ? s_m[jl] : 0;
        const uint32_t inc = dev::warp_inclusive_sum(m);
        const uint64_t obase = o + inc - m;
        const uint64_t j = j0 + jl;
        // the run holds the matches in ascending build row (stable sort)
        for (uint32_t q = 0; q < m; ++q) {
          const uint64_t oo = obase + q;
          if (oo >= a.capacity) break;
          const uint32_t i = a.sorted_ids[s_first[jl] + q];
          if (a.key_out) static_cast<K*>(a.key_out)[oo] = sk[j];
          if (a.ids_r) a.ids_r[oo] = i;
          if (a.ids_s) a.ids_s[oo] = (uint32_t)j;
          for (int c = 0; c < a.nr_cols; ++c) {
            if (a.r_bytes[c] == 4)
              static_cast<uint32_t*>(a.r_dst[c])[oo] = static_cast<const uint32_t*>(a.r_src[c])[i];
            else
              static_cast<uint64_t*>(a.r_dst[c])[oo] = static_cast<const uint64_t*>(a.r_src[c])[i];
          }
          for (int c = 0; c < a.ns_cols; ++c) {
            if (a.s_bytes[c] == 4)
              static_cast<uint32_t*>(a.s_dst[c])[oo] = static_cast<const uint32_t*>(a.s_src[c])[j];
            else
              static_cast<uint64_t*>(a.s_dst[c])[oo] = static_cast<const uint64_t*>(a.s_src[c])[j];
          }
        }
        o += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
  }
}

// Non-unique builds: stable sort of the build keys with their row ids, one
// table slot per distinct key, probes read whole runs (no equal-key chains:
// a key repeated d times used to cost d^2 probe steps).
template <class K>
uint64_t run_sorted(cj_ctx* ctx, NphjArgs a) {
  const uint64_t n = a.nr;
  Scratch skeys(ctx, n * sizeof(K) + kPad), sids(ctx, n * 4 + kPad);
  ValCols v;
  v.n = 1;
  v.gen_ids = 1;
  v.bytes[0] = 4;
  v.out[0] = sids.p;
  lsd_any(ctx, a.rkeys, skeys.p, n, (int)sizeof(K), sort_plan(ctx, a.rkeys, n, sizeof(K), v), v,
          nullptr);
  a.sorted_keys = skeys.p;
  a.sorted_ids = sids.as<uint32_t>();
  a.slot_words = 1 + a.key_words;
  const uint64_t cap = 1ull << a.log2cap;
  Scratch table(ctx, cap * a.slot_words * 4);
  CJ_CUDA(cudaMemsetAsync(table.p, 0, cap * a.slot_words * 4, ctx->stream));
  a.table = table.as<uint32_t>();
  Scratch tot(ctx, 8);
  CJ_CUDA(cudaMemsetAsync(tot.p, 0, 8, ctx->stream));
  a.total_out = tot.as<uint64_t>();
  a.err = ctx->err_word;
  ctx->kbegin("nphj_build", n * (uint64_t)(2 * sizeof(K) + 4ull * a.slot_words));
  k_nphj_build_runs<K><<<grid_for(n, kThreads * 4, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(a);
  ctx->kend();
  a.tiles = (a.ns + kTile - 1) / kTile;
  if (a.tiles > 0) {
    a.status = ctx->status_buffer(a.tiles);
    a.epoch = ctx->next_epoch();
    a.ticket = ctx->ticket(3);
    int per_sm = 0;
    CJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_nphj_probe_runs<K>, kThreads, 0));
    const uint64_t grid = std::min<uint64_t>((uint64_t)ctx->num_sms * std::max(per_sm, 1), a.tiles);
    ctx->kbegin(a.write ? "nphj_probe" : "nphj_count", 0);
    k_nphj_probe_runs<K><<<(unsigned)grid, kThreads, 0, ctx->stream>>>(a);
    ctx->kend();
  }
  CJ_CUDA(cudaGetLastError());
  uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  CJ_CUDA(cudaMemcpyAsync(h, tot.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  return h[0];
}

template <class K>
uint64_t run(cj_ctx* ctx, NphjArgs a) {
  uint32_t log2cap = 1;
  while ((1ull << log2cap) < 2 * std::max<uint64_t>(a.nr, 1)) ++log2cap;
  a.log2cap = log2cap;
  a.key_words = sizeof(K) / 4;
  if (!a.unique && a.nr > 0) return run_sorted<K>(ctx, a);
  uint32_t words = 1 + a.key_words;
  for (int c = 0; c < a.nr_cols; ++c) {
    a.r_word_off[c] = words;
    words += a.r_bytes[c] / 4;
  }
  // 4-byte keys with <= 8 payload bytes: pad to 4 words so a slot is one aligned
  // 16-byte load/store
  if (sizeof(K) == 4 && words <= 4) words = 4;
  a.slot_words = words;
  const uint64_t cap = 1ull << log2cap;
  Scratch table(ctx, cap * words * 4);
  CJ_CUDA(cudaMemsetAsync(table.p, 0, cap * words * 4, ctx->stream));
  a.table = table.as<uint32_t>();
  Scratch tot(ctx, 8);
  CJ_CUDA(cudaMemsetAsync(tot.p, 0, 8, ctx->stream));
  a.total_out = tot.as<uint64_t>();
  a.err = ctx->err_word;
  if (a.nr > 0) {
    ctx->kbegin("nphj_build", a.nr * (uint64_t)(sizeof(K) + 4ull * a.slot_words));
    k_nphj_build<K><<<grid_for(a.nr, kThreads * 4, ctx->num_sms * 16), kThreads, 0, ctx->stream>>>(a);
    ctx->kend();
  }
  a.tiles = (a.ns + kTile - 1) / kTile;
  if (a.tiles > 0 && a.nr > 0) {
    a.status = ctx->status_buffer(a.tiles);
    a.epoch = ctx->next_epoch();
    a.ticket = ctx->ticket(3);
    auto launch = [&](auto kern) {
      int per_sm = 0;
      CJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0));
      const uint64_t grid = std::min<uint64_t>((uint64_t)ctx->num_sms * std::max(per_sm, 1), a.tiles);
      ctx->kbegin(a.write ? "nphj_probe" : "nphj_count", 0);
      kern<<<(unsigned)grid, kThreads, 0, ctx->stream>>>(a);
      ctx->kend();
    };
    // (non-unique builds took run_sorted above)
    const bool vec = sizeof(K) == 4 && a.slot_words == 4;
    if (vec) launch(k_nphj_probe_u<K, true>);
    else launch(k_nphj_probe_u<K, false>);
  }
  CJ_CUDA(cudaGetLastError());
  uint64_t* h = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  CJ_CUDA(cudaMemcpyAsync(h, tot.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CJ_CUDA(cudaStreamSynchronize(ctx->stream));
  return h[0];
}

}  // namespace

uint64_t nphj_find(cj_ctx* ctx, const void* rkeys, uint64_t nr, const void* skeys, uint64_t ns,
                   int key_bytes, const OutSpec& out, uint64_t capacity, bool count_only,
                   bool unique) {
  NphjArgs a{};
  a.unique = unique ? 1 : 0;
  a.rkeys = rkeys;
  a.nr = nr;
  a.skeys = skeys;
  a.ns = ns;
  a.write = count_only ? 0 : 1;
  a.capacity = capacity;
  if (!count_only) {
    a.key_out = out.key;
    a.ids_r = out.ids_r;
    a.ids_s = out.ids_s;
    a.nr_cols = out.nr;
    a.ns_cols = out.ns;
    for (int c = 0; c < out.nr; ++c) {
      a.r_src[c] = out.r_src[c];
      a.r_dst[c] = out.r_dst[c];
      a.r_bytes[c] = out.r_bytes[c];
    }
    for (int c = 0; c < out.ns; ++c) {
      a.s_src[c] = out.s_src[c];
      a.s_dst[c] = out.s_dst[c];
      a.s_bytes[c] = out.s_bytes[c];
    }
  }
  const uint64_t t = key_bytes == 4 ? run<uint32_t>(ctx, a) : run<uint64_t>(ctx, a);
  raise_device_errors(ctx);
  return t;
}

}  // namespace cj
