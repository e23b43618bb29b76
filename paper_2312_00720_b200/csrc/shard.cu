// Radix-sharded multi-GPU join over NCCL (the reference has no
// multi-GPU path).
//
// One process per GPU.  Every rank holds a slice of R and of S.  A row goes to
// rank shard(key) = floor(mix64(key) * world / 2^64) (mix64 = rng.hpp:8-12),
// so equal keys of R and S meet on one rank.  Per relation:
//   1. send layout: ONE stable scatter pass whose digit is (shard, low f key
//      bits) — the destination AND the receiver's first LSD digit
//      (radix.cu shard_partition);
//   2. count exchange: world x 2^f run lengths per rank (control communicator);
//   3. data exchange: grouped ncclSend/ncclRecv of every column, one message
//      per (peer, digit) run, each received run placed by cj_exchange_plan so
//      the received relation is stably grouped by its low f bits;
//   4. the local join skips its first LSD pass (JoinHooks::presorted_bits).
// The shard pass therefore replaces the local first pass instead of adding a
// pass.  R's exchange runs on the data stream while S is shard-partitioned on
// the ctx stream, and S's exchange while R's remaining passes run.
//
// NCCL is bound with dlopen at first use: inside a torch process that is the
// libnccl.so.2 torch already loaded (same soname), in a plain C/C++ host the
// system one; nothing links against a particular copy.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cj_device.cuh"
#include "cj_internal.cuh"

namespace cj {
namespace {

struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommSplit) comm_split = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    x.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!x.h) x.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!x.h) return x;
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(x.h, name));
    };
    sym(x.get_unique_id, "ncclGetUniqueId");
    sym(x.comm_init_rank, "ncclCommInitRank");
    sym(x.comm_split, "ncclCommSplit");
    sym(x.comm_destroy, "ncclCommDestroy");
    sym(x.send, "ncclSend");
    sym(x.recv, "ncclRecv");
    sym(x.group_start, "ncclGroupStart");
    sym(x.group_end, "ncclGroupEnd");
    sym(x.all_reduce, "ncclAllReduce");
    sym(x.error_string, "ncclGetErrorString");
    return x;
  }();
  if (!n.h || !n.send || !n.recv || !n.comm_init_rank || !n.comm_split)
    fail(CJ_ERR_NCCL, "NCCL unavailable (dlopen libnccl.so.2 failed or symbols missing)");
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(CJ_ERR_NCCL, std::string(what) + ": " + nccl().error_string(r));
}
#define CJ_NCCL(x) ::cj::nccl_check((x), #x)

uint64_t now_ns() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Copies of this rank's own runs (send layout -> receive layout) on the data
// stream: run i moves rows [src[i], src[i] + len[i]) to dst[i] in every column.
struct RunCopy {
  const void* in[CJ_MAX_COLS + 1];
  void* out[CJ_MAX_COLS + 1];
  uint32_t bytes[CJ_MAX_COLS + 1];
  int ncols;
  int nruns;
  uint64_t src[256], dst[256], len[256];
};

__global__ void k_copy_runs(const __grid_constant__ RunCopy rc) {
  const int r = blockIdx.y;
  const uint64_t len = rc.len[r];
  for (int c = 0; c < rc.ncols; ++c) {
    if (rc.bytes[c] == 4) {
      const uint32_t* in = static_cast<const uint32_t*>(rc.in[c]) + rc.src[r];
      uint32_t* out = static_cast<uint32_t*>(rc.out[c]) + rc.dst[r];
      for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
           i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
    } else {
      const uint64_t* in = static_cast<const uint64_t*>(rc.in[c]) + rc.src[r];
      uint64_t* out = static_cast<uint64_t*>(rc.out[c]) + rc.dst[r];
      for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
           i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
    }
  }
}

}  // namespace
}  // namespace cj

struct cj_comm {
  cj_ctx* ctx = nullptr;
  int nranks = 1, rank = 0;
  ncclComm_t data = nullptr;   // column exchanges (data stream)
  ncclComm_t ctrl = nullptr;   // count exchanges and reductions (ctrl stream)
  cudaStream_t data_stream = nullptr, ctrl_stream = nullptr;
  uint64_t* ctrl_buf = nullptr;  // device, 2 * 256 * nranks u64
  uint64_t* ctrl_host = nullptr; // pinned
};

namespace cj {
namespace {

// Host-side placement of one exchange (cj_exchange_plan).
void exchange_plan(uint32_t world, uint32_t digits, const uint64_t* send_counts,
                   const uint64_t* recv_counts, uint64_t* send_off, uint64_t* recv_off,
                   uint64_t* recv_total) {
  uint64_t o = 0;
  for (uint32_t p = 0; p < world; ++p)
    for (uint32_t d = 0; d < digits; ++d) {
      send_off[(size_t)p * digits + d] = o;
      o += send_counts[(size_t)p * digits + d];
    }
  // receive side: digit-major, source rank order inside a digit
  uint64_t r = 0;
  for (uint32_t d = 0; d < digits; ++d)
    for (uint32_t p = 0; p < world; ++p) {
      recv_off[(size_t)p * digits + d] = r;
      r += recv_counts[(size_t)p * digits + d];
    }
  *recv_total = r;
}

struct Columns {  // key + payload columns of one relation (device)
  void* key = nullptr;
  std::vector<void*> pay;
};

Columns alloc_like(cj_ctx* ctx, const cj_relation* in, uint64_t rows) {
  Columns c;
  c.key = ctx->alloc(rows * in->key_bytes + kPad);
  for (uint32_t i = 0; i < in->npay; ++i) c.pay.push_back(ctx->alloc(rows * in->pay_bytes[i] + kPad));
  return c;
}

void release(cj_ctx* ctx, Columns& c) {
  if (c.key) ctx->release(c.key);
  for (void* p : c.pay) ctx->release(p);
  c.key = nullptr;
  c.pay.clear();
}

// One relation's shuffle in flight: the send layout, the received columns,
// and the event the consumer waits on.
struct Exchange {
  Columns send, recv;
  uint64_t recv_rows = 0;
  uint64_t bytes_peers_out = 0, bytes_peers_in = 0;
  cudaEvent_t part0 = nullptr, part1 = nullptr, x0 = nullptr, x1 = nullptr;
  Exchange() {
    CJ_CUDA(cudaEventCreate(&part0));
    CJ_CUDA(cudaEventCreate(&part1));
    CJ_CUDA(cudaEventCreate(&x0));
    CJ_CUDA(cudaEventCreate(&x1));
  }
  ~Exchange() {
    cudaEventDestroy(part0);
    cudaEventDestroy(part1);
    cudaEventDestroy(x0);
    cudaEventDestroy(x1);
  }
  Exchange(const Exchange&) = delete;
  Exchange& operator=(const Exchange&) = delete;
  float ms(cudaEvent_t a, cudaEvent_t b) const {
    float m = 0;
    CJ_CUDA(cudaEventElapsedTime(&m, a, b));
    return m;
  }
};

// Sum of a u64 over the ranks (ctrl communicator; host value in, host out).
uint64_t allreduce_sum(cj_comm* cm, uint64_t v) {
  const Nccl& N = nccl();
  cm->ctrl_host[0] = v;
  CJ_CUDA(cudaMemcpyAsync(cm->ctrl_buf, cm->ctrl_host, 8, cudaMemcpyHostToDevice, cm->ctrl_stream));
  CJ_NCCL(N.all_reduce(cm->ctrl_buf, cm->ctrl_buf + 1, 1, ncclUint64, ncclSum, cm->ctrl,
                       cm->ctrl_stream));
  CJ_CUDA(cudaMemcpyAsync(cm->ctrl_host, cm->ctrl_buf + 1, 8, cudaMemcpyDeviceToHost,
                          cm->ctrl_stream));
  CJ_CUDA(cudaStreamSynchronize(cm->ctrl_stream));
  return cm->ctrl_host[0];
}

// Steps 1-3 for one relation; the data exchange is left in flight on the data
// stream (ex.x1 marks its end).
void start_exchange(cj_comm* cm, const cj_relation* in, uint32_t f, Exchange& ex) {
  cj_ctx* ctx = cm->ctx;
  const Nccl& N = nccl();
  const uint32_t W = (uint32_t)cm->nranks, D = 1u << f;
  const uint64_t n = in->rows;
  const int kb = (int)in->key_bytes;
  // 1. send layout: stable by (destination, low f bits)
  ex.send = alloc_like(ctx, in, n);
  ValCols v;
  v.n = (int)in->npay;
  for (uint32_t c = 0; c < in->npay; ++c) {
    v.in[c] = in->pay[c];
    v.out[c] = ex.send.pay[c];
    v.bytes[c] = in->pay_bytes[c];
  }
  std::vector<uint64_t> sc((size_t)W * D), rc((size_t)W * D), so((size_t)W * D), ro((size_t)W * D);
  CJ_CUDA(cudaEventRecord(ex.part0, ctx->stream));
  shard_partition(ctx, in->key, ex.send.key, n, kb, W, f, v, sc.data());
  CJ_CUDA(cudaEventRecord(ex.part1, ctx->stream));
  // 2. run lengths: rank p learns sc[p][*] of every rank (ctrl communicator)
  std::memcpy(cm->ctrl_host, sc.data(), sizeof(uint64_t) * W * D);
  uint64_t* sbuf = cm->ctrl_buf;
  uint64_t* rbuf = cm->ctrl_buf + (size_t)W * 256;
  CJ_CUDA(cudaMemcpyAsync(sbuf, cm->ctrl_host, sizeof(uint64_t) * W * D, cudaMemcpyHostToDevice,
                          cm->ctrl_stream));
  CJ_NCCL(N.group_start());
  for (uint32_t p = 0; p < W; ++p) {
    CJ_NCCL(N.send(sbuf + (size_t)p * D, D, ncclUint64, (int)p, cm->ctrl, cm->ctrl_stream));
    CJ_NCCL(N.recv(rbuf + (size_t)p * D, D, ncclUint64, (int)p, cm->ctrl, cm->ctrl_stream));
  }
  CJ_NCCL(N.group_end());
  CJ_CUDA(cudaMemcpyAsync(cm->ctrl_host, rbuf, sizeof(uint64_t) * W * D, cudaMemcpyDeviceToHost,
                          cm->ctrl_stream));
  CJ_CUDA(cudaStreamSynchronize(cm->ctrl_stream));
  std::memcpy(rc.data(), cm->ctrl_host, sizeof(uint64_t) * W * D);
  exchange_plan(W, D, sc.data(), rc.data(), so.data(), ro.data(), &ex.recv_rows);
  // one rank: the send layout is already the received relation (CJ_SHUFFLE_COPY=1
  // forces the general path, own runs through the copy kernel: tests)
  static const bool force_copy = [] {
    const char* e = std::getenv("CJ_SHUFFLE_COPY");
    return e && std::strcmp(e, "1") == 0;
  }();
  if (W == 1 && !force_copy) {
    ex.recv = ex.send;
    ex.send = Columns();
    CJ_CUDA(cudaEventRecord(ex.x0, ctx->stream));
    CJ_CUDA(cudaEventRecord(ex.x1, ctx->stream));
    return;
  }
  // 3. receive buffers (ctx-stream allocations: the data stream waits for them)
  ex.recv = alloc_like(ctx, in, ex.recv_rows);
  cudaEvent_t ready;
  CJ_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  CJ_CUDA(cudaEventRecord(ready, ctx->stream));
  CJ_CUDA(cudaStreamWaitEvent(cm->data_stream, ready, 0));
  cudaEventDestroy(ready);
  CJ_CUDA(cudaEventRecord(ex.x0, cm->data_stream));
  std::vector<std::pair<const void*, void*>> cols{{ex.send.key, ex.recv.key}};
  std::vector<uint32_t> widths{in->key_bytes};
  for (uint32_t c = 0; c < in->npay; ++c) {
    cols.push_back({ex.send.pay[c], ex.recv.pay[c]});
    widths.push_back(in->pay_bytes[c]);
  }
  // this rank's own runs: one copy kernel on the data stream
  {
    RunCopy rcp{};
    rcp.ncols = (int)cols.size();
    for (size_t c = 0; c < cols.size(); ++c) {
      rcp.in[c] = cols[c].first;
      rcp.out[c] = cols[c].second;
      rcp.bytes[c] = widths[c];
    }
    uint64_t most = 0;
    const uint32_t me = (uint32_t)cm->rank;
    for (uint32_t d = 0; d < D; ++d) {
      const size_t i = (size_t)me * D + d;
      if (!sc[i]) continue;
      rcp.src[rcp.nruns] = so[i];
      rcp.dst[rcp.nruns] = ro[i];
      rcp.len[rcp.nruns] = sc[i];
      most = std::max(most, sc[i]);
      ++rcp.nruns;
    }
    if (rcp.nruns) {
      const unsigned gx = (unsigned)std::min<uint64_t>((most + 4095) / 4096, 64);
      k_copy_runs<<<dim3(std::max(gx, 1u), rcp.nruns), 256, 0, cm->data_stream>>>(rcp);
      CJ_CUDA(cudaGetLastError());
      ++ctx->launches;
    }
  }
  // peers: one group per column, W - 1 peers x D runs each way
  for (size_t c = 0; c < cols.size(); ++c) {
    const uint64_t w = widths[c];
    const uint8_t* sb = static_cast<const uint8_t*>(cols[c].first);
    uint8_t* rb = static_cast<uint8_t*>(cols[c].second);
    CJ_NCCL(N.group_start());
    for (uint32_t p = 0; p < W; ++p)
      for (uint32_t d = 0; d < D && (int)p != cm->rank; ++d) {
        const size_t i = (size_t)p * D + d;
        if (sc[i]) CJ_NCCL(N.send(sb + so[i] * w, sc[i] * w, ncclUint8, (int)p, cm->data, cm->data_stream));
        if (rc[i]) CJ_NCCL(N.recv(rb + ro[i] * w, rc[i] * w, ncclUint8, (int)p, cm->data, cm->data_stream));
      }
    CJ_NCCL(N.group_end());
  }
  CJ_CUDA(cudaEventRecord(ex.x1, cm->data_stream));
  uint64_t row = in->key_bytes;
  for (uint32_t c = 0; c < in->npay; ++c) row += in->pay_bytes[c];
  for (uint32_t p = 0; p < W; ++p) {
    if ((int)p == cm->rank) continue;
    for (uint32_t d = 0; d < D; ++d) {
      ex.bytes_peers_out += sc[(size_t)p * D + d] * row;
      ex.bytes_peers_in += rc[(size_t)p * D + d] * row;
    }
  }
}

cj_relation received(const cj_relation* in, const Exchange& ex) {
  cj_relation r = *in;
  r.key = ex.recv.key;
  r.rows = ex.recv_rows;
  for (uint32_t c = 0; c < in->npay; ++c) r.pay[c] = ex.recv.pay[c];
  return r;
}

uint32_t shard_bits(int world) {
  uint32_t b = 0;
  while ((1 << b) < world) ++b;
  return b;
}

}  // namespace
}  // namespace cj

extern "C" {

int cj_exchange_plan(uint32_t world, uint32_t digits, const uint64_t* send_counts,
                     const uint64_t* recv_counts, uint64_t* send_off, uint64_t* recv_off,
                     uint64_t* recv_total) {
  return cj::guarded(nullptr, [&] {
    if (!send_counts || !recv_counts || !send_off || !recv_off || !recv_total || world == 0 ||
        digits == 0)
      cj::fail(CJ_ERR_SPEC_INVALID, "exchange plan: null argument or empty shape");
    cj::exchange_plan(world, digits, send_counts, recv_counts, send_off, recv_off, recv_total);
  });
}

int cj_comm_unique_id(uint8_t* id_out) {
  return cj::guarded(nullptr, [&] {
    ncclUniqueId id;
    CJ_NCCL(cj::nccl().get_unique_id(&id));
    std::memcpy(id_out, id.internal, CJ_COMM_ID_BYTES);
  });
}

int cj_comm_init(cj_ctx* ctx, const uint8_t* id, int nranks, int rank, cj_comm** out) {
  return cj::guarded(ctx, [&] {
    if (!ctx || !id || !out || nranks < 1 || rank < 0 || rank >= nranks)
      cj::fail(CJ_ERR_SPEC_INVALID, "comm_init: bad arguments");
    const cj::Nccl& N = cj::nccl();
    CJ_CUDA(cudaSetDevice(ctx->device));
    auto* c = new cj_comm();
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    try {
      ncclUniqueId u;
      std::memcpy(u.internal, id, CJ_COMM_ID_BYTES);
      CJ_NCCL(N.comm_init_rank(&c->data, nranks, u, rank));
      CJ_NCCL(N.comm_split(c->data, 0, rank, &c->ctrl, nullptr));
      CJ_CUDA(cudaStreamCreateWithFlags(&c->data_stream, cudaStreamNonBlocking));
      CJ_CUDA(cudaStreamCreateWithFlags(&c->ctrl_stream, cudaStreamNonBlocking));
      CJ_CUDA(cudaMalloc(&c->ctrl_buf, sizeof(uint64_t) * 2 * 256 * nranks + 64));
      CJ_CUDA(cudaMallocHost(&c->ctrl_host, sizeof(uint64_t) * 256 * nranks + 64));
    } catch (...) {
      cj_comm_destroy(c);
      throw;
    }
    *out = c;
  });
}

int cj_comm_destroy(cj_comm* c) {
  if (!c) return CJ_OK;
  cudaSetDevice(c->ctx->device);
  if (c->data_stream) cudaStreamSynchronize(c->data_stream);
  if (c->ctrl_stream) cudaStreamSynchronize(c->ctrl_stream);
  try {
    const cj::Nccl& N = cj::nccl();
    if (c->ctrl) N.comm_destroy(c->ctrl);
    if (c->data) N.comm_destroy(c->data);
  } catch (...) {
  }
  if (c->data_stream) cudaStreamDestroy(c->data_stream);
  if (c->ctrl_stream) cudaStreamDestroy(c->ctrl_stream);
  if (c->ctrl_buf) cudaFree(c->ctrl_buf);
  if (c->ctrl_host) cudaFreeHost(c->ctrl_host);
  delete c;
  return CJ_OK;
}

int cj_comm_size(const cj_comm* c) { return c ? c->nranks : 0; }
int cj_comm_rank(const cj_comm* c) { return c ? c->rank : -1; }

int cj_shuffle_relation(cj_ctx* ctx, cj_comm* cm, const cj_relation* in, uint32_t first_bits,
                        cj_relation* out, cj_shuffle_stats* st) {
  return cj::guarded(ctx, [&] {
    if (!cm || !in || !out || cm->ctx != ctx) cj::fail(CJ_ERR_SPEC_INVALID, "shuffle: bad arguments");
    cj::validate_relation(in, "a relation");
    const uint64_t t0 = cj::now_ns();
    cj::Exchange ex;
    try {
      cj::start_exchange(cm, in, first_bits, ex);
    } catch (...) {
      CJ_CUDA(cudaStreamSynchronize(cm->data_stream));
      cj::release(ctx, ex.send);
      cj::release(ctx, ex.recv);
      throw;
    }
    CJ_CUDA(cudaStreamWaitEvent(ctx->stream, ex.x1, 0));
    cj::release(ctx, ex.send);
    CJ_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = cj::received(in, ex);
    if (st) {
      std::memset(st, 0, sizeof(*st));
      st->first_bits = first_bits;
      st->r_rows_received = ex.recv_rows;
      st->bytes_sent_peers = ex.bytes_peers_out;
      st->bytes_received_peers = ex.bytes_peers_in;
      st->shard_ns = (uint64_t)(ex.ms(ex.part0, ex.part1) * 1e6);
      st->exchange_r_ns = (uint64_t)(ex.ms(ex.x0, ex.x1) * 1e6);
      st->wall_ns = cj::now_ns() - t0;
    }
  });
}

int cj_relation_free(cj_ctx* ctx, cj_relation* rel) {
  return cj::guarded(ctx, [&] {
    if (!rel) return;
    if (rel->key) ctx->release(const_cast<void*>(rel->key));
    for (uint32_t c = 0; c < rel->npay && c < CJ_MAX_COLS; ++c)
      if (rel->pay[c]) ctx->release(const_cast<void*>(rel->pay[c]));
    rel->key = nullptr;
    for (auto& p : rel->pay) p = nullptr;
    rel->rows = 0;
  });
}

int cj_run_join_sharded(cj_ctx* ctx, cj_comm* cm, const cj_relation* R, const cj_relation* S,
                        const cj_join_options* opt, cj_join_result* res, cj_shuffle_stats* st) {
  return cj::guarded(ctx, [&] {
    if (!cm || !R || !S || !opt || !res || cm->ctx != ctx)
      cj::fail(CJ_ERR_SPEC_INVALID, "sharded join: bad arguments");
    cj::validate_relation(R, "a build relation");
    cj::validate_relation(S, "a probe relation");
    if (R->key_bytes != S->key_bytes) cj::fail(CJ_ERR_KIND, "build and probe key kinds differ");
    const uint64_t t0 = cj::now_ns();
    std::memset(res, 0, sizeof(*res));
    // the partition bits every rank uses: default_total_radix_bits of the
    // expected shard of R (|R| summed over the ranks / ranks)
    cj_join_options o = *opt;
    const uint32_t sb = cj::shard_bits(cm->nranks);
    if (sb > 8) cj::fail(CJ_ERR_UNSUPPORTED, "at most 256 ranks");
    if (o.algo == CJ_PHJ && o.total_radix_bits < 0) {
      const uint64_t r_total = cj::allreduce_sum(cm, R->rows);
      o.total_radix_bits =
          (int)cj::default_total_radix_bits((r_total + cm->nranks - 1) / cm->nranks);
    }
    // the receiver's first LSD digit rides in the shard pass
    // (shard, first digit) in at most 64 digits: the shard pass costs what a
    // local 6-bit pass costs (64-entry digit tables)
    uint32_t f = 0;
    if (o.algo == CJ_PHJ) f = std::min<uint32_t>((uint32_t)o.total_radix_bits, sb < 6 ? 6u - sb : 0u);
    else if (o.algo == CJ_SMJ) f = sb < 6 ? 6u - sb : 0u;
    cj::Exchange xr, xs;
    auto cleanup = [&] {
      cudaStreamSynchronize(cm->data_stream);
      cudaStreamSynchronize(ctx->stream);
      cj::release(ctx, xr.send);
      cj::release(ctx, xr.recv);
      cj::release(ctx, xs.send);
      cj::release(ctx, xs.recv);
    };
    try {
      cj::start_exchange(cm, R, f, xr);  // R travels while S is shard-partitioned
      cj::start_exchange(cm, S, f, xs);
      const cj_relation Rr = cj::received(R, xr), Sr = cj::received(S, xs);
      cj::JoinHooks h;
      h.presorted_bits = f;
      h.before_side = [&](int side) {
        CJ_CUDA(cudaStreamWaitEvent(ctx->stream, side == 0 ? xr.x1 : xs.x1, 0));
      };
      cj::run_join_dev(ctx, &Rr, &Sr, &o, res, &h);
    } catch (...) {
      cj::free_output(ctx, res);
      cleanup();
      throw;
    }
    if (st) {
      std::memset(st, 0, sizeof(*st));
      st->first_bits = f;
      st->r_rows_received = xr.recv_rows;
      st->s_rows_received = xs.recv_rows;
      st->bytes_sent_peers = xr.bytes_peers_out + xs.bytes_peers_out;
      st->bytes_received_peers = xr.bytes_peers_in + xs.bytes_peers_in;
      st->shard_ns = (uint64_t)((xr.ms(xr.part0, xr.part1) + xs.ms(xs.part0, xs.part1)) * 1e6);
      st->exchange_r_ns = (uint64_t)(xr.ms(xr.x0, xr.x1) * 1e6);
      st->exchange_s_ns = (uint64_t)(xs.ms(xs.x0, xs.x1) * 1e6);
    }
    cleanup();
    if (st) st->wall_ns = cj::now_ns() - t0;
  });
}

}  // extern "C"
