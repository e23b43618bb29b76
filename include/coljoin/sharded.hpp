// Radix-sharded multi-GPU join for C++ callers of the reference API (the
// reference has no multi-GPU path).  One process per
// GPU: every rank passes its slices of R and S in a JoinTask and receives its
// share of the output; the union over the ranks is run_join's result.
//
// Implementation: host/coljoin_host.cpp over the C-ABI (cj_comm_*,
// cj_run_join_sharded in include/cj_api.h; csrc/shard.cu).  The caller ships
// the communicator id from rank 0 to the other ranks (MPI, a file, a socket).
#pragma once

#include <array>
#include <cstdint>

#include "cj_api.h"
#include "coljoin/join_engine.hpp"

namespace coljoin::sharded {

using CommId = std::array<uint8_t, CJ_COMM_ID_BYTES>;

// A fresh communicator id (ncclGetUniqueId), made on rank 0.
CommId make_comm_id();

// This rank's NCCL communicator on the library's device.
class Comm {
 public:
  Comm(const CommId& id, int nranks, int rank);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  int size() const;
  int rank() const;
  cj_comm* handle() const { return comm_; }

 private:
  cj_comm* comm_ = nullptr;
};

struct ShuffleStats {
  unsigned first_bits = 0;          // low key bits the exchange pre-sorted
  uint64_t r_rows_received = 0, s_rows_received = 0;
  uint64_t bytes_sent_peers = 0, bytes_received_peers = 0;
  uint64_t shard_ns = 0, exchange_r_ns = 0, exchange_s_ns = 0, wall_ns = 0;
};

// run_join (join_engine.hpp:68) across the ranks of `comm`: collective, every
// rank calls it with the same algorithm, pattern and options.
JoinOutput run_join(const JoinTask& task, Comm& comm, ShuffleStats* stats = nullptr);

}  // namespace coljoin::sharded
