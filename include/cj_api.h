/* cj_api.h — C-ABI of the B200-native equi-join path (libcoljoin_b200.so).
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch
 * types.  The C++ host library (include/coljoin/ headers, libcoljoin_host) keeps
 * the reference's operator API on top of it; other hosts bind these symbols
 * directly (ctypes / cgo / JNI — see INTEGRATION.md).
 *
 * Each entry point names the reference interface it replaces (paths relative
 * to the reference's proj/ directory).
 *
 * Conventions
 *  - Every function returns a cj_status (0 = OK).  Codes 1..15 are 1:1 with the
 *    reference's exception classes (include/coljoin/errors.hpp:19-33); the
 *    host C++ layer rethrows the same class.  cj_last_error() has the text.
 *  - `_dev` pointers are device pointers (borrowed; the caller keeps them
 *    alive until the call returns or the ctx stream is synchronised).  Buffers
 *    the library allocates for results are released with cj_free().
 *  - One ctx per stream; a ctx is not thread-safe, distinct ctxs are.
 *  - Keys and payloads are unsigned 4- or 8-byte integers (column.hpp:14-19);
 *    tuple ids are u32 (column.hpp:21, kMaxRows = 2^31-1).
 */
#ifndef CJ_API_H
#define CJ_API_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CJ_OK = 0,
  CJ_ERR_LENGTH_MISMATCH = 1,     /* LengthMismatch      errors.hpp:19 */
  CJ_ERR_KIND = 2,                /* KindError           errors.hpp:20 */
  CJ_ERR_FANOUT_TOO_LARGE = 3,    /* FanoutTooLarge      errors.hpp:21 */
  CJ_ERR_INDEX_OUT_OF_BOUNDS = 4, /* IndexOutOfBounds    errors.hpp:22 */
  CJ_ERR_EMPTY_INPUT = 5,         /* EmptyInput          errors.hpp:23 */
  CJ_ERR_NOT_SORTED = 6,          /* NotSorted           errors.hpp:24 */
  CJ_ERR_DUPLICATE_BUILD_KEYS = 7,/* DuplicateBuildKeys  errors.hpp:25 */
  CJ_ERR_FANOUT_MISMATCH = 8,     /* FanoutMismatch      errors.hpp:26 */
  CJ_ERR_CAPACITY_EXCEEDED = 9,   /* CapacityExceeded    errors.hpp:27 */
  CJ_ERR_TRANSFORM_MISMATCH = 10, /* TransformMismatch   errors.hpp:28 */
  CJ_ERR_PHASE_ORDER = 11,        /* PhaseOrderViolation errors.hpp:29 */
  CJ_ERR_SPEC_INVALID = 12,       /* SpecInvalid         errors.hpp:30 */
  CJ_ERR_UNKNOWN_SHAPE = 13,      /* UnknownShape        errors.hpp:31 */
  CJ_ERR_SCHEMA = 14,             /* SchemaError         errors.hpp:32 */
  CJ_ERR_UNSUPPORTED = 15,        /* Unsupported         errors.hpp:33 */
  CJ_ERR_CUDA = 100,
  CJ_ERR_NCCL = 101,
  CJ_ERR_OUT_OF_MEMORY = 102
} cj_status;

enum { CJ_SMJ = 0, CJ_PHJ = 1, CJ_NPHJ = 2 };   /* JoinAlgo    task.hpp:12 (+ NPHJ) */
enum { CJ_GFUR = 0, CJ_GFTR = 1 };              /* JoinPattern task.hpp:13 */
enum { CJ_IDS_PHYSICAL = 0, CJ_IDS_VIRTUAL = 1 };/* TupleIdSemantics column.hpp:130 */

#define CJ_MAX_COLS 16     /* payload columns per relation side */
#define CJ_MAX_PASSES 8    /* radix passes in one plan (8 x 8 bits = 64-bit key) */

typedef struct cj_ctx cj_ctx;

/* ---- context ------------------------------------------------------------ */
/* stream: a cudaStream_t (NULL = a new non-blocking stream owned by the ctx). */
int cj_ctx_create(int device, void* stream, cj_ctx** out);
int cj_ctx_destroy(cj_ctx* ctx);
/* The cudaStream_t the ctx works on (callers order their own streams
 * against it, e.g. torch.cuda.ExternalStream + wait_stream). */
void* cj_ctx_stream(const cj_ctx* ctx);
const char* cj_last_error(const cj_ctx* ctx);
int cj_sync(cj_ctx* ctx);
int cj_free(cj_ctx* ctx, void* dev_ptr);
/* Stream-ordered device allocation from the ctx pool (test/bench helper). */
int cj_alloc(cj_ctx* ctx, uint64_t bytes, void** dev_ptr);
/* Stream-ordered copy on the ctx stream; kind 1 = host->device, 2 =
 * device->host, 3 = device->device.  Host->device/device->host copies are
 * synchronous with respect to the host (the call returns when done). */
int cj_copy(cj_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind);
/* Peak device scratch (bytes) held by operators since the last reset; the
 * host library charges it to the caller's Workspace ledger. */
uint64_t cj_scratch_peak(cj_ctx* ctx, int reset);
/* Kernel launches issued through this ctx since creation (bench evidence). */
uint64_t cj_launch_count(const cj_ctx* ctx);
/* Record (cudaEventRecord) a named timing mark on the ctx stream; elapsed ms
 * between two marks after cj_sync. */
int cj_mark(cj_ctx* ctx, int slot);
int cj_elapsed_ms(cj_ctx* ctx, int slot_a, int slot_b, float* ms);

/* Per-launch timing: when on, every kernel launched through the ctx is
 * bracketed by CUDA events on the ctx stream and recorded with its name and
 * algorithmic bytes (inputs read once + outputs written once).  Turning it on
 * clears the records.  cj_kernel_records fills up to max entries (names are
 * static strings) and returns the total record count in *count. */
int cj_set_kernel_timing(cj_ctx* ctx, int on);
int cj_kernel_records(cj_ctx* ctx, int max, const char** names, float* ms, uint64_t* bytes,
                      int* count);

/* ---- primitives (primitives.hpp:25-77) ---------------------------------- */

/* histogram(keys, low_bit, high_bit) — primitives.hpp:27-28.
 * counts_host: 2^(hi-lo) u32 on the HOST. */
int cj_histogram(cj_ctx* ctx, const void* keys_dev, uint64_t n, uint32_t key_bytes,
                 uint32_t low_bit, uint32_t high_bit, uint32_t* counts_host);

/* radix_partition(_keys) — primitives.hpp:38-47: ONE stable pass over
 * [low_bit, high_bit) carrying nvals value columns (nvals may be 0).
 * offsets_host: 2^(hi-lo)+1 u64 on the HOST (PartitionLayout::offsets). */
int cj_radix_partition(cj_ctx* ctx, const void* keys_dev, void* keys_out_dev, uint64_t n,
                       uint32_t key_bytes, uint32_t low_bit, uint32_t high_bit,
                       const void* const* vals_dev, void* const* vals_out_dev,
                       const uint32_t* val_bytes, uint32_t nvals, uint64_t* offsets_host);

/* radix_partition_passes(_keys) — primitives.hpp:52-59: stable LSD over the
 * plan (npasses <= 64), constant-digit passes skipped (primitives.cpp:217-256).
 * gen_ids != 0: value column 0 is not read but generated as the source row
 * index (u32) — GFUR's tuple ids born in pass 1 (join_engine.cpp:74-78). */
int cj_radix_partition_passes(cj_ctx* ctx, const void* keys_dev, void* keys_out_dev, uint64_t n,
                              uint32_t key_bytes, const uint32_t* plan_lo,
                              const uint32_t* plan_hi, uint32_t npasses,
                              const void* const* vals_dev, void* const* vals_out_dev,
                              const uint32_t* val_bytes, uint32_t nvals, int gen_ids);

/* sort_pairs / sort_keys — primitives.hpp:63-68: stable full-width sort. */
int cj_sort_pairs(cj_ctx* ctx, const void* keys_dev, void* keys_out_dev, uint64_t n,
                  uint32_t key_bytes, const void* const* vals_dev, void* const* vals_out_dev,
                  const uint32_t* val_bytes, uint32_t nvals, int gen_ids);

/* gather / gather_copy — primitives.hpp:71-74: out[c][i] = in[c][map[i]] for
 * ncols columns sharing one map; CJ_ERR_INDEX_OUT_OF_BOUNDS on map[i] >= n_in. */
int cj_gather(cj_ctx* ctx, const void* const* in_dev, uint64_t n_in, const uint32_t* map_dev,
              uint64_t m, void* const* out_dev, const uint32_t* col_bytes, uint32_t ncols);

/* ---- hash join (hash_match.hpp:26-81) ------------------------------------ */

/* partition_relation(_keys) — hash_match.hpp:26-38: LSD by the low
 * total_bits in passes of bits_per_pass; offsets_dev (2^total_bits + 1 u64,
 * DEVICE) receives the layout. */
int cj_partition_relation(cj_ctx* ctx, const void* keys_dev, void* keys_out_dev, uint64_t n,
                          uint32_t key_bytes, uint32_t total_bits, uint32_t bits_per_pass,
                          const void* const* vals_dev, void* const* vals_out_dev,
                          const uint32_t* val_bytes, uint32_t nvals, int gen_ids,
                          uint64_t* offsets_dev);

/* A partitioned side: keys + layout (+ carried u32 ids for physical mode). */
typedef struct {
  const void* keys;       /* device */
  const uint64_t* offsets;/* device, fanout + 1 */
  const uint32_t* carried;/* device or NULL */
  uint64_t rows;
} cj_partitioned;

/* hash_match_count + hash_match_fill — hash_match.cpp:212-302 in one device
 * pass (count, decoupled look-back over work units, fill).  Output order is
 * the reference's: (partition, build chunk of <= limit rows, probe position,
 * build insertion order).  *total_host receives the match count; the three
 * outputs are allocated by the library (cj_free). */
int cj_hash_find_matches(cj_ctx* ctx, const cj_partitioned* build, const cj_partitioned* probe,
                         uint32_t fanout, uint32_t key_bytes, uint32_t limit, int id_mode,
                         uint64_t* total_host, void** keys_out, uint32_t** ids_r_out,
                         uint32_t** ids_s_out);

/* ---- merge join (merge_match.hpp:25-52) --------------------------------- */

/* merge_match_count + merge_match_fill — emits every (i, j) with
 * r[i] == s[j] in (s-position, r-position) order (merge_match.hpp:44-47);
 * pk_fk emits only the first r match (merge_match.cpp:65-68). */
int cj_merge_find_matches(cj_ctx* ctx, const void* r_sorted_dev, uint64_t nr,
                          const void* s_sorted_dev, uint64_t ns, uint32_t key_bytes, int pk_fk,
                          int validate, uint64_t* total_host, void** keys_out,
                          uint32_t** ids_r_out, uint32_t** ids_s_out);

/* ---- end to end (join_engine.hpp:68 run_join) ----------------------------- */

typedef struct {
  const void* key;                 /* device (cj_run_join) or host (cj_run_join_host) */
  uint32_t key_bytes;              /* 4 | 8 */
  uint64_t rows;
  uint32_t npay;                   /* <= CJ_MAX_COLS */
  const void* pay[CJ_MAX_COLS];
  uint32_t pay_bytes[CJ_MAX_COLS];
  int key_unique;                  /* Relation::key_unique (column.hpp:120) */
} cj_relation;

typedef struct {                   /* JoinOptions (task.hpp:24-32) */
  int algo;                        /* CJ_SMJ | CJ_PHJ | CJ_NPHJ */
  int pattern;                     /* CJ_GFUR | CJ_GFTR */
  uint32_t radix_bits_per_pass;    /* default 8 */
  int total_radix_bits;            /* -1: default_total_radix_bits(|R|) */
  uint32_t sub_partition_limit;    /* default 4096 */
  int validate;
  int want_ids;                    /* also return the final gather maps (ids) */
  int want_stats;                  /* clusteredness of the gather maps (needs ids) */
} cj_join_options;

typedef struct {
  uint64_t rows;
  /* key (r.key kind), then R payloads, then S payloads (join_engine.cpp:115-123) */
  void* key;
  void* pay[2 * CJ_MAX_COLS];
  uint32_t* ids_r;                 /* when want_ids */
  uint32_t* ids_s;
  uint64_t transform_ns, find_ns, materialize_ns;   /* PhaseReport (mem_ledger.hpp:231-246) */
  double clusteredness_r, clusteredness_s;          /* JoinStats (join_engine.hpp:54-58) */
  uint64_t device_bytes_peak;      /* scratch + outputs held by the call */
  /* device bytes the call held (outputs included) at its high-water mark in
   * each phase */
  uint64_t peak_transform_b, peak_find_b, peak_materialize_b;
  /* PhaseReport::peak_by_phase (mem_ledger.hpp:26-100, 231-246): per phase
   * [transform, find, materialize], at the high-water mark of their sum, the
   * logical bytes of column-sized working data (transformed keys and carried
   * columns, tuple-id maps) and of scratch (LSD ping-pong, histograms,
   * layouts, find scratch); the output relation is not counted */
  uint64_t ledger_column_b[3];
  uint64_t ledger_scratch_b[3];
} cj_join_result;

void cj_default_options(cj_join_options* opt);

/* Device-resident run_join: inputs and outputs in HBM (outputs allocated by the
 * library, release each with cj_free or all with cj_result_free). */
int cj_run_join(cj_ctx* ctx, const cj_relation* build, const cj_relation* probe,
                const cj_join_options* opt, cj_join_result* res);
int cj_result_free(cj_ctx* ctx, cj_join_result* res);

/* Host-buffer run_join: the drop-in for coljoin::run_join(const JoinTask&).
 * Concurrent calls on one device (one ctx per host thread) take turns per
 * copy direction, so one call's download overlaps another's upload.
 * Uploads the host columns, runs cj_run_join, downloads the output into
 * host buffers allocated by the callback alloc(bytes, user) (e.g. a
 * std::vector resize, or a pinned arena).  Phase times exclude the copies;
 * h2d_ns / d2h_ns report them. */
typedef void* (*cj_host_alloc_fn)(uint64_t bytes, void* user);
int cj_run_join_host(cj_ctx* ctx, const cj_relation* build, const cj_relation* probe,
                     const cj_join_options* opt, cj_host_alloc_fn alloc, void* user,
                     cj_join_result* res_host, uint64_t* h2d_ns, uint64_t* d2h_ns);

/* ---- chained star joins (sequence.hpp:10-26 run_join_sequence) ----------- */
typedef struct {                   /* SequenceStep (sequence.hpp:10-15) */
  uint64_t rows;                   /* output cardinality of this join */
  uint32_t output_columns;         /* key + carried payloads + dim payload */
  uint64_t transform_ns, find_ns, materialize_ns;
  uint64_t fk_fetch_ns;            /* gathering the next FK column, between joins (GFUR;
                                      GFTR carries the FK columns through the earlier
                                      joins as probe payloads: 0) */
} cj_sequence_step;

/* run_join_sequence(fact, dims, algorithm, pattern, options) — sequence.cpp:9-67,
 * device-resident: join i probes (FK_i, ID, P_1..P_{i-1}) against dims[i]; the
 * result's ID column gathers FK_{i+1} on the device (no host copy between the
 * joins; every intermediate is released as soon as the next probe no longer
 * needs it).  fact: key = u32 tuple ids, pay[0..n_dims) = FK columns.  steps
 * receives n_dims entries; last (optional) receives the final join's output
 * (release with cj_result_free), else it is released. */
int cj_run_join_sequence(cj_ctx* ctx, const cj_relation* fact, const cj_relation* dims,
                         uint32_t n_dims, const cj_join_options* opt, cj_sequence_step* steps,
                         cj_join_result* last);

/* workloads::gen_star (workloads.cpp:135-160), bit-identical: fact_ids u32
 * iota; fks[d] (key_bytes) FK_d; dim_keys[d] (key_bytes) a Fisher-Yates
 * permutation of [0, dim_rows); dim_pays[d] (pay_bytes) its payload. */
int cj_gen_star(cj_ctx* ctx, uint64_t fact_rows, uint32_t dims, uint64_t dim_rows, uint64_t seed,
                uint32_t key_bytes, uint32_t pay_bytes, void* fact_ids, void* const* fks,
                void* const* dim_keys, void* const* dim_pays);

/* ---- multi-GPU radix sharding (no reference counterpart) ---- */
/* Stable partition of a relation's rows by shard s(key) = floor(mix64(key) *
 * parts / 2^64) (mix64 = rng.hpp:8-12), the send layout of the all-to-all
 * shuffle: rows of shard d land contiguously, in input order, in shard order;
 * counts_host[d] = rows of shard d.  Key-deterministic, so co-partitions of R
 * and S meet on one GPU. */
int cj_shard_partition(cj_ctx* ctx, const void* keys_dev, void* keys_out_dev, uint64_t n,
                       uint32_t key_bytes, uint32_t parts, const void* const* vals_dev,
                       void* const* vals_out_dev, const uint32_t* val_bytes, uint32_t nvals,
                       uint64_t* counts_host);

/* cj_shard_partition with the receiver's first LSD digit folded in: rows are
 * stably grouped by digit = shard << first_bits | (key & (2^first_bits - 1)),
 * i.e. by destination and, inside a destination, by the low first_bits key
 * bits; counts_host[parts << first_bits] rows per digit (row-major
 * [destination][low bits]).  parts << first_bits <= 256.  Rows wider than the
 * staging allows go in column groups (same permutation). */
int cj_shard_partition_ex(cj_ctx* ctx, const void* keys_dev, void* keys_out_dev, uint64_t n,
                          uint32_t key_bytes, uint32_t parts, uint32_t first_bits,
                          const void* const* vals_dev, void* const* vals_out_dev,
                          const uint32_t* val_bytes, uint32_t nvals, uint64_t* counts_host);

/* Placement of one all-to-all exchange of shard-grouped rows (host only, no
 * device work).  send_counts[dst][d]: rows this rank sends to dst with low
 * digit d (its cj_shard_partition_ex counts); recv_counts[src][d]: rows src
 * sends here.  send_off[dst][d] = row offset of that run in the send layout;
 * recv_off[src][d] = where src's digit-d run lands so that the received
 * relation is stably grouped by d (runs of one digit in source-rank order):
 * the first LSD pass of the local join is then already done.
 * *recv_total = rows received. */
int cj_exchange_plan(uint32_t world, uint32_t digits, const uint64_t* send_counts,
                     const uint64_t* recv_counts, uint64_t* send_off, uint64_t* recv_off,
                     uint64_t* recv_total);

/* ---- NCCL communicator and the sharded join -------------- */
/* NCCL is bound at run time (dlopen "libnccl.so.2": the copy a host process
 * already loaded, e.g. torch's, else the system one); CJ_ERR_NCCL when absent. */
#define CJ_COMM_ID_BYTES 128
typedef struct cj_comm cj_comm;
/* ncclGetUniqueId: rank 0 creates the id, the caller broadcasts the bytes. */
int cj_comm_unique_id(uint8_t* id_out);
/* One rank's communicator on ctx's device (ncclCommInitRank, plus a split
 * control communicator for count exchanges that must not queue behind data). */
int cj_comm_init(cj_ctx* ctx, const uint8_t* id, int nranks, int rank, cj_comm** out);
int cj_comm_destroy(cj_comm* comm);
int cj_comm_size(const cj_comm* comm);
int cj_comm_rank(const cj_comm* comm);

typedef struct {
  uint32_t first_bits;              /* low key bits pre-sorted by the exchange */
  uint64_t r_rows_received, s_rows_received;
  uint64_t bytes_sent_peers;        /* to other ranks (self excluded), R + S */
  uint64_t bytes_received_peers;
  uint64_t shard_ns;                /* both shard partitions (device time, ctx stream) */
  uint64_t exchange_r_ns, exchange_s_ns;  /* data exchanges (device time, comm stream) */
  uint64_t wall_ns;                 /* the whole call, host clock */
} cj_shuffle_stats;

/* Shuffle one relation: shard partition (with the first digit), count
 * exchange, grouped ncclSend/ncclRecv of every column into runs placed by
 * cj_exchange_plan.  out receives library-allocated device columns (release
 * with cj_relation_free); it is stably grouped by its low first_bits bits. */
int cj_shuffle_relation(cj_ctx* ctx, cj_comm* comm, const cj_relation* in, uint32_t first_bits,
                        cj_relation* out, cj_shuffle_stats* stats);
int cj_relation_free(cj_ctx* ctx, cj_relation* rel);

/* run_join on relations already stably grouped by their low presorted_bits
 * key bits (what cj_shuffle_relation delivers): the first LSD pass of the
 * transform is skipped.  Output multiset = cj_run_join's. */
int cj_run_join_presorted(cj_ctx* ctx, const cj_relation* build, const cj_relation* probe,
                          const cj_join_options* opt, uint32_t presorted_bits,
                          cj_join_result* res);

/* The radix-sharded join: every rank passes its slice of R and S; rows move to
 * shard(key)'s rank (the shuffle above, R's exchange overlapping S's shard
 * partition, S's overlapping R's local transform), and each rank joins its
 * shard.  res = this rank's share of the output (the union over ranks is the
 * join).  Collective: every rank of comm calls it with the same options. */
int cj_run_join_sharded(cj_ctx* ctx, cj_comm* comm, const cj_relation* build,
                        const cj_relation* probe, const cj_join_options* opt,
                        cj_join_result* res, cj_shuffle_stats* stats);

/* Weak-scaling shard generator: rank r of `ranks` gets |R|/ranks rows of a PK
 * domain that is a bijective scramble of [0, |R|) (|R| a power of two; a
 * 4-round Feistel permutation keyed by seed) and |S|/ranks uniform foreign
 * keys over [0, |R|) from the counter RNG; payload c is the stream 0x7000+c /
 * 0x8000+c at the global row index (workloads.cpp:124-129).  The reference
 * generator is sequential and capped at 2^31-1 rows (workloads.cpp:26-51), so
 * config C5 needs this one. */
int cj_gen_shard(cj_ctx* ctx, uint64_t r_rows_total, uint64_t s_rows_total, uint32_t rank,
                 uint32_t ranks, uint32_t r_pay, uint32_t s_pay, uint64_t seed, void* r_key_dev,
                 void* const* r_pay_dev, void* s_key_dev, void* const* s_pay_dev);

/* ---- workload generation (workloads.hpp:11-33 gen_pk_fk) ----------------- */
/* Bit-identical to workloads::gen_pk_fk: the Fisher-Yates permutation and the
 * Zipf CDF run on the host (sequential by definition), everything else on the
 * device.  Outputs are caller-provided device buffers; pay_bytes 4 or 8. */
int cj_gen_pk_fk(cj_ctx* ctx, uint64_t r_rows, uint64_t s_rows, uint32_t r_pay, uint32_t s_pay,
                 uint32_t key_bytes, uint32_t pay_bytes, double match_ratio, double zipf,
                 uint64_t seed, void* r_key_dev, void* const* r_pay_dev, void* s_key_dev,
                 void* const* s_pay_dev);

#ifdef __cplusplus
}
#endif
#endif
