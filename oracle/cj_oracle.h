/* cj_oracle — CPU restatement of the reference join path (TEST INFRASTRUCTURE).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library, and only as the checker.  It is never linked into the product.
 *
 * Every column is widened to uint64_t (keys compare unsigned, column.hpp:13-14;
 * widening preserves order and the Fibonacci slot hash, which the reference
 * computes on the u64-widened key, hash_match.cpp:24-26).  A column's storage
 * width (4 or 8 bytes) is passed where it matters: digit-range checks
 * (primitives.cpp:25-30), the full-width sort plan (primitives.cpp:258-261),
 * and u32 truncation of generated payloads (workloads.cpp:13-23).
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks this restatement against
 * outputs of the unmodified reference (oracle/_ref/refjoin) recorded in
 * tests/golden/ by tests/golden/make_golden.py.
 */
#ifndef CJ_ORACLE_H
#define CJ_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { CJO_OK = 0, CJO_FANOUT_TOO_LARGE = 3, CJO_INDEX_OOB = 4, CJO_EMPTY = 5,
       CJO_CAPACITY = 9, CJO_SPEC_INVALID = 12, CJO_NOMEM = 99 };

uint64_t cjo_mix64(uint64_t x);
uint64_t cjo_digest(const uint64_t* w, uint64_t n);
uint64_t cjo_digest_continue(uint64_t h, const uint64_t* w, uint64_t n, uint64_t i0);

/* workloads.cpp:89-133 gen_pk_fk.  Output arrays are caller-allocated:
 * r_key[r_rows], r_pay[r_pay * r_rows] (column-major), same for S.
 * pay_bytes 4 truncates payload draws to u32 (workloads.cpp:17). */
int cjo_gen_pk_fk(uint64_t r_rows, uint64_t s_rows, unsigned r_pay, unsigned s_pay,
                  double match_ratio, double zipf, uint64_t seed, unsigned pay_bytes,
                  uint64_t* r_key, uint64_t* r_pay_cols, uint64_t* s_key,
                  uint64_t* s_pay_cols);

/* task.hpp:45-50 */
unsigned cjo_default_total_radix_bits(uint64_t build_rows);

/* primitives.cpp:117-139 one stable pass (nvals columns, column-major).
 * offsets[(1<<(hi-lo))+1] out.  key_bytes bounds hi (primitives.cpp:25-30). */
int cjo_radix_partition(const uint64_t* keys, const uint64_t* vals, unsigned nvals,
                        uint64_t n, unsigned key_bytes, unsigned lo, unsigned hi,
                        uint64_t* keys_out, uint64_t* vals_out, uint64_t* offsets);

/* primitives.cpp:217-256 LSD multi-pass over plan (lo[i], hi[i]). */
int cjo_radix_partition_passes(const uint64_t* keys, const uint64_t* vals, unsigned nvals,
                               uint64_t n, unsigned key_bytes, const unsigned* plan_lo,
                               const unsigned* plan_hi, unsigned npasses,
                               uint64_t* keys_out, uint64_t* vals_out);

/* primitives.cpp:358-362 full-width 8-bit LSD sort. */
int cjo_sort_pairs(const uint64_t* keys, const uint64_t* vals, unsigned nvals, uint64_t n,
                   unsigned key_bytes, uint64_t* keys_out, uint64_t* vals_out);

/* hash_match.cpp:140-158 partition by the low total_bits; offsets[2^bits+1]. */
int cjo_partition_relation(const uint64_t* keys, const uint64_t* vals, unsigned nvals,
                           uint64_t n, unsigned key_bytes, unsigned total_bits,
                           unsigned bits_per_pass, uint64_t* keys_out, uint64_t* vals_out,
                           uint64_t* offsets);

/* primitives.cpp:369-396; returns CJO_INDEX_OOB on a map entry >= n_in. */
int cjo_gather(const uint64_t* in, uint64_t n_in, const uint32_t* map, uint64_t m,
               uint64_t* out);

/* hash_match.cpp:186-302: plan (limit), count, fill with Virtual ids.
 * Two calls: first with keys_out == NULL returns *total; then fill. */
int cjo_hash_find_matches(const uint64_t* bkeys, const uint64_t* boff, uint64_t nb,
                          const uint64_t* pkeys, const uint64_t* poff, uint64_t np,
                          unsigned fanout, uint32_t limit, uint64_t* total,
                          uint64_t* keys_out, uint32_t* ids_r, uint32_t* ids_s);

/* merge_match.cpp:53-168 (the output is identical for every part count). */
int cjo_merge_find_matches(const uint64_t* r, uint64_t nr, const uint64_t* s, uint64_t ns,
                           int pk_fk, uint64_t* total, uint64_t* keys_out,
                           uint32_t* ids_r, uint32_t* ids_s);

/* join_engine.cpp:255-361 run_join.  algo 0 = SMJ, 1 = PHJ; pattern 0 = GFUR,
 * 1 = GFTR (task.hpp:12-13).  Inputs are column-major payload blocks.  Call
 * once with out_key == NULL to get *rows_out, then with buffers:
 * out_key[rows], out_pay[(r_pay + s_pay) * rows] (R payloads first,
 * join_engine.cpp:115-123), ids_r/ids_s (may be NULL) = final gather maps. */
int cjo_run_join(int algo, int pattern, const uint64_t* r_key, const uint64_t* r_pay,
                 unsigned r_npay, uint64_t nr, int r_key_unique, const uint64_t* s_key,
                 const uint64_t* s_pay, unsigned s_npay, uint64_t ns, unsigned key_bytes,
                 int total_bits, uint32_t limit, uint64_t* rows_out, uint64_t* out_key,
                 uint64_t* out_pay, uint32_t* ids_r, uint32_t* ids_s);

/* oracle.cpp:77-88 canonical rows (row-major, lexicographically sorted) and the
 * digest h = 0x12345678; h = mix64(h ^ w[i]) + i over them.
 * cols: ncols column pointers of nrows each. */
uint64_t cjo_canonical_digest(const uint64_t* const* cols, unsigned ncols, uint64_t nrows);

/* oracle.cpp:41-75 nested loop join, canonical order, two-call protocol. */
int cjo_nested_loop_join(const uint64_t* r_key, const uint64_t* r_pay, unsigned r_npay,
                         uint64_t nr, const uint64_t* s_key, const uint64_t* s_pay,
                         unsigned s_npay, uint64_t ns, uint64_t* rows_out,
                         uint64_t* out_rows /* row-major, width 1+r_npay+s_npay */);

#ifdef __cplusplus
}
#endif
#endif
