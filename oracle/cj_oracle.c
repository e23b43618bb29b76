/* cj_oracle.c — plain-C restatement of the reference join path.
 * TEST INFRASTRUCTURE ONLY (see cj_oracle.h).  Every function cites the
 * reference file:line (paths relative to /root/reference/proj/) it restates.
 * Single-threaded and deliberately naive: it is the checker, not a baseline.
 */
#define _GNU_SOURCE
#include "cj_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GOLD 0x9E3779B97F4A7C15ull

/* include/coljoin/rng.hpp:8-12 — SplitMix64 finaliser */
uint64_t cjo_mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* BASELINE.md §2 digest over the flat canonical-row words */
uint64_t cjo_digest(const uint64_t* w, uint64_t n) {
  uint64_t h = 0x12345678ull;
  for (uint64_t i = 0; i < n; ++i) h = cjo_mix64(h ^ w[i]) + i;
  return h;
}

/* The same digest fed in pieces: h from the previous piece (0x12345678 for the
 * first), i0 = number of words already digested. */
uint64_t cjo_digest_continue(uint64_t h, const uint64_t* w, uint64_t n, uint64_t i0) {
  for (uint64_t i = 0; i < n; ++i) h = cjo_mix64(h ^ w[i]) + (i0 + i);
  return h;
}

/* ---- rng.hpp:18-37 CounterRng ------------------------------------------ */
typedef struct { uint64_t seed; } rng_t;
static rng_t rng_make(uint64_t seed) { rng_t r = {seed}; return r; }
static rng_t rng_stream(rng_t r, uint64_t tag) {
  rng_t o = {cjo_mix64(r.seed ^ cjo_mix64(tag + GOLD))};
  return o;
}
static uint64_t rng_at(rng_t r, uint64_t i) { return cjo_mix64(r.seed + (i + 1) * GOLD); }
static double rng_u01(rng_t r, uint64_t i) {
  return (double)(rng_at(r, i) >> 11) * 0x1.0p-53;
}
static uint64_t rng_below(rng_t r, uint64_t i, uint64_t bound) {
  return (uint64_t)(((unsigned __int128)rng_at(r, i) * bound) >> 64);
}

/* workloads.cpp:26-34 Fisher-Yates over [0, n) */
static uint64_t* permutation(uint64_t n, rng_t rng) {
  uint64_t* p = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  if (!p) return NULL;
  for (uint64_t i = 0; i < n; ++i) p[i] = i;
  for (uint64_t i = n; i > 1; --i) {
    const uint64_t j = rng_below(rng, i, i);
    const uint64_t t = p[i - 1];
    p[i - 1] = p[j];
    p[j] = t;
  }
  return p;
}

/* workloads.cpp:55-81 ZipfSampler + workloads.cpp:89-133 gen_pk_fk */
int cjo_gen_pk_fk(uint64_t r_rows, uint64_t s_rows, unsigned r_pay, unsigned s_pay,
                  double match_ratio, double zipf, uint64_t seed, unsigned pay_bytes,
                  uint64_t* r_key, uint64_t* r_pay_cols, uint64_t* s_key,
                  uint64_t* s_pay_cols) {
  if (match_ratio < 0.0 || match_ratio > 1.0 || zipf < 0.0) return CJO_SPEC_INVALID;
  if (r_rows > 0x7fffffffull || s_rows > 0x7fffffffull) return CJO_SPEC_INVALID;
  const rng_t master = rng_make(seed);
  uint64_t* perm = permutation(r_rows, rng_stream(master, 0x52000001ull));
  if (!perm) return CJO_NOMEM;
  memcpy(r_key, perm, r_rows * sizeof(uint64_t));
  free(perm);

  if (r_rows > 0 && s_rows > 0) {
    const rng_t zr = rng_stream(rng_make(seed), 0x5a1bf001ull);
    double* cdf = NULL;
    uint64_t* rank_to_key = NULL;
    if (zipf > 0.0) {
      cdf = (double*)malloc(r_rows * sizeof(double));
      if (!cdf) return CJO_NOMEM;
      double acc = 0.0;
      for (uint64_t k = 0; k < r_rows; ++k) {
        acc += pow((double)(k + 1), -zipf);
        cdf[k] = acc;
      }
      const double norm = 1.0 / acc;
      for (uint64_t k = 0; k < r_rows; ++k) cdf[k] *= norm;
      cdf[r_rows - 1] = 1.0;
      rank_to_key = permutation(r_rows, rng_stream(master, 0x53000001ull));
      if (!rank_to_key) { free(cdf); return CJO_NOMEM; }
    }
    for (uint64_t j = 0; j < s_rows; ++j) {
      const double u = rng_u01(zr, j);
      uint64_t rank;
      if (!cdf) {
        rank = (uint64_t)(u * (double)r_rows);
        if (rank >= r_rows) rank = r_rows - 1;
      } else {
        /* std::upper_bound: first cdf[k] > u */
        uint64_t lo = 0, hi = r_rows;
        while (lo < hi) {
          const uint64_t mid = lo + (hi - lo) / 2;
          if (cdf[mid] > u) hi = mid; else lo = mid + 1;
        }
        rank = lo == r_rows ? r_rows - 1 : lo;
      }
      s_key[j] = rank_to_key ? rank_to_key[rank] : rank;
    }
    free(cdf);
    free(rank_to_key);
  } else {
    memset(s_key, 0, s_rows * sizeof(uint64_t));
  }

  /* workloads.cpp:113-120 displace non-matching primary keys */
  const uint64_t keep = (uint64_t)llround(match_ratio * (double)r_rows);
  if (keep < r_rows)
    for (uint64_t i = 0; i < r_rows; ++i)
      if (r_key[i] >= keep) r_key[i] += r_rows;

  /* workloads.cpp:124-129 payload streams 0x7000+c / 0x8000+c */
  for (unsigned c = 0; c < r_pay; ++c) {
    const rng_t pr = rng_stream(master, 0x7000ull + c);
    for (uint64_t i = 0; i < r_rows; ++i) {
      const uint64_t v = rng_at(pr, i);
      r_pay_cols[(uint64_t)c * r_rows + i] = pay_bytes == 4 ? (uint32_t)v : v;
    }
  }
  for (unsigned c = 0; c < s_pay; ++c) {
    const rng_t pr = rng_stream(master, 0x8000ull + c);
    for (uint64_t i = 0; i < s_rows; ++i) {
      const uint64_t v = rng_at(pr, i);
      s_pay_cols[(uint64_t)c * s_rows + i] = pay_bytes == 4 ? (uint32_t)v : v;
    }
  }
  return CJO_OK;
}

/* task.hpp:45-50 */
unsigned cjo_default_total_radix_bits(uint64_t build_rows) {
  if (build_rows > (1ull << 20)) return 16;
  unsigned bits = 0;
  while ((build_rows >> bits) > 1024) ++bits;
  return bits > 16 ? 16 : bits;
}

/* primitives.cpp:25-30 */
static int check_bit_range(unsigned lo, unsigned hi, unsigned key_bits) {
  if (hi < lo || hi - lo > 8) return CJO_FANOUT_TOO_LARGE;
  if (hi > key_bits) return CJO_FANOUT_TOO_LARGE;
  return CJO_OK;
}

/* reference.cpp:8-26 stable counting sort by the digit in [lo, hi); the
 * parallel form (primitives.cpp:33-114) is output-identical by construction. */
static int stable_pass(const uint64_t* keys, const uint64_t* vals, unsigned nvals,
                       uint64_t n, unsigned lo, unsigned hi, uint64_t* ko, uint64_t* vo,
                       uint64_t* offsets) {
  const uint64_t fanout = 1ull << (hi - lo);
  const uint64_t mask = fanout - 1;
  uint64_t* cursor = (uint64_t*)calloc(fanout + 1, sizeof(uint64_t));
  if (!cursor) return CJO_NOMEM;
  for (uint64_t i = 0; i < n; ++i) ++cursor[((keys[i] >> lo) & mask) + 1];
  for (uint64_t d = 1; d <= fanout; ++d) cursor[d] += cursor[d - 1];
  if (offsets) memcpy(offsets, cursor, (fanout + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t pos = cursor[(keys[i] >> lo) & mask]++;
    ko[pos] = keys[i];
    for (unsigned c = 0; c < nvals; ++c) vo[(uint64_t)c * n + pos] = vals[(uint64_t)c * n + i];
  }
  free(cursor);
  return CJO_OK;
}

int cjo_radix_partition(const uint64_t* keys, const uint64_t* vals, unsigned nvals,
                        uint64_t n, unsigned key_bytes, unsigned lo, unsigned hi,
                        uint64_t* keys_out, uint64_t* vals_out, uint64_t* offsets) {
  int st = check_bit_range(lo, hi, key_bytes * 8);
  if (st) return st;
  if (lo == hi) { /* primitives.cpp:300-305: fan-out 1 is the identity */
    memcpy(keys_out, keys, n * sizeof(uint64_t));
    if (nvals) memcpy(vals_out, vals, (uint64_t)nvals * n * sizeof(uint64_t));
    if (offsets) { offsets[0] = 0; offsets[1] = n; }
    return CJO_OK;
  }
  return stable_pass(keys, vals, nvals, n, lo, hi, keys_out, vals_out, offsets);
}

/* primitives.cpp:169-256: digit totals, skip constant-digit passes, LSD
 * ping-pong.  Skipping never changes the output (a constant digit's stable
 * pass is the identity), so this restatement simply runs the live passes. */
int cjo_radix_partition_passes(const uint64_t* keys, const uint64_t* vals, unsigned nvals,
                               uint64_t n, unsigned key_bytes, const unsigned* plan_lo,
                               const unsigned* plan_hi, unsigned npasses,
                               uint64_t* keys_out, uint64_t* vals_out) {
  for (unsigned p = 0; p < npasses; ++p) {
    int st = check_bit_range(plan_lo[p], plan_hi[p], key_bytes * 8);
    if (st) return st;
  }
  memcpy(keys_out, keys, n * sizeof(uint64_t));
  if (nvals) memcpy(vals_out, vals, (uint64_t)nvals * n * sizeof(uint64_t));
  uint64_t* tk = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  uint64_t* tv = (uint64_t*)malloc(((uint64_t)nvals * n + 1) * sizeof(uint64_t));
  if (!tk || !tv) { free(tk); free(tv); return CJO_NOMEM; }
  for (unsigned p = 0; p < npasses; ++p) {
    const unsigned lo = plan_lo[p], hi = plan_hi[p];
    if (lo == hi) continue;
    /* single_digit (primitives.cpp:207-212): a digit holding all n keys */
    const uint64_t mask = (1ull << (hi - lo)) - 1;
    int constant = 1;
    for (uint64_t i = 1; i < n; ++i)
      if (((keys_out[i] >> lo) & mask) != ((keys_out[0] >> lo) & mask)) { constant = 0; break; }
    if (constant) continue;
    int st = stable_pass(keys_out, vals_out, nvals, n, lo, hi, tk, tv, NULL);
    if (st) { free(tk); free(tv); return st; }
    memcpy(keys_out, tk, n * sizeof(uint64_t));
    if (nvals) memcpy(vals_out, tv, (uint64_t)nvals * n * sizeof(uint64_t));
  }
  free(tk);
  free(tv);
  return CJO_OK;
}

/* primitives.cpp:258-261 + 358-362 */
int cjo_sort_pairs(const uint64_t* keys, const uint64_t* vals, unsigned nvals, uint64_t n,
                   unsigned key_bytes, uint64_t* keys_out, uint64_t* vals_out) {
  unsigned lo[8], hi[8], np = 0;
  for (unsigned b = 0; b < key_bytes * 8; b += 8, ++np) { lo[np] = b; hi[np] = b + 8; }
  return cjo_radix_partition_passes(keys, vals, nvals, n, key_bytes, lo, hi, np, keys_out,
                                    vals_out);
}

/* hash_match.cpp:30-69 + 140-158 */
int cjo_partition_relation(const uint64_t* keys, const uint64_t* vals, unsigned nvals,
                           uint64_t n, unsigned key_bytes, unsigned total_bits,
                           unsigned bits_per_pass, uint64_t* keys_out, uint64_t* vals_out,
                           uint64_t* offsets) {
  if (total_bits > 20 || total_bits > key_bytes * 8) return CJO_FANOUT_TOO_LARGE;
  if (total_bits == 0) {
    memcpy(keys_out, keys, n * sizeof(uint64_t));
    if (nvals) memcpy(vals_out, vals, (uint64_t)nvals * n * sizeof(uint64_t));
    if (offsets) { offsets[0] = 0; offsets[1] = n; }
    return CJO_OK;
  }
  if (bits_per_pass == 0 || bits_per_pass > 8) return CJO_FANOUT_TOO_LARGE; /* task.hpp:56 */
  unsigned lo[24], hi[24], np = 0;
  for (unsigned b = 0; b < total_bits; b += bits_per_pass, ++np) {
    lo[np] = b;
    hi[np] = b + bits_per_pass < total_bits ? b + bits_per_pass : total_bits;
  }
  int st = cjo_radix_partition_passes(keys, vals, nvals, n, key_bytes, lo, hi, np, keys_out,
                                      vals_out);
  if (st) return st;
  if (offsets) { /* wide_offsets: joint histogram of the low bits */
    const uint64_t fanout = 1ull << total_bits;
    memset(offsets, 0, (fanout + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) ++offsets[(keys_out[i] & (fanout - 1)) + 1];
    for (uint64_t d = 1; d <= fanout; ++d) offsets[d] += offsets[d - 1];
  }
  return CJO_OK;
}

/* primitives.cpp:369-396 */
int cjo_gather(const uint64_t* in, uint64_t n_in, const uint32_t* map, uint64_t m,
               uint64_t* out) {
  for (uint64_t i = 0; i < m; ++i) {
    if (map[i] >= n_in) return CJO_INDEX_OOB;
    out[i] = in[map[i]];
  }
  return CJO_OK;
}

/* hash_match.cpp:24-26 */
static uint64_t slot_of(uint64_t key, unsigned log2_cap) {
  return (key * GOLD) >> (64 - log2_cap);
}

/* hash_match.cpp:73-121 ChunkTable + scan_unit, and :186-302 plan/count/fill.
 * Emission order: (unit, probe position, build insertion order). */
static int hash_units(const uint64_t* bkeys, const uint64_t* boff, const uint64_t* pkeys,
                      const uint64_t* poff, unsigned fanout, uint32_t limit, uint64_t* total,
                      uint64_t* keys_out, uint32_t* ids_r, uint32_t* ids_s,
                      const uint32_t* bcarry, const uint32_t* pcarry) {
  if (limit == 0) return CJO_SPEC_INVALID;
  uint64_t cap_max = 2;
  while (cap_max < 2ull * limit) cap_max <<= 1;
  uint64_t* tkey = (uint64_t*)malloc(cap_max * sizeof(uint64_t));
  uint32_t* tpos = (uint32_t*)malloc(cap_max * sizeof(uint32_t));
  if (!tkey || !tpos) { free(tkey); free(tpos); return CJO_NOMEM; }
  uint64_t out = 0;
  for (unsigned p = 0; p < fanout; ++p) {
    const uint64_t b_lo = boff[p], b_hi = boff[p + 1];
    const uint64_t s_lo = poff[p], s_hi = poff[p + 1];
    if (b_hi == b_lo || s_hi == s_lo) continue;
    for (uint64_t c = b_lo; c < b_hi; c += limit) {
      const uint64_t c_hi = c + limit < b_hi ? c + limit : b_hi;
      const uint64_t n = c_hi - c;
      uint64_t cap = 2;
      while (cap < 2 * n) cap <<= 1;
      unsigned log2cap = 0;
      while ((1ull << log2cap) < cap) ++log2cap;
      const uint64_t mask = cap - 1;
      for (uint64_t s = 0; s < cap; ++s) tpos[s] = UINT32_MAX;
      for (uint64_t i = c; i < c_hi; ++i) {
        uint64_t s = slot_of(bkeys[i], log2cap);
        while (tpos[s] != UINT32_MAX) s = (s + 1) & mask;
        tkey[s] = bkeys[i];
        tpos[s] = (uint32_t)(i - c);
      }
      for (uint64_t j = s_lo; j < s_hi; ++j) {
        const uint64_t k = pkeys[j];
        uint64_t s = slot_of(k, log2cap);
        while (tpos[s] != UINT32_MAX) {
          if (tkey[s] == k) {
            if (keys_out) {
              const uint64_t i = c + tpos[s];
              keys_out[out] = k;
              ids_r[out] = bcarry ? bcarry[i] : (uint32_t)i;
              ids_s[out] = pcarry ? pcarry[j] : (uint32_t)j;
            }
            ++out;
          }
          s = (s + 1) & mask;
        }
      }
    }
  }
  free(tkey);
  free(tpos);
  *total = out;
  return CJO_OK;
}

int cjo_hash_find_matches(const uint64_t* bkeys, const uint64_t* boff, uint64_t nb,
                          const uint64_t* pkeys, const uint64_t* poff, uint64_t np,
                          unsigned fanout, uint32_t limit, uint64_t* total,
                          uint64_t* keys_out, uint32_t* ids_r, uint32_t* ids_s) {
  (void)nb;
  (void)np;
  return hash_units(bkeys, boff, pkeys, poff, fanout, limit, total, keys_out, ids_r, ids_s,
                    NULL, NULL);
}

/* merge_match.cpp:53-71 walk_part with a single part (output is invariant in
 * the part count, merge_match.hpp:47-52). */
int cjo_merge_find_matches(const uint64_t* r, uint64_t nr, const uint64_t* s, uint64_t ns,
                           int pk_fk, uint64_t* total, uint64_t* keys_out,
                           uint32_t* ids_r, uint32_t* ids_s) {
  uint64_t out = 0;
  if (ns > 0) {
    uint64_t lo = 0, hi = nr; /* std::lower_bound(r, s[0]) */
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo) / 2;
      if (r[mid] < s[0]) lo = mid + 1; else hi = mid;
    }
    uint64_t cur = lo;
    for (uint64_t j = 0; j < ns; ++j) {
      const uint64_t key = s[j];
      while (cur < nr && r[cur] < key) ++cur;
      if (cur >= nr) break;
      if (r[cur] != key) continue;
      for (uint64_t i = cur; i < nr && r[i] == key; ++i) {
        if (keys_out) { keys_out[out] = key; ids_r[out] = (uint32_t)i; ids_s[out] = (uint32_t)j; }
        ++out;
        if (pk_fk) break;
      }
    }
  }
  *total = out;
  return CJO_OK;
}

/* join_engine.cpp:52-113 transform_side for one relation. */
typedef struct {
  uint64_t* keys;
  uint64_t* carried; /* ids (GFUR) or payload 0 (GFTR) or NULL */
  uint64_t* offsets; /* PHJ layout */
} side_t;

static int transform(int algo, const uint64_t* key, const uint64_t* carried_in, uint64_t n,
                     unsigned key_bytes, unsigned total_bits, side_t* out) {
  out->keys = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  out->carried = carried_in ? (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t)) : NULL;
  out->offsets = algo == 1 ? (uint64_t*)malloc(((1ull << total_bits) + 1) * sizeof(uint64_t))
                           : NULL;
  if (!out->keys || (carried_in && !out->carried) || (algo == 1 && !out->offsets))
    return CJO_NOMEM;
  if (algo == 0)
    return cjo_sort_pairs(key, carried_in, carried_in ? 1 : 0, n, key_bytes, out->keys,
                          out->carried);
  return cjo_partition_relation(key, carried_in, carried_in ? 1 : 0, n, key_bytes, total_bits,
                                8, out->keys, out->carried, out->offsets);
}

static void side_free(side_t* s) {
  free(s->keys);
  free(s->carried);
  free(s->offsets);
}

/* join_engine.cpp:255-361 run_join (+ materialize_gfur :161-176,
 * materialize_gftr :180-253). */
int cjo_run_join(int algo, int pattern, const uint64_t* r_key, const uint64_t* r_pay,
                 unsigned r_npay, uint64_t nr, int r_key_unique, const uint64_t* s_key,
                 const uint64_t* s_pay, unsigned s_npay, uint64_t ns, unsigned key_bytes,
                 int total_bits_opt, uint32_t limit, uint64_t* rows_out, uint64_t* out_key,
                 uint64_t* out_pay, uint32_t* ids_r_out, uint32_t* ids_s_out) {
  const unsigned total_bits = total_bits_opt >= 0 ? (unsigned)total_bits_opt
                                                  : cjo_default_total_radix_bits(nr);
  const int gfur = pattern == 0;
  uint64_t* iota_r = NULL;
  uint64_t* iota_s = NULL;
  const uint64_t* carry_r = NULL;
  const uint64_t* carry_s = NULL;
  int st = CJO_OK;
  if (gfur) {
    iota_r = (uint64_t*)malloc((nr ? nr : 1) * sizeof(uint64_t));
    iota_s = (uint64_t*)malloc((ns ? ns : 1) * sizeof(uint64_t));
    if (!iota_r || !iota_s) { free(iota_r); free(iota_s); return CJO_NOMEM; }
    for (uint64_t i = 0; i < nr; ++i) iota_r[i] = i;
    for (uint64_t i = 0; i < ns; ++i) iota_s[i] = i;
    carry_r = iota_r;
    carry_s = iota_s;
  } else {
    carry_r = r_npay ? r_pay : NULL;
    carry_s = s_npay ? s_pay : NULL;
  }
  side_t tr = {0}, ts = {0};
  st = transform(algo, r_key, carry_r, nr, key_bytes, total_bits, &tr);
  if (!st) st = transform(algo, s_key, carry_s, ns, key_bytes, total_bits, &ts);
  uint64_t total = 0;
  uint64_t* mkeys = NULL;
  uint32_t* ids_r = NULL;
  uint32_t* ids_s = NULL;
  uint32_t* cr32 = NULL;
  uint32_t* cs32 = NULL;
  if (!st) {
    if (algo == 0) {
      st = cjo_merge_find_matches(tr.keys, nr, ts.keys, ns, r_key_unique, &total, NULL, NULL,
                                  NULL);
    } else {
      st = hash_units(tr.keys, tr.offsets, ts.keys, ts.offsets, 1u << total_bits, limit,
                      &total, NULL, NULL, NULL, NULL, NULL);
    }
  }
  if (!st && out_key) {
    mkeys = (uint64_t*)malloc((total ? total : 1) * sizeof(uint64_t));
    ids_r = (uint32_t*)malloc((total ? total : 1) * sizeof(uint32_t));
    ids_s = (uint32_t*)malloc((total ? total : 1) * sizeof(uint32_t));
    if (!mkeys || !ids_r || !ids_s) st = CJO_NOMEM;
    if (!st && gfur) {
      cr32 = (uint32_t*)malloc((nr ? nr : 1) * sizeof(uint32_t));
      cs32 = (uint32_t*)malloc((ns ? ns : 1) * sizeof(uint32_t));
      if (!cr32 || !cs32) st = CJO_NOMEM;
      for (uint64_t i = 0; !st && i < nr; ++i) cr32[i] = (uint32_t)tr.carried[i];
      for (uint64_t i = 0; !st && i < ns; ++i) cs32[i] = (uint32_t)ts.carried[i];
    }
    if (!st) {
      uint64_t t2 = 0;
      if (algo == 0) {
        st = cjo_merge_find_matches(tr.keys, nr, ts.keys, ns, r_key_unique, &t2, mkeys, ids_r,
                                    ids_s);
        if (gfur) { /* resolve_ids, join_engine.cpp:37-45 */
          for (uint64_t o = 0; o < total; ++o) {
            ids_r[o] = cr32[ids_r[o]];
            ids_s[o] = cs32[ids_s[o]];
          }
        }
      } else {
        st = hash_units(tr.keys, tr.offsets, ts.keys, ts.offsets, 1u << total_bits, limit, &t2,
                        mkeys, ids_r, ids_s, gfur ? cr32 : NULL, gfur ? cs32 : NULL);
      }
    }
    if (!st) {
      memcpy(out_key, mkeys, total * sizeof(uint64_t));
      /* materialise */
      const unsigned npay = r_npay + s_npay;
      for (unsigned c = 0; c < npay && !st; ++c) {
        const int is_r = c < r_npay;
        const unsigned cc = is_r ? c : c - r_npay;
        const uint64_t n = is_r ? nr : ns;
        const uint32_t* ids = is_r ? ids_r : ids_s;
        const uint64_t* src_col = (is_r ? r_pay : s_pay) + (uint64_t)cc * n;
        uint64_t* dst = out_pay + (uint64_t)c * total;
        if (gfur) {
          st = cjo_gather(src_col, n, ids, total, dst);
        } else if (cc == 0) {
          st = cjo_gather(is_r ? tr.carried : ts.carried, n, ids, total, dst);
        } else { /* on-demand transform of (key, p_c), join_engine.cpp:180-213 */
          side_t t = {0};
          st = transform(algo, is_r ? r_key : s_key, src_col, n, key_bytes, total_bits, &t);
          if (!st) st = cjo_gather(t.carried, n, ids, total, dst);
          side_free(&t);
        }
      }
      if (ids_r_out) memcpy(ids_r_out, ids_r, total * sizeof(uint32_t));
      if (ids_s_out) memcpy(ids_s_out, ids_s, total * sizeof(uint32_t));
    }
  }
  *rows_out = total;
  free(mkeys); free(ids_r); free(ids_s); free(cr32); free(cs32);
  free(iota_r); free(iota_s);
  side_free(&tr);
  side_free(&ts);
  return st;
}

/* ---- oracle.cpp:21-37, 77-88 canonical rows ----------------------------- */
static unsigned g_width;
static const uint64_t* g_flat;
static int row_cmp(const void* a, const void* b) {
  const uint64_t* ra = g_flat + (uint64_t)(*(const uint64_t*)a) * g_width;
  const uint64_t* rb = g_flat + (uint64_t)(*(const uint64_t*)b) * g_width;
  for (unsigned c = 0; c < g_width; ++c) {
    if (ra[c] < rb[c]) return -1;
    if (ra[c] > rb[c]) return 1;
  }
  return 0;
}

static uint64_t digest_sorted_rows(uint64_t* flat, unsigned width, uint64_t nrows) {
  uint64_t* order = (uint64_t*)malloc((nrows ? nrows : 1) * sizeof(uint64_t));
  if (!order) return 0;
  for (uint64_t i = 0; i < nrows; ++i) order[i] = i;
  g_width = width;
  g_flat = flat;
  qsort(order, nrows, sizeof(uint64_t), row_cmp);
  uint64_t h = 0x12345678ull, idx = 0;
  for (uint64_t i = 0; i < nrows; ++i) {
    const uint64_t* row = flat + order[i] * width;
    for (unsigned c = 0; c < width; ++c, ++idx) h = cjo_mix64(h ^ row[c]) + idx;
  }
  free(order);
  return h;
}

uint64_t cjo_canonical_digest(const uint64_t* const* cols, unsigned ncols, uint64_t nrows) {
  uint64_t* flat = (uint64_t*)malloc((nrows * ncols + 1) * sizeof(uint64_t));
  if (!flat) return 0;
  for (uint64_t i = 0; i < nrows; ++i)
    for (unsigned c = 0; c < ncols; ++c) flat[i * ncols + c] = cols[c][i];
  const uint64_t h = digest_sorted_rows(flat, ncols, nrows);
  free(flat);
  return h;
}

/* oracle.cpp:41-75 */
int cjo_nested_loop_join(const uint64_t* r_key, const uint64_t* r_pay, unsigned r_npay,
                         uint64_t nr, const uint64_t* s_key, const uint64_t* s_pay,
                         unsigned s_npay, uint64_t ns, uint64_t* rows_out,
                         uint64_t* out_rows) {
  uint64_t count = 0;
  const unsigned width = 1 + r_npay + s_npay;
  for (uint64_t i = 0; i < nr; ++i)
    for (uint64_t j = 0; j < ns; ++j)
      if (s_key[j] == r_key[i]) {
        if (out_rows) {
          uint64_t* row = out_rows + count * width;
          row[0] = r_key[i];
          for (unsigned c = 0; c < r_npay; ++c) row[1 + c] = r_pay[(uint64_t)c * nr + i];
          for (unsigned c = 0; c < s_npay; ++c)
            row[1 + r_npay + c] = s_pay[(uint64_t)c * ns + j];
        }
        ++count;
      }
  if (out_rows && count > 1) {
    uint64_t* order = (uint64_t*)malloc(count * sizeof(uint64_t));
    uint64_t* tmp = (uint64_t*)malloc(count * width * sizeof(uint64_t));
    if (!order || !tmp) { free(order); free(tmp); return CJO_NOMEM; }
    for (uint64_t i = 0; i < count; ++i) order[i] = i;
    g_width = width;
    g_flat = out_rows;
    qsort(order, count, sizeof(uint64_t), row_cmp);
    for (uint64_t i = 0; i < count; ++i)
      memcpy(tmp + i * width, out_rows + order[i] * width, width * sizeof(uint64_t));
    memcpy(out_rows, tmp, count * width * sizeof(uint64_t));
    free(order);
    free(tmp);
  }
  *rows_out = count;
  return CJO_OK;
}
