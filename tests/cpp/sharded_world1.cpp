// coljoin::sharded::run_join on a one-rank communicator (the C++ entry point of
// the multi-GPU path) against coljoin::run_join on the same task: the same row
// multiset for every algorithm and pattern.  Built and run by
// tests/test_gpu_shard.py (needs a GPU).
#include <algorithm>
#include <array>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#include "coljoin/join_engine.hpp"
#include "coljoin/sharded.hpp"

using namespace coljoin;

static std::vector<std::array<uint64_t, 4>> rows_of(const Relation& r) {
  std::vector<std::array<uint64_t, 4>> v(r.rows());
  for (size_t i = 0; i < r.rows(); ++i)
    v[i] = {r.key.at(i), r.payloads[0].at(i), r.payloads[1].at(i), r.payloads[2].at(i)};
  std::sort(v.begin(), v.end());
  return v;
}

int main() {
  const size_t nr = 1 << 14, ns = 1 << 16;
  std::mt19937_64 g(7);
  Column rk(ValueKind::u32, nr), rp(ValueKind::u32, nr), sk(ValueKind::u32, ns),
      sp(ValueKind::u64, ns), sq(ValueKind::u32, ns);
  std::vector<uint32_t> perm(nr);
  std::iota(perm.begin(), perm.end(), 1u);
  std::shuffle(perm.begin(), perm.end(), g);
  for (size_t i = 0; i < nr; ++i) {
    rk.u32()[i] = perm[i];
    rp.u32()[i] = (uint32_t)g();
  }
  for (size_t i = 0; i < ns; ++i) {
    sk.u32()[i] = 1 + (uint32_t)(g() % (nr + nr / 4));  // ~80% match
    sp.u64()[i] = g();
    sq.u32()[i] = (uint32_t)g();
  }
  Relation R = make_relation(rk, {rp}, "R", true);
  Relation S = make_relation(sk, {sp, sq}, "S");
  sharded::Comm comm(sharded::make_comm_id(), 1, 0);
  int bad = 0;
  for (auto algo : {JoinAlgo::PHJ, JoinAlgo::SMJ})
    for (auto pat : {JoinPattern::GFTR, JoinPattern::GFUR}) {
      JoinTask t;
      t.algorithm = algo;
      t.pattern = pat;
      t.build = &R;
      t.probe = &S;
      const JoinOutput a = run_join(t);
      sharded::ShuffleStats st;
      const JoinOutput b = sharded::run_join(t, comm, &st);
      const bool ok = rows_of(a.relation) == rows_of(b.relation) && st.r_rows_received == nr &&
                      st.s_rows_received == ns;
      std::printf("%s-%s rows %zu/%zu first_bits %u %s\n", algo == JoinAlgo::PHJ ? "PHJ" : "SMJ",
                  pat == JoinPattern::GFTR ? "GFTR" : "GFUR", a.relation.rows(), b.relation.rows(),
                  st.first_bits, ok ? "ok" : "MISMATCH");
      bad += !ok;
    }
  return bad ? 1 : 0;
}
