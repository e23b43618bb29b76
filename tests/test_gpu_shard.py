"""Multi-GPU building blocks on one device: the shard
partition (the all-to-all send layout), the weak-scaling shard generator, and
the whole radix-sharded join with the exchange simulated in one process —
W "ranks" each shard their slice, the slices for destination d are
concatenated in rank order (what all_to_all_single delivers), and the union of
the per-destination joins must be the single-GPU join's row multiset."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

cj = pytest.importorskip("paper_2312_00720_b200")
from paper_2312_00720_b200 import distributed as D  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = cj.Context(0)
    yield c
    c.close()


def H(t):
    return cj.to_host(t).astype(np.uint64)


@pytest.mark.parametrize("parts", [1, 2, 3, 8, 256])
@pytest.mark.parametrize("kb", [4, 8])
def test_shard_partition_is_the_stable_send_layout(ctx, parts, kb):
    g = np.random.default_rng(parts + kb)
    n = 100_003
    keys = g.integers(0, 2 ** (8 * kb - 1), n, dtype=np.uint64)
    keys = keys.astype(np.uint32 if kb == 4 else np.uint64)
    pay = g.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    rel = cj.Relation(cj.to_device(keys), [cj.to_device(pay)], "X", False)
    out, counts = D.shard_partition(ctx, rel, parts)
    shard = D.host_shard_of(keys, parts)
    assert counts == np.bincount(shard, minlength=parts).tolist()
    order = np.argsort(shard, kind="stable")
    assert np.array_equal(H(out.key), keys[order].astype(np.uint64))
    assert np.array_equal(H(out.payloads[0]), pay[order].astype(np.uint64))


def test_gen_shard_slices_form_one_workload(ctx):
    ranks, nr, ns = 4, 1 << 16, 1 << 17
    rk, sk = [], []
    for r in range(ranks):
        R, S = D.gen_shard(ctx, nr, ns, r, ranks, 2, 2, 42)
        assert R.rows() == nr // ranks and S.rows() == ns // ranks
        rk.append(H(R.key))
        sk.append(H(S.key))
        again, _ = D.gen_shard(ctx, nr, ns, r, ranks, 2, 2, 42)
        assert np.array_equal(H(again.key), rk[-1])  # deterministic per rank
    allr = np.concatenate(rk)
    assert np.array_equal(np.sort(allr), np.arange(nr, dtype=np.uint64))  # a permutation
    assert np.concatenate(sk).max() < nr  # foreign keys inside the PK domain


@pytest.mark.parametrize("world", [2, 4])  # the generator needs |R|, |S| divisible by the ranks
@pytest.mark.parametrize("algo,pattern", [("phj", "gftr"), ("smj", "gftr"), ("phj", "gfur")])
def test_sharded_join_equals_single_join(ctx, world, algo, pattern):
    nr, ns = 1 << 15, 1 << 17
    slices = [D.gen_shard(ctx, nr, ns, r, world, 2, 2, 7) for r in range(world)]
    # every rank partitions its slices by destination shard
    sent = [(D.shard_partition(ctx, R, world), D.shard_partition(ctx, S, world))
            for R, S in slices]

    def receive(side, d):  # what destination d gets: its shard of every rank, in rank order
        cols = None
        for (rp, rc), (sp, sc) in sent:
            rel, counts = (rp, rc) if side == "R" else (sp, sc)
            lo = sum(counts[:d])
            part = [H(c)[lo:lo + counts[d]] for c in [rel.key] + list(rel.payloads)]
            cols = part if cols is None else [np.concatenate([a, b]) for a, b in zip(cols, part)]
        return [c.astype(np.uint32) for c in cols]

    got = []
    for d in range(world):
        rcols, scols = receive("R", d), receive("S", d)
        Rd = cj.Relation(cj.to_device(rcols[0]), [cj.to_device(c) for c in rcols[1:]], "R", True)
        Sd = cj.Relation(cj.to_device(scols[0]), [cj.to_device(c) for c in scols[1:]], "S", False)
        out = cj.run_join(ctx, Rd, Sd, algo, pattern)
        got.append([H(out.relation.key)] + [H(p) for p in out.relation.payloads])
    union = [np.concatenate([g[c] for g in got]) for c in range(len(got[0]))]
    Rall = cj.Relation(cj.to_device(np.concatenate([H(R.key) for R, _ in slices]).astype(np.uint32)),
                       [cj.to_device(np.concatenate([H(R.payloads[c]) for R, _ in slices])
                                     .astype(np.uint32)) for c in range(2)], "R", True)
    Sall = cj.Relation(cj.to_device(np.concatenate([H(S.key) for _, S in slices]).astype(np.uint32)),
                       [cj.to_device(np.concatenate([H(S.payloads[c]) for _, S in slices])
                                     .astype(np.uint32)) for c in range(2)], "S", False)
    single = cj.run_join(ctx, Rall, Sall, algo, pattern)
    assert union[0].size == single.matches == ns
    assert O.canonical_digest(union) == O.canonical_digest(
        [H(single.relation.key)] + [H(p) for p in single.relation.payloads])
