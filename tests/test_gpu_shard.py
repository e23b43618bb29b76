"""Multi-GPU path on one device.

- the shard pass (cj_shard_partition_ex) is the stable send layout, grouped by
  (shard, low f key bits), for narrow and wide rows;
- the weak-scaling shard generator's slices form one workload;
- a presorted join (cj_run_join_presorted: first LSD pass skipped) gives
  run_join's rows in run_join's order on an input grouped by its low f bits;
- W = 2 / 4 / 8 simulated ranks: every rank's send layout, the library's
  exchange placement (cj_exchange_plan) and the presorted local joins give the
  single join's row multiset;
- the real NCCL path at world 1 (cj_run_join_sharded / cj_shuffle_relation
  over a one-rank communicator: shard pass, count and data exchange through
  ncclSend/ncclRecv to self, presorted join)."""
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


def host_digit(keys, parts, f):
    return (D.host_shard_of(keys, parts) << f) | (keys.astype(np.int64) & ((1 << f) - 1))


@pytest.mark.parametrize("parts,f", [(1, 0), (2, 0), (3, 0), (8, 0), (256, 0), (1, 6), (2, 5),
                                     (3, 6), (8, 5), (4, 6)])
@pytest.mark.parametrize("kb", [4, 8])
def test_shard_partition_is_the_stable_send_layout(ctx, parts, f, kb):
    g = np.random.default_rng(parts + kb + f)
    n = 100_003
    keys = g.integers(0, 2 ** (8 * kb - 1), n, dtype=np.uint64)
    keys = keys.astype(np.uint32 if kb == 4 else np.uint64)
    pay = g.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    rel = cj.Relation(cj.to_device(keys), [cj.to_device(pay)], "X", False)
    out, counts = D.shard_partition(ctx, rel, parts, f)
    digit = host_digit(keys, parts, f)
    assert np.array_equal(counts.ravel(), np.bincount(digit, minlength=parts << f))
    order = np.argsort(digit, kind="stable")
    assert np.array_equal(H(out.key), keys[order].astype(np.uint64))
    assert np.array_equal(H(out.payloads[0]), pay[order].astype(np.uint64))


def test_shard_partition_wide_rows_go_in_column_groups(ctx):
    """16 x 8-byte payloads (132-byte rows, more than one TMA stage holds): the
    column groups share one permutation."""
    g = np.random.default_rng(5)
    n = 50_001
    keys = g.integers(0, 2 ** 31, n, dtype=np.uint64).astype(np.uint32)
    pays = [g.integers(0, 2 ** 63, n, dtype=np.uint64) for _ in range(16)]
    rel = cj.Relation(cj.to_device(keys), [cj.to_device(p) for p in pays], "X", False)
    out, counts = D.shard_partition(ctx, rel, 4, 4)
    order = np.argsort(host_digit(keys, 4, 4), kind="stable")
    assert np.array_equal(H(out.key), keys[order].astype(np.uint64))
    for p, q in zip(pays, out.payloads):
        assert np.array_equal(H(q), p[order])


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


VARIANTS = [("phj", "gftr"), ("smj", "gftr"), ("phj", "gfur"), ("smj", "gfur"), ("nphj", "gftr")]


def first_bits(algo, world, total_bits=16):
    sb = max(0, (world - 1).bit_length())
    return {"phj": min(6, total_bits, 8 - sb), "smj": min(7, 8 - sb), "nphj": 0}[algo]


@pytest.mark.parametrize("f", [1, 5, 6])
@pytest.mark.parametrize("algo,pattern", VARIANTS)
def test_presorted_join_is_run_join(ctx, algo, pattern, f):
    """An input already stably grouped by its low f bits: skipping the first
    LSD pass gives exactly run_join's output, emission order included."""
    R, S = O.gen_pk_fk(1 << 14, 1 << 16, 2, 2, match=0.8, zipf=0.7, seed=11)

    def grouped(X, uniq):
        o = np.argsort(X["key"].astype(np.int64) & ((1 << f) - 1), kind="stable")
        return cj.Relation(cj.to_device(X["key"][o]), [cj.to_device(p[o]) for p in X["payloads"]],
                           "", uniq)
    Rg, Sg = grouped(R, True), grouped(S, False)
    kw = {"total_radix_bits": 10} if algo == "phj" else {}  # f <= the partition bits
    a = cj.run_join(ctx, Rg, Sg, algo, pattern, **kw)
    b = cj.run_join_presorted(ctx, Rg, Sg, f, algo, pattern, **kw)
    assert a.matches == b.matches
    for x, y in zip([a.relation.key] + a.relation.payloads, [b.relation.key] + b.relation.payloads):
        assert np.array_equal(H(x), H(y))


@pytest.mark.parametrize("world", [2, 4, 8])  # the generator needs |R|, |S| divisible by the ranks
@pytest.mark.parametrize("algo,pattern", VARIANTS)
def test_sharded_join_equals_single_join(ctx, world, algo, pattern):
    import torch
    nr, ns = 1 << 15, 1 << 17
    f = first_bits(algo, world, 11)
    slices = [D.gen_shard(ctx, nr, ns, r, world, 2, 2, 7) for r in range(world)]
    # every rank's send layout and run lengths [dst][digit]
    sent = [(D.shard_partition(ctx, R, world, f), D.shard_partition(ctx, S, world, f))
            for R, S in slices]

    def receive(side, d):
        """What destination d assembles: every source's runs at the library's
        cj_exchange_plan offsets (the NCCL receive placement)."""
        k = 0 if side == "R" else 1
        rc = np.stack([sent[src][k][1][d] for src in range(world)])
        _, ro, total = D.exchange_plan(sent[0][k][1], rc)
        proto = sent[0][k][0]
        cols = [torch.empty(total, dtype=c.dtype, device=c.device)
                for c in [proto.key] + list(proto.payloads)]
        for src in range(world):
            rel, sc = sent[src][k]
            so, _, _ = D.exchange_plan(sc, rc)
            for dg in range(1 << f):
                n = int(sc[d, dg])
                lo = int(so[d, dg])
                for c, col in enumerate([rel.key] + list(rel.payloads)):
                    cols[c][ro[src, dg]:ro[src, dg] + n] = col[lo:lo + n]
        # the copies run on torch's stream, the join on the library's
        torch.cuda.current_stream().synchronize()
        return cj.Relation(cols[0], cols[1:], side, side == "R")

    got = []
    for d in range(world):
        out = cj.run_join_presorted(ctx, receive("R", d), receive("S", d), f, algo, pattern,
                                    total_radix_bits=11 if algo == "phj" else -1)
        got.append([H(out.relation.key)] + [H(p) for p in out.relation.payloads])
    union = [np.concatenate([g[c] for g in got]) for c in range(len(got[0]))]
    cat = lambda xs: torch.cat(xs)  # noqa: E731
    Rall = cj.Relation(cat([R.key for R, _ in slices]),
                       [cat([R.payloads[c] for R, _ in slices]) for c in range(2)], "R", True)
    Sall = cj.Relation(cat([S.key for _, S in slices]),
                       [cat([S.payloads[c] for _, S in slices]) for c in range(2)], "S", False)
    torch.cuda.current_stream().synchronize()
    single = cj.run_join(ctx, Rall, Sall, algo, pattern)
    assert union[0].size == single.matches == ns
    assert O.canonical_digest(union) == O.canonical_digest(
        [H(single.relation.key)] + [H(p) for p in single.relation.payloads])


@pytest.fixture(scope="module")
def comm(ctx):
    c = D.Comm.single(ctx)
    yield c
    c.close()


@pytest.mark.parametrize("f", [0, 6])
@pytest.mark.parametrize("copy", [False, True])
def test_nccl_shuffle_world1_is_the_grouped_input(ctx, comm, f, copy):
    """World 1: the send layout is the received relation; with CJ_SHUFFLE_COPY=1
    the general path runs (own runs placed by the copy kernel at the
    cj_exchange_plan offsets), as every rank of a larger world does for its
    own shard."""
    if copy:
        import subprocess
        import sys
        code = (f"import sys; sys.argv=['x']; import tests.test_gpu_shard as T; "
                f"T._shuffle_check({f})")
        r = subprocess.run([sys.executable, "-c", code], env={**__import__("os").environ,
                           "CJ_SHUFFLE_COPY": "1"}, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        return
    _shuffle_check(f, ctx, comm)


def _shuffle_check(f, ctx=None, comm=None):
    if ctx is None:
        ctx = cj.Context(0)
        comm = D.Comm.single(ctx)
    g = np.random.default_rng(f)
    n = 70_001
    keys = g.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    pays = [g.integers(0, 2 ** 63, n, dtype=np.uint64), g.integers(0, 2 ** 32, n, dtype=np.uint64)
            .astype(np.uint32)]
    rel = cj.Relation(cj.to_device(keys), [cj.to_device(p) for p in pays], "X", False)
    st = {}
    out = D.shuffle(ctx, comm, rel, f, st)
    order = np.argsort(keys.astype(np.int64) & ((1 << f) - 1), kind="stable")
    assert np.array_equal(H(out.key), keys[order].astype(np.uint64))
    for p, q in zip(pays, out.payloads):
        assert np.array_equal(H(q), p[order].astype(np.uint64))
    assert st["r_rows_received"] == n and st["bytes_sent_peers"] == 0


@pytest.mark.parametrize("algo,pattern", VARIANTS)
def test_nccl_sharded_join_world1_matches_oracle(ctx, comm, algo, pattern):
    R, S = O.gen_pk_fk(1 << 13, 1 << 15, 2, 1, match=0.75, zipf=1.0, seed=4)
    Rd = cj.Relation(cj.to_device(R["key"]), [cj.to_device(p) for p in R["payloads"]], "R", True)
    Sd = cj.Relation(cj.to_device(S["key"]), [cj.to_device(p) for p in S["payloads"]], "S", False)
    t = {}
    out = D.distributed_join(ctx, Rd, Sd, algo, pattern, comm=comm, timings=t)
    ref = O.run_join(R, S, "phj", "gftr")
    assert out.matches == len(ref["key"])
    assert O.canonical_digest([H(out.relation.key)] + [H(p) for p in out.relation.payloads]) == \
        O.canonical_digest([ref["key"]] + ref["payloads"])
    assert t["r_rows_received"] == len(R["key"]) and t["s_rows_received"] == len(S["key"])


@pytest.mark.slow
def test_nccl_sharded_join_world1_c2_digest(ctx, comm):
    """C2 through the real NCCL path: the reference's canonical digest."""
    from tests.test_gpu_scale import C2_DIGEST, canonical_digest_device
    R, S = cj.gen_pk_fk(ctx, 1 << 27, 1 << 28, 2, 2, 4, 4, 1.0, 0.0, 42)
    for algo in ("phj", "smj"):
        out = D.distributed_join(ctx, R, S, algo, "gftr", comm=comm)
        assert out.matches == 1 << 28
        assert canonical_digest_device([out.relation.key] + list(out.relation.payloads)) == \
            C2_DIGEST
        del out


def test_cpp_sharded_run_join_world1(tmp_path):
    """coljoin::sharded::run_join (include/coljoin/sharded.hpp) — the C++ entry
    point a caller of the reference API uses — on a one-rank communicator
    gives coljoin::run_join's rows for PHJ/SMJ x GFTR/GFUR."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2312_00720_b200")
    exe = tmp_path / "sharded_world1"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "sharded_world1.cpp"), "-o", str(exe),
                    "-L", pkg, "-lcoljoin_host", "-lcoljoin_b200", f"-Wl,-rpath,{pkg}"],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    assert r.stdout.count(" ok") == 4


def test_nccl_sharded_join_wide_rows(ctx, comm):
    """C3-shaped rows (8-byte keys, [4,8,4,8] payloads + 12 more 8-byte columns
    on the probe side: wider than one shard-pass stage) through the sharded
    path: the shard pass runs in column groups; rows equal the single join's."""
    g = np.random.default_rng(21)
    nr, ns = 1 << 13, 1 << 15
    rk = g.permutation(np.arange(1, nr + 1, dtype=np.uint64) * 977)
    sk = rk[g.integers(0, nr, ns)]
    sk[::5] += 1  # some misses
    def cols(n, widths):
        return [g.integers(0, 2 ** 62, n, dtype=np.uint64).astype(np.uint32 if w == 4 else np.uint64)
                for w in widths]
    Rp, Sp = cols(nr, (4, 8, 4, 8)), cols(ns, (4, 8, 4, 8) + (8,) * 12)
    Rd = cj.Relation(cj.to_device(rk), [cj.to_device(p) for p in Rp], "R", True)
    Sd = cj.Relation(cj.to_device(sk), [cj.to_device(p) for p in Sp], "S", False)
    for algo in ("phj", "smj"):
        a = cj.run_join(ctx, Rd, Sd, algo, "gftr")
        b = D.distributed_join(ctx, Rd, Sd, algo, "gftr", comm=comm)
        assert a.matches == b.matches
        ca = [H(a.relation.key)] + [H(p) for p in a.relation.payloads]
        cb = [H(b.relation.key)] + [H(p) for p in b.relation.payloads]
        assert O.canonical_digest(ca) == O.canonical_digest(cb)
