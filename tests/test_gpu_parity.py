"""GPU parity: the sm_100a kernels (through the C-ABI) against the C
restatement of the reference (oracle/, pinned to the reference by
tests/test_oracle_golden.py).  Integer work: every comparison is bit-exact,
including the emission order of the join output."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.cells import cell_id, make_cell

pytestmark = pytest.mark.gpu

cj = pytest.importorskip("paper_2312_00720_b200")


@pytest.fixture(scope="module")
def ctx():
    c = cj.Context(0)
    yield c
    c.close()


def rng_cols(n, seed, kb=4, dup=None):
    g = np.random.default_rng(seed)
    if dup:
        k = g.integers(0, dup, n, dtype=np.uint64)
    else:
        k = g.integers(0, 2 ** 63, n, dtype=np.uint64) >> g.integers(0, 40, n, dtype=np.uint64)
    k = k.astype(np.uint32 if kb == 4 else np.uint64)
    v4 = g.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    v8 = g.integers(0, 2 ** 63, n, dtype=np.uint64)
    return k, v4, v8


def H(t):
    return cj.to_host(t).astype(np.uint64)


SIZES = [0, 1, 33, 4095, 4096, 4097, 100_003]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("kb,lo,hi", [(4, 0, 8), (4, 3, 11), (4, 24, 32), (4, 0, 3), (8, 56, 64),
                                      (8, 20, 28), (4, 5, 5)])
def test_radix_partition(ctx, n, kb, lo, hi):
    k, v4, v8 = rng_cols(n, n + lo, kb, dup=None if n % 2 else 50)
    ko, vo, off = cj.radix_partition(ctx, cj.to_device(k), [cj.to_device(v4), cj.to_device(v8)],
                                     lo, hi)
    ek, (e4, e8), eoff = O.radix_partition(k, [v4, v8], lo, hi, key_bytes=kb)
    assert np.array_equal(H(ko), ek)
    assert np.array_equal(H(vo[0]), e4)
    assert np.array_equal(H(vo[1]), e8)
    assert np.array_equal(off, eoff[: off.size])


def test_radix_partition_known_answer(ctx):
    # tests/test_primitives.cpp:25-34
    ko, (vo,), off = cj.radix_partition(ctx, cj.to_device(np.array([5, 2, 7, 0], np.uint32)),
                                        [cj.to_device(np.array([10, 20, 30, 40], np.uint32))], 0, 1)
    assert list(H(ko)) == [2, 0, 5, 7] and list(H(vo)) == [20, 40, 10, 30]
    assert list(off) == [0, 2, 4]


def test_radix_partition_errors(ctx):
    k = cj.to_device(np.array([1, 2], np.uint32))
    with pytest.raises(cj.FanoutTooLarge):
        cj.radix_partition(ctx, k, [k], 0, 9)
    with pytest.raises(cj.FanoutTooLarge):
        cj.radix_partition(ctx, k, [k], 30, 36)
    with pytest.raises(cj.LengthMismatch):
        cj.radix_partition(ctx, k, [cj.to_device(np.array([1], np.uint32))], 0, 1)


@pytest.mark.parametrize("n", [0, 1, 4097, 65_536, 300_001])
@pytest.mark.parametrize("kb,dup", [(4, None), (4, 13), (8, None), (8, 7)])
def test_sort_pairs(ctx, n, kb, dup):
    k, v4, v8 = rng_cols(n, 7 * n + kb, kb, dup)
    ko, vo = cj.sort_pairs(ctx, cj.to_device(k), [cj.to_device(v4), cj.to_device(v8)])
    ek, (e4, e8) = O.sort_pairs(k, [v4, v8], key_bytes=kb)
    assert np.array_equal(H(ko), ek)
    assert np.array_equal(H(vo[0]), e4) and np.array_equal(H(vo[1]), e8)


def test_sort_pairs_gen_ids_stable(ctx):
    k, _, _ = rng_cols(50_000, 3, 4, dup=7)
    ko, (ids,) = cj.sort_pairs(ctx, cj.to_device(k), [], gen_ids=True)
    ek, (eids,) = O.sort_pairs(k, [np.arange(k.size, dtype=np.uint32)])
    assert np.array_equal(H(ko), ek) and np.array_equal(H(ids), eids)


@pytest.mark.parametrize("n,kb,bits,per", [(100_000, 4, 16, 8), (100_000, 8, 13, 5),
                                           (5000, 4, 10, 8), (70_000, 4, 20, 7), (0, 4, 16, 8),
                                           (1000, 4, 0, 8)])
def test_partition_relation(ctx, n, kb, bits, per):
    k, v4, v8 = rng_cols(n, bits * 31 + n, kb)
    ko, vo, off = cj.partition_relation(ctx, cj.to_device(k), [cj.to_device(v4), cj.to_device(v8)],
                                        bits, per)
    ek, (e4, e8), eoff = O.partition_relation(k, [v4, v8], bits, per, key_bytes=kb)
    assert np.array_equal(H(ko), ek)
    assert np.array_equal(H(vo[0]), e4) and np.array_equal(H(vo[1]), e8)
    assert np.array_equal(cj.to_host(off).astype(np.uint64), eoff)


@pytest.mark.parametrize("m", [0, 1, 10_000, 1_000_003])
def test_gather(ctx, m):
    g = np.random.default_rng(m)
    n = 50_000
    c4 = g.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    c8 = g.integers(0, 2 ** 63, n, dtype=np.uint64)
    idx = g.integers(0, n, m, dtype=np.uint64).astype(np.uint32)
    o4, o8 = cj.gather(ctx, [cj.to_device(c4), cj.to_device(c8)], cj.to_device(idx))
    assert np.array_equal(H(o4), O.gather(c4, idx)) and np.array_equal(H(o8), O.gather(c8, idx))


def test_gather_oob(ctx):
    c = cj.to_device(np.arange(10, dtype=np.uint32))
    with pytest.raises(cj.IndexOutOfBounds):
        cj.gather(ctx, [c], cj.to_device(np.array([1, 10], np.uint32)))


@pytest.mark.parametrize("kb,dup,limit,nb,np_", [(4, 97, 16, 2000, 2000), (4, None, 4096, 70_000, 140_000),
                                                 (8, 13, 64, 3000, 5000), (4, 5, 4096, 20_000, 9000),
                                                 (4, None, 1024, 300_000, 10_000)])
def test_hash_find_matches(ctx, kb, dup, limit, nb, np_):
    g = np.random.default_rng(nb + np_)
    if dup:
        bk = g.integers(0, dup, nb, dtype=np.uint64)
        pk = g.integers(0, dup + 3, np_, dtype=np.uint64)
    else:
        bk = g.permutation(nb).astype(np.uint64)
        pk = g.integers(0, nb * 2, np_, dtype=np.uint64)
    dt = np.uint32 if kb == 4 else np.uint64
    bk, pk = bk.astype(dt), pk.astype(dt)
    bits = 4 if dup else 10
    bko, _, boff = cj.partition_relation(ctx, cj.to_device(bk), [], bits)
    pko, _, poff = cj.partition_relation(ctx, cj.to_device(pk), [], bits)
    keys, ir, js = cj.hash_find_matches(ctx, bko, boff, pko, poff, limit)
    ebk, _, eboff = O.partition_relation(bk, [], bits, key_bytes=kb)
    epk, _, epoff = O.partition_relation(pk, [], bits, key_bytes=kb)
    ek, eir, ejs = O.hash_find_matches(ebk, eboff, epk, epoff, limit)
    assert np.array_equal(H(keys), ek)
    assert np.array_equal(cj.to_host(ir), eir) and np.array_equal(cj.to_host(js), ejs)


@pytest.mark.parametrize("kb,dup,pk_fk,nr,ns", [(4, None, True, 100_000, 300_000),
                                                (4, 50, False, 3000, 4000),
                                                (8, 9, False, 2000, 2000),
                                                (4, None, True, 10, 200_000),
                                                (4, None, True, 200_000, 10)])
def test_merge_find_matches(ctx, kb, dup, pk_fk, nr, ns):
    g = np.random.default_rng(nr * 3 + ns)
    if dup:
        r = np.sort(g.integers(0, dup, nr, dtype=np.uint64))
        s = np.sort(g.integers(0, dup + 5, ns, dtype=np.uint64))
    else:
        r = np.sort(g.permutation(nr * 2)[:nr].astype(np.uint64))
        s = np.sort(g.integers(0, nr * 2, ns, dtype=np.uint64))
    dt = np.uint32 if kb == 4 else np.uint64
    r, s = r.astype(dt), s.astype(dt)
    keys, ir, js = cj.merge_find_matches(ctx, cj.to_device(r), cj.to_device(s), pk_fk)
    ek, eir, ejs = O.merge_find_matches(r, s, pk_fk)
    assert np.array_equal(H(keys), ek)
    assert np.array_equal(cj.to_host(ir), eir) and np.array_equal(cj.to_host(js), ejs)


def test_merge_validation(ctx):
    r = cj.to_device(np.array([3, 1, 2], np.uint32))
    s = cj.to_device(np.array([1, 2], np.uint32))
    with pytest.raises(cj.NotSorted):
        cj.merge_find_matches(ctx, r, s, True, validate=True)
    with pytest.raises(cj.DuplicateBuildKeys):
        cj.merge_find_matches(ctx, cj.to_device(np.array([1, 1, 2], np.uint32)), s, True,
                              validate=True)


# ---- end to end -----------------------------------------------------------------

def _rows(golden):
    return [g for g in golden["join"] if g["cell"].get("name") != "C1"]


def _dev_rel(X, uniq, name):
    return cj.Relation(cj.to_device(X["key"]), [cj.to_device(p) for p in X["payloads"]], name, uniq)


def _load():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")) as f:
        return json.load(f)


_GOLD = _load()
_CELLS = []
for _g in _GOLD["join"]:
    if _g["cell"] not in _CELLS:
        _CELLS.append(_g["cell"])


@pytest.mark.parametrize("cell", _CELLS, ids=[cell_id(c) for c in _CELLS])
def test_run_join_matches_reference_exactly(ctx, cell):
    """Every variant: output columns equal the reference's (same emission order);
    the canonical digest equals the golden one recorded from the reference."""
    R, S, uniq = make_cell(cell)
    Rd, Sd = _dev_rel(R, uniq, "R"), _dev_rel(S, False, "S")
    digests = set()
    for g in [x for x in _GOLD["join"] if x["cell"] == cell]:
        out = cj.run_join(ctx, Rd, Sd, g["algo"], g["pattern"], want_stats=True)
        cols = [H(out.relation.key)] + [H(p) for p in out.relation.payloads]
        assert out.matches == g["rows_out"]
        if cell.get("name") != "C1":
            ref = O.run_join(R, S, g["algo"], g["pattern"], r_key_unique=uniq)
            for a, b in zip(cols, [ref["key"]] + ref["payloads"]):
                assert np.array_equal(a, b), (g["algo"], g["pattern"])
        else:
            flat = np.concatenate(cols)
            assert "%016x" % O.digest(flat) == g["order_digest"]
        d = "%016x" % O.canonical_digest(cols)
        assert d == g["digest"]
        digests.add(d)
        if out.matches > 1:
            assert abs(out.clusteredness_r - g["clusteredness_r"]) <= 1e-6 * max(1, g["clusteredness_r"])
            assert abs(out.clusteredness_s - g["clusteredness_s"]) <= 1e-6 * max(1, g["clusteredness_s"])
    # the non-partitioned hash join yields the same row multiset
    for pattern in ("gftr", "gfur"):
        out = cj.run_join(ctx, Rd, Sd, "nphj", pattern)
        cols = [H(out.relation.key)] + [H(p) for p in out.relation.payloads]
        assert "%016x" % O.canonical_digest(cols) in digests


def test_run_join_host_drop_in(ctx):
    R, S = O.gen_pk_fk(1 << 16, 1 << 17, 2, 2, seed=5)
    Rh = cj.Relation(R["key"], R["payloads"], "R", True)
    Sh = cj.Relation(S["key"], S["payloads"], "S", False)
    for algo in ("phj", "smj"):
        out, h2d, d2h = cj.run_join_host(ctx, Rh, Sh, algo, "gftr")
        ref = O.run_join(R, S, algo, "gftr")
        assert np.array_equal(out.relation.key.astype(np.uint64), ref["key"])
        for a, b in zip(out.relation.payloads, ref["payloads"]):
            assert np.array_equal(a.astype(np.uint64), b)
        assert h2d > 0 and d2h > 0


def test_run_join_errors(ctx):
    a = cj.Relation(cj.to_device(np.array([1, 2], np.uint32)), [], "a", True)
    b = cj.Relation(cj.to_device(np.array([1, 2], np.uint64)), [], "b")
    with pytest.raises(cj.KindError):
        cj.run_join(ctx, a, b)
    with pytest.raises(cj.FanoutTooLarge):
        cj.run_join(ctx, a, a, radix_bits_per_pass=9)
    with pytest.raises(cj.FanoutTooLarge):
        cj.run_join(ctx, a, a, total_radix_bits=21)


def test_empty_inputs_full_arity(ctx):
    # tests/test_engine.cpp:57-67
    e = cj.Relation(cj.to_device(np.zeros(0, np.uint32)), [cj.to_device(np.zeros(0, np.uint32))],
                    "e", True)
    for algo in ("phj", "smj", "nphj"):
        for pat in ("gftr", "gfur"):
            out = cj.run_join(ctx, e, e, algo, pat)
            assert out.matches == 0 and len(out.relation.payloads) == 2


@pytest.mark.parametrize("cell", [g["cell"] for g in _GOLD["gen"] if g["cell"].get("name") != "C2"],
                         ids=lambda c: cell_id(c))
def test_device_generator_matches_reference(ctx, cell):
    d = [g for g in _GOLD["gen"] if g["cell"] == cell][0]["digests"]
    widths = cell.get("widths")
    kb = 8 if cell["key"] == "u64" else 4
    pb = 8 if (cell["pay"] == "u64" or widths) else 4
    npay_r = len(widths.split(",")) if widths else cell["rpay"]
    npay_s = len(widths.split(",")) if widths else cell["spay"]
    R, S = cj.gen_pk_fk(ctx, cell["r"], cell["s"], npay_r, npay_s, kb, pb, cell["match"],
                        cell["zipf"], cell["seed"])
    ws = [int(w) for w in widths.split(",")] if widths else [pb] * max(npay_r, npay_s)

    def dg(t, w):
        a = cj.to_host(t)
        return "%016x" % O.digest(a.astype(np.uint32).astype(np.uint64) if w == 4 else a)

    assert dg(R.key, 8) == d["r_key"] and dg(S.key, 8) == d["s_key"]
    for i, p in enumerate(R.payloads):
        assert dg(p, ws[i]) == d[f"r_p{i}"]
    for i, p in enumerate(S.payloads):
        assert dg(p, ws[i]) == d[f"s_p{i}"]


def _skewed_keys(kind, n, kb, seed):
    """Key sets that defeat interpolation in the SMJ count pass's lower-bound
    guess: geometric gaps, values at both ends of the key range, long runs."""
    g = np.random.default_rng(seed)
    top = (1 << (8 * kb)) - 1
    if kind == "geometric":
        k = np.unique(np.minimum(np.exp(g.uniform(0, 8 * kb * np.log(2) - 1e-9, n)), top)
                      .astype(np.uint64))
    elif kind == "ends":
        lo = g.integers(0, 64, n // 2, dtype=np.uint64)
        hi = np.uint64(top) - g.integers(0, 64, n - n // 2, dtype=np.uint64)
        k = np.concatenate([lo, hi])
    else:  # runs: few distinct keys, long duplicate runs
        k = g.integers(0, 7, n, dtype=np.uint64) * np.uint64(top // 8)
    return k.astype(np.uint32 if kb == 4 else np.uint64)


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("kind", ["geometric", "ends", "runs"])
def test_smj_windows_with_skewed_key_gaps(ctx, kb, kind):
    """The count pass guesses each thread's first lower bound by interpolating
    between the window's end keys, then steps back and gallops; every key
    distribution must still give the reference's output exactly."""
    g = np.random.default_rng(7)
    rk = _skewed_keys(kind, 3000, kb, 1)
    uniq = kind != "runs"
    if uniq:
        rk = np.unique(rk)
        g.shuffle(rk)
    sk = np.concatenate([rk[g.integers(0, rk.size, 9000)], _skewed_keys(kind, 3000, kb, 2)])
    g.shuffle(sk)
    R = {"key": rk, "payloads": [g.integers(0, 2 ** 32, rk.size, dtype=np.uint64).astype(np.uint32)]}
    S = {"key": sk, "payloads": [g.integers(0, 2 ** 32, sk.size, dtype=np.uint64).astype(np.uint32)]}
    Rd = cj.Relation(cj.to_device(R["key"]), [cj.to_device(p) for p in R["payloads"]], "R", uniq)
    Sd = cj.Relation(cj.to_device(S["key"]), [cj.to_device(p) for p in S["payloads"]], "S", False)
    for pattern in ("gftr", "gfur"):
        out = cj.run_join(ctx, Rd, Sd, "smj", pattern)
        ref = O.run_join(R, S, "smj", pattern, r_key_unique=uniq)
        assert out.matches == ref["key"].size
        assert np.array_equal(H(out.relation.key), ref["key"])
        for a, b in zip(out.relation.payloads, ref["payloads"]):
            assert np.array_equal(H(a), b)


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("limit,bits", [(4096, -1), (512, 4), (97, 2)])
def test_phj_duplicate_builds_split_into_chunks(ctx, kb, limit, bits):
    """Duplicate-heavy builds whose partitions exceed the sub-partition limit
    (several build chunks per partition, duplicate-key tables, ragged last
    probe chunks) against the reference's emission order (C restatement)."""
    g = np.random.default_rng(11 + kb + limit)
    rk = (g.zipf(1.3, 5003) % 40).astype(np.uint64) * np.uint64(0x9E3779B1)
    sk = np.concatenate([rk[g.integers(0, rk.size, 7001)], g.integers(0, 2 ** 20, 999, dtype=np.uint64)])
    if kb == 4:
        rk, sk = rk.astype(np.uint32), sk.astype(np.uint32)
    g.shuffle(sk)
    R = {"key": rk, "payloads": [g.integers(0, 2 ** 32, rk.size, dtype=np.uint64).astype(np.uint32)]}
    S = {"key": sk, "payloads": [g.integers(0, 2 ** 63, sk.size, dtype=np.uint64)]}
    Rd = cj.Relation(cj.to_device(R["key"]), [cj.to_device(p) for p in R["payloads"]], "R", False)
    Sd = cj.Relation(cj.to_device(S["key"]), [cj.to_device(p) for p in S["payloads"]], "S", False)
    for pattern in ("gftr", "gfur"):
        out = cj.run_join(ctx, Rd, Sd, "phj", pattern, sub_partition_limit=limit,
                          total_radix_bits=bits)
        ref = O.run_join(R, S, "phj", pattern, total_bits=bits, limit=limit, r_key_unique=False)
        assert out.matches == ref["key"].size
        assert np.array_equal(H(out.relation.key), ref["key"])
        for a, b in zip(out.relation.payloads, ref["payloads"]):
            assert np.array_equal(H(a), b)
        # the non-partitioned hash join: same row multiset (its own order)
        nh = cj.run_join(ctx, Rd, Sd, "nphj", pattern)
        assert O.canonical_digest([H(nh.relation.key)] + [H(p) for p in nh.relation.payloads]) == \
            O.canonical_digest([ref["key"]] + ref["payloads"])


# ---- non-PK SMJ windows whose duplicates stand in for gaps ------------------------
# merge_match.cpp:53-71: a non-PK walk emits the whole r run of every probe key;
# a PK-FK walk (pk_fk = build.key_unique, join_engine.cpp:271) emits the lower bound.

def _smj_case(ctx, rk, sk, uniq, seed=0):
    g = np.random.default_rng(seed)
    R = {"key": rk, "payloads": [g.integers(0, 2 ** 32, rk.size, dtype=np.uint64).astype(np.uint32)]}
    S = {"key": sk, "payloads": [g.integers(0, 2 ** 63, sk.size, dtype=np.uint64)]}
    Rd, Sd = _dev_rel(R, uniq, "R"), _dev_rel(S, False, "S")
    for algo in ("smj", "phj"):
        for pattern in ("gftr", "gfur"):
            out = cj.run_join(ctx, Rd, Sd, algo, pattern)
            ref = O.run_join(R, S, algo, pattern, r_key_unique=uniq)
            assert out.matches == ref["key"].size, (algo, pattern)
            assert np.array_equal(H(out.relation.key), ref["key"]), (algo, pattern)
            for a, b in zip(out.relation.payloads, ref["payloads"]):
                assert np.array_equal(H(a), b), (algo, pattern)


@pytest.mark.parametrize("uniq", [False, True])
def test_smj_duplicates_in_place_of_gaps(ctx, uniq):
    """Build [5,5,7] |x| probe [5,6,7]: the window spans 7-5 = w-1 like a gap-free
    unique window.  Non-PK: (5,r0,s0),(5,r1,s0),(7,r2,s2).  Mislabelled unique
    (pk_fk without validation): the lower bound, (5,r0,s0),(7,r2,s2)."""
    rk = np.array([5, 5, 7], np.uint32)
    sk = np.array([5, 6, 7], np.uint32)
    _smj_case(ctx, rk, sk, uniq)
    R = {"key": rk, "payloads": [np.array([10, 11, 12], np.uint32)]}
    S = {"key": sk, "payloads": [np.array([20, 21, 22], np.uint32)]}
    out = cj.run_join(ctx, _dev_rel(R, uniq, "R"), _dev_rel(S, False, "S"), "smj", "gftr")
    want = ([5, 5, 7], [10, 11, 12], [20, 20, 22]) if not uniq else ([5, 7], [10, 12], [20, 22])
    assert list(H(out.relation.key)) == want[0]
    assert list(H(out.relation.payloads[0])) == want[1]
    assert list(H(out.relation.payloads[1])) == want[2]


@pytest.mark.parametrize("logn", [12, 14, 16, 18, 20])
@pytest.mark.parametrize("kb", [4, 8])
def test_smj_sparse_duplicate_builds(ctx, logn, kb):
    """Non-PK builds with about one row per key (uniform draws from [0, n)),
    probed by every key of [0, n) and some misses, in exact reference order."""
    n = 1 << logn
    g = np.random.default_rng(logn * 10 + kb)
    dt = np.uint32 if kb == 4 else np.uint64
    rk = g.integers(0, n, n, dtype=np.uint64).astype(dt)
    sk = np.concatenate([g.permutation(n).astype(np.uint64),
                         g.integers(n, 2 * n, n // 8, dtype=np.uint64)]).astype(dt)
    g.shuffle(sk)
    _smj_case(ctx, rk, sk, False, seed=logn)


@pytest.mark.parametrize("kb", [4, 8])
def test_smj_mislabelled_unique_build(ctx, kb):
    """A build declared unique that is not (no validation): every variant
    keeps the reference's PK-FK emission (one match per probe, the lower
    bound for SMJ, the first inserted for PHJ)."""
    n = 1 << 15
    g = np.random.default_rng(99 + kb)
    dt = np.uint32 if kb == 4 else np.uint64
    rk = g.integers(0, n, n, dtype=np.uint64).astype(dt)
    sk = g.permutation(n).astype(dt)
    _smj_case(ctx, rk, sk, True, seed=kb)


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("miss", ["none", "interior", "last"])
def test_pk_fk_speculation_misses(ctx, kb, miss):
    """PK-FK joins whose probe keys all match but for one key inside a merge
    tile (its first and last keys still match, so SMJ's tile-boundary check
    lets the speculative fill run and fail), or the largest probe key: the
    speculative one-pass fills (PHJ units, SMJ tiles) must fall back to count +
    fill and give the reference's rows in order."""
    n = 1 << 16
    g = np.random.default_rng(7 + kb)
    dt = np.uint32 if kb == 4 else np.uint64
    rk = (2 * g.permutation(n)).astype(dt)                  # unique even keys
    sk = np.repeat(np.arange(n, dtype=np.uint64) * 2, 2)    # every key twice
    if miss == "interior":
        sk[1001] = 1001  # sorted position ~1001 of a 2048-row tile: odd, absent
    elif miss == "last":
        sk[-1] = 2 * n + 1
    sk = sk.astype(dt)
    g.shuffle(sk)
    _smj_case(ctx, rk, sk, True, seed=kb)


# ---- MemLedger view of the device arena (mem_ledger.hpp:26-100) --------------
def dev_rel(X, uniq):
    return cj.Relation(cj.to_device(X["key"]), [cj.to_device(p) for p in X["payloads"]], "",
                       uniq)


# |R| = |S| = |T| = n at full match, 4-byte key + one 4-byte payload per side,
# M_c = 4n (one column).  This engine's closed forms:
#   GFUR: transform 4 M_c (keys + ids per side; the ids are born in the first
#         scatter pass, no iota column: the reference's 5th M_c),
#         find 6 M_c (+ the two id maps), materialise 2 M_c (the id maps);
#   GFTR: transform 4 M_c, find 4 M_c + 2 M_c when id maps are requested (the
#         fused find writes finished rows), materialise: the id maps only
#         (the transformed payloads were consumed by the fused find; the
#         reference's 4 M_c holds them until its gather).
@pytest.mark.parametrize("algo", ["phj", "smj"])
@pytest.mark.parametrize("rows", [4096, 65536])
def test_ledger_closed_forms(ctx, algo, rows):
    R, S = O.gen_pk_fk(rows, rows, 1, 1, seed=77)
    Rd, Sd = dev_rel(R, True), dev_rel(S, False)
    mc = rows * 4
    gfur = cj.run_join(ctx, Rd, Sd, algo, "gfur", want_ids=True).report
    assert gfur.column_bytes == (4 * mc, 6 * mc, 2 * mc)
    assert gfur.scratch_bytes[0] > 0
    gftr = cj.run_join(ctx, Rd, Sd, algo, "gftr", want_ids=True).report
    assert gftr.column_bytes == (4 * mc, 6 * mc, 2 * mc)
    plain = cj.run_join(ctx, Rd, Sd, algo, "gftr").report
    assert plain.column_bytes == (4 * mc, 4 * mc, 0)
    total = lambda r: max(c + s for c, s in zip(r.column_bytes, r.scratch_bytes))  # noqa: E731
    assert total(gftr) <= total(gfur)
    assert total(plain) <= total(gfur)


def test_ledger_zero_rows(ctx):
    e = np.zeros(0, np.uint32)
    Rd = cj.Relation(cj.to_device(e), [cj.to_device(e)], "R", True)
    Sd = cj.Relation(cj.to_device(e), [cj.to_device(e)], "S", False)
    out = cj.run_join(ctx, Rd, Sd, "phj", "gftr")
    assert out.report.column_bytes[0] == 0 and out.report.column_bytes[2] == 0


@pytest.mark.parametrize("algo_bits,limit", [(2, 4096), (4, 1024), (6, 4096)])
@pytest.mark.parametrize("pattern", ["gftr", "gfur"])
@pytest.mark.parametrize("match", [1.0, 0.6])
def test_phj_build_partitions_above_the_limit(ctx, algo_bits, limit, pattern, match):
    """Partitions holding more build rows than the sub-partition limit split into
    several build chunks (hash_match.cpp:186-210): every probe chunk meets every
    build chunk of its partition.  Exact rows and order against the oracle."""
    R, S = O.gen_pk_fk(1 << 16, 1 << 17, 2, 1, match=match, seed=31 + algo_bits)
    Rd = cj.Relation(cj.to_device(R["key"]), [cj.to_device(p) for p in R["payloads"]], "R", True)
    Sd = cj.Relation(cj.to_device(S["key"]), [cj.to_device(p) for p in S["payloads"]], "S", False)
    out = cj.run_join(ctx, Rd, Sd, "phj", pattern, total_radix_bits=algo_bits,
                      sub_partition_limit=limit)
    ref = O.run_join(R, S, "phj", pattern, total_bits=algo_bits, limit=limit)
    got = [H(out.relation.key)] + [H(p) for p in out.relation.payloads]
    want = [ref["key"]] + ref["payloads"]
    assert out.matches == len(ref["key"])
    for g, w in zip(got, want):
        assert np.array_equal(g, w.astype(np.uint64))
