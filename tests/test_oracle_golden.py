"""Pins the C restatement (oracle/cj_oracle.c) to the unmodified reference.

The golden values were produced by oracle/_ref/refjoin (the reference library
compiled from /root/reference) via tests/golden/make_golden.py.  CPU only.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.cells import cell_id, make_cell


def _h(x):
    return "%016x" % x


def test_c1_digest_all_variants(golden):
    rows = [g for g in golden["join"] if g["cell"].get("name") == "C1"]
    assert len(rows) == 4
    R, S, uniq = make_cell(rows[0]["cell"])
    for g in rows:
        out = O.run_join(R, S, g["algo"], g["pattern"], r_key_unique=uniq)
        assert len(out["key"]) == g["rows_out"] == 1 << 22
        assert _h(O.canonical_digest([out["key"]] + out["payloads"])) == g["digest"]
    assert rows[0]["digest"] == "1cead81753bfbb71"


def _small_join_rows(golden):
    return [g for g in golden["join"] if g["cell"].get("name") != "C1"]


def _load_rows():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")) as f:
        return _small_join_rows(json.load(f))


_ROWS = _load_rows()


@pytest.mark.parametrize("g", _ROWS, ids=[f"{cell_id(g['cell'])}-{g['algo']}-{g['pattern']}"
                                         for g in _ROWS])
def test_join_grid_exact_order(g):
    R, S, uniq = make_cell(g["cell"])
    out = O.run_join(R, S, g["algo"], g["pattern"], r_key_unique=uniq)
    assert len(out["key"]) == g["rows_out"], cell_id(g["cell"])
    assert _h(O.canonical_digest([out["key"]] + out["payloads"])) == g["digest"]
    flat = np.concatenate([out["key"]] + out["payloads"]) if len(out["key"]) else np.zeros(0)
    assert _h(O.digest(flat)) == g["order_digest"]
    if len(out["ids_r"]) > 1:
        cr = np.abs(np.diff(out["ids_r"].astype(np.int64))).mean()
        cs = np.abs(np.diff(out["ids_s"].astype(np.int64))).mean()
        assert abs(cr - g["clusteredness_r"]) < 1e-5 * max(1.0, cr)
        assert abs(cs - g["clusteredness_s"]) < 1e-5 * max(1.0, cs)


def test_generator_digests(golden):
    for g in golden["gen"]:
        c = g["cell"]
        if c.get("name") == "C2":
            continue
        R, S, _ = make_cell(c)
        if c.get("swap"):
            R, S = S, R
        d = g["digests"]
        assert _h(O.digest(R["key"])) == d["r_key"], cell_id(c)
        assert _h(O.digest(S["key"])) == d["s_key"], cell_id(c)
        for i, p in enumerate(R["payloads"]):
            assert _h(O.digest(p)) == d[f"r_p{i}"]
        for i, p in enumerate(S["payloads"]):
            assert _h(O.digest(p)) == d[f"s_p{i}"]


def prim_inputs(n, seed):
    """Seeded inputs of refjoin.cpp cmd_prim, restated with the counter RNG."""
    import ctypes  # noqa: F401
    mix = np.vectorize(O.mix64, otypes=[np.uint64])
    gold = np.uint64(0x9E3779B97F4A7C15)

    def stream(s, tag):
        return int(mix(np.uint64(s) ^ mix(np.uint64(tag) + gold)))

    def at(s, i):
        with np.errstate(over="ignore"):
            return mix(np.uint64(s) + (i.astype(np.uint64) + np.uint64(1)) * gold)

    def below(s, i, b):
        a = at(s, i)
        hi = (a >> np.uint64(32)).astype(object)
        lo = (a & np.uint64(0xFFFFFFFF)).astype(object)
        return np.array([((int(h) << 32 | int(l)) * int(bb)) >> 64
                         for h, l, bb in zip(hi, lo, np.broadcast_to(b, a.shape))], np.uint64)

    i = np.arange(n, dtype=np.uint64)
    k32 = at(seed, i).astype(np.uint32)
    v32 = at(stream(seed, 1), i).astype(np.uint32)
    dup32 = below(stream(seed, 2), i, 97).astype(np.uint32)
    k64 = at(stream(seed, 3), i) >> below(stream(seed, 4), i, 40)
    mp = below(stream(seed, 5), i, n).astype(np.uint32)
    return k32, v32, dup32, k64, mp


def test_primitive_known_answers(golden):
    g = golden["prim"]["5000:2"]
    k32, v32, dup32, k64, mp = prim_inputs(5000, 2)
    ko, (vo,), off = O.radix_partition(k32, [v32], 3, 11)
    assert (_h(O.digest(ko)), _h(O.digest(vo)), _h(O.digest(off))) == (
        g["part32_k"], g["part32_v"], g["part32_off"])
    ko, (vo,) = O.sort_pairs(k32, [v32])
    assert (_h(O.digest(ko)), _h(O.digest(vo))) == (g["sort32_k"], g["sort32_v"])
    ko, (vo,) = O.sort_pairs(dup32, [v32])
    assert (_h(O.digest(ko)), _h(O.digest(vo))) == (g["sortdup_k"], g["sortdup_v"])
    ko, (vo,) = O.sort_pairs(k64, [v32], key_bytes=8)
    assert (_h(O.digest(ko)), _h(O.digest(vo))) == (g["sort64_k"], g["sort64_v"])
    ko, (vo,), off = O.partition_relation(k32, [v32], 16, 8)
    assert (_h(O.digest(ko)), _h(O.digest(vo)), _h(O.digest(off))) == (
        g["prel32_k"], g["prel32_v"], g["prel32_off"])
    ko, (vo,), off = O.partition_relation(k64, [v32], 13, 5, key_bytes=8)
    assert (_h(O.digest(ko)), _h(O.digest(vo)), _h(O.digest(off))) == (
        g["prel64_k"], g["prel64_v"], g["prel64_off"])
    assert _h(O.digest(O.gather(v32, mp))) == g["gather32"]
    assert _h(O.digest(O.gather(k64, mp))) == g["gather64"]
    m = 4000
    rk, sk = dup32[: m // 2], dup32[m // 2: m]
    rko, _, lr = O.partition_relation(rk, [], 4, 8)
    sko, _, ls = O.partition_relation(sk, [], 4, 8)
    keys, ir, js = O.hash_find_matches(rko, lr, sko, ls, limit=16)
    assert (_h(O.digest(keys)), _h(O.digest(ir)), _h(O.digest(js))) == (
        g["hash_keys"], g["hash_ids_r"], g["hash_ids_s"])
    rs, _ = O.sort_pairs(rk, [])
    ss, _ = O.sort_pairs(sk, [])
    keys, ir, js = O.merge_find_matches(rs, ss, False)
    assert (_h(O.digest(keys)), _h(O.digest(ir)), _h(O.digest(js))) == (
        g["merge_keys"], g["merge_ids_r"], g["merge_ids_s"])


def test_reference_known_answers():
    # tests/test_primitives.cpp:25-34
    ko, (vo,), off = O.radix_partition([5, 2, 7, 0], [[10, 20, 30, 40]], 0, 1)
    assert list(ko) == [2, 0, 5, 7] and list(vo) == [20, 40, 10, 30] and list(off) == [0, 2, 4]
    # tests/test_primitives.cpp:71-78
    ko, (vo,) = O.sort_pairs([3, 1, 3, 0], [[10, 20, 30, 40]])
    assert list(ko) == [0, 1, 3, 3] and list(vo) == [40, 20, 10, 30]
    # tests/test_merge_match.cpp:105-112
    k, ir, js = O.merge_find_matches([1, 3, 5], [1, 1, 5], False)
    assert list(ir) == [0, 0, 2] and list(js) == [0, 1, 2]
    # tests/test_merge_match.cpp:173-179
    k, ir, js = O.merge_find_matches([2, 4, 6], [2, 2, 4, 5], True)
    assert list(ir) == [0, 0, 1] and list(js) == [0, 1, 2]
    # tests/test_engine.cpp:41-55 hand example {1,2,3}/{11,12,13} join {3,1}/{21,22}
    R = {"key": np.array([1, 2, 3], np.uint32), "payloads": [np.array([11, 12, 13], np.uint32)]}
    S = {"key": np.array([3, 1], np.uint32), "payloads": [np.array([21, 22], np.uint32)]}
    for a in ("phj", "smj"):
        for p in ("gftr", "gfur"):
            out = O.run_join(R, S, a, p)
            rows = sorted(zip(out["key"], out["payloads"][0], out["payloads"][1]))
            assert rows == [(1, 11, 22), (3, 13, 21)]
    with pytest.raises(O.OracleError):
        O.radix_partition([1, 2], [[1, 2]], 0, 9)
