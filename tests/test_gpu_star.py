"""Chained star joins (sequence.cpp:9-67 run_join_sequence) on the device.

Golden vectors (tests/golden/golden.json "star") come from the UNMODIFIED
reference: workloads::gen_star + the reference's run_join / gather_copy chain
(oracle/refjoin.cpp cmd_star).  The device chain must reproduce the generator
bit for bit, every step's cardinality and column count, and the final join's
output exactly (canonical-row digest and emission-order digest)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

cj = pytest.importorskip("paper_2312_00720_b200")


def _cells(golden):
    return [g for g in golden.get("star", []) if g["cell"].get("name") != "STAR3"]


def _load():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")) as f:
        return json.load(f)


_G = _cells(_load())


@pytest.fixture(scope="module")
def ctx():
    c = cj.Context(0)
    yield c
    c.close()


def _h(t):
    return "%016x" % O.digest(cj.to_host(t).astype(np.uint32).astype(np.uint64))


@pytest.mark.parametrize("g", _G, ids=lambda g: f"{g['cell']['fact']}x{g['cell']['dims']}-"
                                                f"{g['algo']}-{g['pattern']}")
def test_star_chain_matches_reference(ctx, g):
    c, ref = g["cell"], g["ref"]
    fact, dims = cj.gen_star(ctx, c["fact"], c["dims"], c["dim_rows"], c["seed"])
    assert _h(fact.key) == ref["fact_ids"]
    for d in range(c["dims"]):
        assert _h(fact.payloads[d]) == ref[f"fk{d}"]
        assert _h(dims[d].key) == ref[f"dim{d}_key"]
        assert _h(dims[d].payloads[0]) == ref[f"dim{d}_p0"]
    steps, last = cj.run_join_sequence(ctx, fact, dims, g["algo"], g["pattern"])
    assert [s.rows for s in steps] == [r["rows"] for r in ref["steps"]]
    assert [s.output_columns for s in steps] == [r["columns"] for r in ref["steps"]]
    # GFUR gathers each next FK column between the joins (sequence.cpp:43-55);
    # GFTR carries the FK columns through the earlier joins instead
    if g["pattern"] == "gfur":
        assert all(s.fk_fetch_ns > 0 for s in steps[:-1])
    else:
        assert all(s.fk_fetch_ns == 0 for s in steps)
    cols = [cj.to_host(last.relation.key).astype(np.uint64)] + \
           [cj.to_host(p).astype(np.uint32).astype(np.uint64) for p in last.relation.payloads]
    assert "%016x" % O.canonical_digest(cols) == ref["steps"][-1]["digest"]
    assert "%016x" % O.digest(np.concatenate(cols)) == ref["steps"][-1]["order_digest"]


def test_star_chain_errors(ctx):
    fact, dims = cj.gen_star(ctx, 100, 2, 10, 1)
    short = cj.Relation(fact.key, fact.payloads[:1], "fact", True)
    with pytest.raises(cj.SpecInvalid):  # sequence.cpp:14-15
        cj.run_join_sequence(ctx, short, dims)
    wide = cj.Relation(fact.payloads[0], fact.payloads, "fact", True)
    bad_ids = cj.Relation(cj.to_device(np.zeros(100, np.uint64)), fact.payloads, "fact", True)
    with pytest.raises(cj.SpecInvalid):  # sequence.cpp:16-17
        cj.run_join_sequence(ctx, bad_ids, dims)
    del wide
