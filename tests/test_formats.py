"""Data formats either side of the join path, checked
against the reference's own implementations:

- relation manifests (relation_io.cpp:48-103): directories written by the
  reference's export_relation are read by ours (C++: cj_bench manifest, which
  goes through libcoljoin_host's import_relation; Python: import_relation),
  and ours are read by the reference's import_relation (refjoin import);
- the bench CSV wire format + markdown report (bench_io.cpp:16-184): our
  render_report (cj_bench report) prints what the reference's prints for the
  same CSV, and both reject the same schema violations;
- the reference's own unit tests for both (test_workloads.cpp:216-235,
  test_bench_io.cpp) linked against our library (oracle/_ref/dropin_unit).

CPU only: no device work happens on these paths."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

import paper_2312_00720_b200 as cj

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFJOIN = os.path.join(ROOT, "oracle", "_ref", "refjoin")
CJ_BENCH = os.path.join(ROOT, "paper_2312_00720_b200", "cj_bench")
UNIT = os.path.join(ROOT, "oracle", "_ref", "dropin_unit")

need_ref = pytest.mark.skipif(not os.path.exists(REFJOIN), reason="oracle/_ref/refjoin not built")
need_bench = pytest.mark.skipif(not os.path.exists(CJ_BENCH), reason="cj_bench not built")


def run(*args, ok=True):
    r = subprocess.run([str(a) for a in args], capture_output=True, text=True, timeout=300)
    if ok:
        assert r.returncode == 0, r.stderr
    return r


def digests(rel):
    cols = [rel.key] + list(rel.payloads)
    return ["%016x" % O.digest(np.asarray(c).astype(np.uint64)) for c in cols]


@need_ref
@need_bench
@pytest.mark.parametrize("spec", [
    dict(r=1000, s=3000, rpay=2, spay=1, key="u32", pay="u64", match=1.0, zipf=0.0, seed=7),
    dict(r=4096, s=1, rpay=0, spay=3, key="u64", pay="u32", match=0.5, zipf=1.0, seed=3),
    dict(r=1, s=0, rpay=1, spay=1, key="u32", pay="u32", match=1.0, zipf=0.0, seed=1),
])
def test_reference_manifests_read_by_ours(tmp_path, spec):
    args = [REFJOIN, "export", "--dir", tmp_path]
    for k, v in spec.items():
        args += [f"--{k}", v]
    gen = json.loads(run(*args).stdout)
    for side, tag in (("R", "r"), ("S", "s")):
        want = [gen[f"{tag}_key"]] + [gen[f"{tag}_p{c}"] for c in range(spec[f"{tag}pay"])]
        ours_cpp = json.loads(run(CJ_BENCH, "manifest", tmp_path / side).stdout)
        ref = json.loads(run(REFJOIN, "import", "--dir", tmp_path / side).stdout)
        assert ours_cpp == ref
        assert [c["digest"] for c in ours_cpp["columns"]] == want
        rel = cj.import_relation(str(tmp_path / side))
        assert rel.name == side and rel.key_unique == (side == "R")
        assert rel.rows() == spec[tag]
        assert digests(rel) == want
        assert [c.dtype.itemsize for c in rel.payloads] == [4 if spec["pay"] == "u32" else 8] * \
            spec[f"{tag}pay"]


@need_ref
@need_bench
def test_our_manifests_read_by_reference(tmp_path):
    rng = np.random.default_rng(5)
    rel = cj.Relation(rng.integers(0, 2**32, 777, dtype=np.uint64).astype(np.uint32),
                      [rng.integers(0, 2**63, 777, dtype=np.uint64),
                       rng.integers(0, 2**32, 777, dtype=np.uint64).astype(np.uint32)],
                      "dim2", True)
    cj.export_relation(rel, str(tmp_path / "x"))
    ref = json.loads(run(REFJOIN, "import", "--dir", tmp_path / "x").stdout)
    assert ref["name"] == "dim2" and ref["rows"] == 777 and ref["key_unique"] == 1
    assert [c["kind"] for c in ref["columns"]] == ["u32", "u64", "u32"]
    assert [c["digest"] for c in ref["columns"]] == digests(rel)
    assert json.loads(run(CJ_BENCH, "manifest", tmp_path / "x").stdout) == ref
    # a relation without a name is written as "relation" (relation_io.cpp:52)
    cj.export_relation(cj.Relation(np.arange(3, dtype=np.uint32), []), str(tmp_path / "y"))
    assert json.loads(run(REFJOIN, "import", "--dir", tmp_path / "y").stdout)["name"] == "relation"


@need_bench
def test_manifest_errors(tmp_path):
    d = tmp_path / "bad"
    d.mkdir()
    with pytest.raises(cj.SchemaError):  # no manifest
        cj.import_relation(str(d))
    assert run(CJ_BENCH, "manifest", d, ok=False).returncode == 1
    cases = {
        "short": "rows 10\ncolumn key u32 key.bin\n",
        "kind": "rows 2\ncolumn key u16 key.bin\n",
        "field": "rows 2\nbogus 1\ncolumn key u32 key.bin\n",
        "nokey": "rows 2\ncolumn payload0 u32 key.bin\n",
        "malformed": "rows 2\ncolumn key u32\n",
    }
    for name, text in cases.items():
        d = tmp_path / name
        d.mkdir()
        np.arange(2, dtype=np.uint32).tofile(d / "key.bin")
        (d / "manifest.txt").write_text(text)
        with pytest.raises(cj.SchemaError):
            cj.import_relation(str(d))
        assert run(CJ_BENCH, "manifest", d, ok=False).returncode == 1, name
        if os.path.exists(REFJOIN):
            assert run(REFJOIN, "import", "--dir", d, ok=False).returncode == 1, name
    # comments and blank lines are skipped
    d = tmp_path / "comments"
    d.mkdir()
    np.arange(2, dtype=np.uint32).tofile(d / "key.bin")
    (d / "manifest.txt").write_text("# c\n\nrows 2\ncolumn key u32 key.bin\n")
    assert cj.import_relation(str(d)).rows() == 2


HEADER = ("experiment,algo,pattern,r_rows,s_rows,r_payloads,s_payloads,key_bytes,payload_bytes,"
          "match_ratio,zipf,workers,seed,rep,transform_ns,find_ns,materialize_ns,total_ns,"
          "throughput_tps,peak_transform_b,peak_find_b,peak_materialize_b,clusteredness_s,"
          "clusteredness_r")


def csv_rows():
    rows = []
    for exp, algo, pat in (("join", "phj", "gftr"), ("join", "smj", "gfur"),
                           ("gather-unclustered", "-", "-"), ("sequence-1", "phj", "gftr")):
        for rep in range(5):
            tot = 1_000_000 + 137_000 * ((rep * 3) % 5)
            t, f = tot // 5, tot // 2
            rows.append([exp, algo, pat, 1 << 20, 1 << 22, 1, 2, 4, 8, 0.5, 1.25, 148, 42, rep,
                         t, f, tot - t - f, tot, (5 << 20) / (tot * 1e-9), 1, 2, 3, 0.75, 1])
    return rows


@need_ref
@need_bench
def test_report_matches_reference(tmp_path):
    p = tmp_path / "rows.csv"
    p.write_text(HEADER + "\n" + "\n".join(",".join(map(str, r)) for r in csv_rows()) + "\n")
    ours = run(CJ_BENCH, "report", p).stdout
    assert ours == run(REFJOIN, "report", "--in", p).stdout
    assert "## join" in ours and "## gather-unclustered" in ours and "| 5 |" in ours
    out = tmp_path / "r.md"
    run(CJ_BENCH, "report", p, "--out", out)
    assert out.read_text() == ours
    empty = tmp_path / "empty.csv"
    empty.write_text(HEADER + "\n")
    assert run(CJ_BENCH, "report", empty).stdout == ""
    for bad in ("foo,bar\n1,2\n", HEADER + "\n1,2,3\n",
                HEADER + "\n" + ",".join(["x"] * 24) + "\n"):
        q = tmp_path / "bad.csv"
        q.write_text(bad)
        assert run(CJ_BENCH, "report", q, ok=False).returncode == 1
        assert run(REFJOIN, "report", "--in", q, ok=False).returncode == 1


@need_bench
def test_cli_usage_errors():
    assert run(CJ_BENCH, ok=False).returncode == 2
    assert run(CJ_BENCH, "nope", ok=False).returncode == 2
    assert run(CJ_BENCH, "report", ok=False).returncode == 2
    assert run(CJ_BENCH, "join", "--reps", ok=False).returncode == 2


@pytest.mark.skipif(not os.path.exists(UNIT), reason="dropin_unit not built (needs /root/reference)")
def test_reference_format_unit_tests_pass_against_ours():
    cases = ["relations round-trip through the manifest format",
             "throughput is total tuples over total seconds",
             "csv rows round-trip through the pinned schema", "schema violations are rejected",
             "single-row report carries phase percentages summing to 100",
             "empty input renders an empty report", "repetition groups collapse to the median row"]
    args = [UNIT]
    for c in cases:
        args += ["--only", c]
    r = run(*args)
    assert f"test cases: {len(cases)} run, 0 failed" in r.stdout, r.stdout
