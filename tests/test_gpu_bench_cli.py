"""cj_bench on the device (tools/bench_main.cpp counterpart): the join, gather,
sequence and gen subcommands write the reference's CSV schema / manifest format,
and what they generate is the reference's workload bit for bit."""
import csv
import io
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFJOIN = os.path.join(ROOT, "oracle", "_ref", "refjoin")
CJ_BENCH = os.path.join(ROOT, "paper_2312_00720_b200", "cj_bench")
need_ref = pytest.mark.skipif(not os.path.exists(REFJOIN), reason="oracle/_ref/refjoin not built")


def run(*args, ok=True):
    r = subprocess.run([str(a) for a in args], capture_output=True, text=True, timeout=600)
    if ok:
        assert r.returncode == 0, r.stderr
    return r


def rows_of(text):
    rd = list(csv.DictReader(io.StringIO(text)))
    return rd


@pytest.mark.parametrize("algo,pattern", [("phj", "gftr"), ("smj", "gftr"), ("phj", "gfur"),
                                          ("nphj", "gftr")])
def test_join_rows(algo, pattern, tmp_path):
    out = tmp_path / "j.csv"
    run(CJ_BENCH, "join", "--r-rows", 1 << 16, "--s-rows", 1 << 18, "--payloads", 2, "--reps", 3,
        "--algo", algo, "--pattern", pattern, "--out", out, "--stats")
    text = out.read_text()
    rows = rows_of(text)
    assert len(rows) == 3 and [r["rep"] for r in rows] == ["0", "1", "2"]
    for r in rows:
        assert (r["experiment"], r["algo"], r["pattern"]) == ("join", algo, pattern)
        t = int(r["transform_ns"]) + int(r["find_ns"]) + int(r["materialize_ns"])
        assert int(r["total_ns"]) == t > 0
        assert float(r["throughput_tps"]) == pytest.approx(((1 << 16) + (1 << 18)) / (t * 1e-9))
        # per-phase device high-water marks: the find phase holds the output
        out_bytes = (1 << 18) * 4 * 5  # PK-FK, match 1: |S| rows of key + 2 + 2 u32
        assert int(r["peak_find_b"]) >= out_bytes
        assert int(r["peak_transform_b"]) > 0 if algo != "nphj" else True
        assert float(r["clusteredness_s"]) >= 0.0  # mean |map step| (gather_clusteredness)
    md = run(CJ_BENCH, "report", out).stdout
    assert "## join" in md and "| 3 |" in md
    if os.path.exists(REFJOIN):
        assert run(REFJOIN, "report", "--in", out).stdout == md


@need_ref
def test_gen_matches_reference_generator(tmp_path):
    run(CJ_BENCH, "gen", "--shape", "pkfk", "--r-rows", 5000, "--s-rows", 20000, "--payloads", 2,
        "--key-bytes", 8, "--payload-bytes", 4, "--match", 0.5, "--zipf", 1.0, "--seed", 9,
        "--out-dir", tmp_path)
    want = json.loads(run(REFJOIN, "gen", "--r", 5000, "--s", 20000, "--rpay", 2, "--spay", 2,
                          "--key", "u64", "--pay", "u32", "--match", 0.5, "--zipf", 1.0,
                          "--seed", 9).stdout)
    for side, tag in (("R", "r"), ("S", "s")):
        got = json.loads(run(REFJOIN, "import", "--dir", tmp_path / side).stdout)
        assert got["name"] == side and got["key_unique"] == (1 if side == "R" else 0)
        assert [c["digest"] for c in got["columns"]] == \
            [want[f"{tag}_key"], want[f"{tag}_p0"], want[f"{tag}_p1"]]
    run(CJ_BENCH, "gen", "--shape", "star", "--r-rows", 4096, "--s-rows", 512, "--star-joins", 2,
        "--seed", 3, "--out-dir", tmp_path / "star")
    assert sorted(os.listdir(tmp_path / "star")) == ["dim1", "dim2", "fact"]
    fact = json.loads(run(REFJOIN, "import", "--dir", tmp_path / "star" / "fact").stdout)
    assert fact["rows"] == 4096 and len(fact["columns"]) == 3


@need_ref
def test_join_from_reference_manifests(tmp_path):
    run(REFJOIN, "export", "--r", 3000, "--s", 9000, "--rpay", 1, "--spay", 2, "--match", 0.25,
        "--seed", 4, "--dir", tmp_path)
    out = tmp_path / "j.csv"
    run(CJ_BENCH, "join", "--in-r", tmp_path / "R", "--in-s", tmp_path / "S", "--reps", 2,
        "--out", out)
    rows = rows_of(out.read_text())
    assert len(rows) == 2
    assert (rows[0]["r_rows"], rows[0]["s_rows"], rows[0]["r_payloads"], rows[0]["s_payloads"]) == \
        ("3000", "9000", "1", "2")
    assert run(CJ_BENCH, "join", "--in-r", tmp_path / "R", ok=False).returncode == 1


def test_gather_and_sequence(tmp_path):
    for mode in ("clustered", "unclustered"):
        rows = rows_of(run(CJ_BENCH, "gather", "--items", 1 << 20, "--mode", mode, "--reps",
                           2).stdout)
        assert len(rows) == 2 and rows[0]["experiment"] == "gather-" + mode
        c = float(rows[0]["clusteredness_s"])
        assert (c == 1.0) if mode == "clustered" else (c > 1e4)  # mean |map step|
        assert int(rows[0]["materialize_ns"]) == int(rows[0]["total_ns"]) > 0
    assert run(CJ_BENCH, "gather", "--mode", "sideways", ok=False).returncode == 1
    rows = rows_of(run(CJ_BENCH, "sequence", "--joins", 3, "--fact-rows", 1 << 16, "--dim-rows",
                       1 << 12, "--reps", 2).stdout)
    assert [r["experiment"] for r in rows] == ["sequence-1", "sequence-2", "sequence-3"] * 2
    assert [r["s_payloads"] for r in rows[:3]] == ["1", "2", "3"]
