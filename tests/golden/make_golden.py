"""Regenerate tests/golden/golden.json from the UNMODIFIED reference.

Runs oracle/_ref/refjoin (the reference library compiled from
/root/reference/proj/src by oracle/Makefile) and records:
  * join:  canonical-row digest (oracle.cpp:77-88 + BASELINE.md §2 formula),
           emission-order digest, output rows and clusteredness for every
           variant over the acceptance criterion-1 grid
           (tests/acceptance_main.cpp:63-79, r_pay=2, s_pay=1) plus C1, the
           mixed-width C3 shape and duplicate-build (--swap) cells;
  * gen:   column digests of workloads::gen_pk_fk outputs;
  * prim:  primitive known-answer digests (refjoin.cpp cmd_prim).
Only runs where /root/reference exists (this container); the JSON is committed.

    python tests/golden/make_golden.py            # everything
    python tests/golden/make_golden.py --c2-gen   # append the C2 generator digests only
    python tests/golden/make_golden.py --star     # (re)write the star-chain cells only
    python tests/golden/make_golden.py --sparse-dup  # (re)write the ~1-row-per-key non-PK cells
    python tests/golden/make_golden.py --full C3 C4z0.5 ...  # full-size BASELINE configs
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def grid():
    cells, seed = [], 1
    for rows in (1024, 16384):
        for match in (0.0, 0.25, 0.5, 1.0):
            for zipf in (0.0, 1.0, 2.0):
                for key in ("u32", "u64"):
                    cells.append(dict(r=rows, s=2 * rows, match=match, zipf=zipf, key=key,
                                      pay=key, rpay=2, spay=1, seed=seed))
                    seed += 1
    return cells


def wl_args(c):
    a = ["--r", str(c["r"]), "--s", str(c["s"]), "--rpay", str(c["rpay"]), "--spay",
         str(c["spay"]), "--key", c["key"], "--pay", c["pay"], "--match", str(c["match"]),
         "--zipf", str(c["zipf"]), "--seed", str(c["seed"])]
    if c.get("widths"):
        a += ["--widths", c["widths"]]
    if c.get("swap"):
        a += ["--swap"]
    return a


C2 = dict(r=1 << 27, s=1 << 28, match=1.0, zipf=0.0, key="u32", pay="u32", rpay=2, spay=2,
          seed=42, name="C2")


def add_c2_gen():
    """Generator digests of the full-size headline config (BASELINE.json configs[1])."""
    path = os.path.join(HERE, "golden.json")
    with open(path) as f:
        out = json.load(f)
    out["gen"] = [g for g in out["gen"] if g["cell"].get("name") != "C2"]
    out["gen"].append(dict(cell=C2, digests=O.refjoin("gen", *wl_args(C2))))
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


STAR_CELLS = [dict(fact=4096, dims=3, dim_rows=1024, seed=42),
              dict(fact=1 << 18, dims=4, dim_rows=1 << 16, seed=44),
              dict(fact=1 << 20, dims=3, dim_rows=1 << 18, seed=42)]
STAR3 = dict(fact=1 << 27, dims=3, dim_rows=1 << 25, seed=42, name="STAR3")


def add_star():
    """workloads::gen_star + the chained joins (refjoin star): column digests of
    the inputs and, per join, rows / columns / canonical and emission digests."""
    path = os.path.join(HERE, "golden.json")
    with open(path) as f:
        out = json.load(f)
    out["star"] = []
    cells = STAR_CELLS + ([STAR3] if os.environ.get("GOLDEN_STAR3") else [])
    for c in cells:
        for algo, pat in (("phj", "gftr"), ("smj", "gfur"), ("phj", "gfur"), ("smj", "gftr")):
            if c.get("name") == "STAR3" and (algo, pat) != ("phj", "gftr"):
                continue
            r = O.refjoin("star", "--fact", str(c["fact"]), "--dims", str(c["dims"]), "--dim-rows",
                          str(c["dim_rows"]), "--seed", str(c["seed"]), "--algo", algo, "--pattern",
                          pat, "--threads", "8")
            out["star"].append(dict(cell=c, algo=algo, pattern=pat, ref=r))
            print(c, algo, pat, file=sys.stderr)
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


# Non-PK builds with about one row per key value (--swap with |S| = |R|: the
# build is S, uniform draws from [0, |R|), so ~37% of key values are missing
# and ~26% repeat).  A sorted window of such a build can span exactly its
# length with duplicates standing in for gaps ([5,5,7] vs [5,6,7]), which is
# what broke the SMJ dense-window shortcut in round 1.
SPARSE_DUP_CELLS = [dict(r=n, s=n, match=1.0, zipf=0.0, key=k, pay="u32", rpay=1, spay=2, seed=s,
                         swap=True, name=f"sparse-dup-{k}-{n}")
                    for n, k, s in ((4096, "u32", 201), (65536, "u64", 202), (1 << 20, "u32", 203))]


def join_rows(c):
    rows = []
    for algo in ("phj", "smj"):
        for pat in ("gftr", "gfur"):
            r = O.refjoin("join", *wl_args(c), "--algo", algo, "--pattern", pat, "--digest",
                          "--threads", "4")
            rows.append(dict(cell=c, algo=algo, pattern=pat, rows_out=r["rows_out"],
                             digest=r["digest"], order_digest=r["order_digest"],
                             clusteredness_r=r["clusteredness_r"],
                             clusteredness_s=r["clusteredness_s"]))
    return rows


def add_sparse_dup():
    path = os.path.join(HERE, "golden.json")
    with open(path) as f:
        out = json.load(f)
    out["join"] = [g for g in out["join"] if not g["cell"].get("name", "").startswith("sparse-dup")]
    for c in SPARSE_DUP_CELLS:
        out["join"] += join_rows(c)
        print(c, file=sys.stderr)
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


# BASELINE.json configs[1..3] at full size (|R| = 2^27, |S| = 2^28, seed 42).
# The reference generates the inputs (workloads::gen_pk_fk; C4 z=0.5 takes ~10
# min single-threaded) and runs all four variants; the canonical digest goes
# through refjoin's parallel canonical sort (--pdigest, checked against
# oracle::canonical_rows on small cells by --digest --pdigest).  Each entry
# keeps rows_out, the canonical digest and the emission-order digest of every
# variant.
FULL_CELLS = {
    "C2": dict(r=1 << 27, s=1 << 28, match=1.0, zipf=0.0, key="u32", pay="u32", rpay=2, spay=2,
               seed=42),
    "C3": dict(r=1 << 27, s=1 << 28, match=0.5, zipf=0.0, key="u64", pay="u64", rpay=4, spay=4,
               seed=42, widths="4,8,4,8"),
    **{f"C4z{z}": dict(r=1 << 27, s=1 << 28, match=1.0, zipf=z, key="u32", pay="u32", rpay=2,
                       spay=2, seed=42) for z in (0.5, 1.0, 1.5)},
}


def add_full(names):
    path = os.path.join(HERE, "golden.json")
    for name in names:
        c = dict(FULL_CELLS[name], name=name)
        p = subprocess.run([O.REFJOIN, "join", *wl_args(c), "--all-variants", "--pdigest",
                            "--threads", str(os.cpu_count())], capture_output=True, text=True,
                           check=True)
        variants = [json.loads(line) for line in p.stdout.splitlines() if line.strip()]
        rec = dict(cell=c, variants={v["variant"]: {k: v[k] for k in (
            "rows_out", "digest", "order_digest", "clusteredness_r", "clusteredness_s",
            "total_ns_median", "threads")} for v in variants})
        with open(path) as f:
            out = json.load(f)
        out.setdefault("full", [])
        out["full"] = [g for g in out["full"] if g["cell"]["name"] != name] + [rec]
        with open(path, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)
        print(name, rec["variants"], file=sys.stderr, flush=True)


def main():
    O.build()
    if "--full" in sys.argv:
        return add_full(sys.argv[sys.argv.index("--full") + 1:])
    if "--sparse-dup" in sys.argv:
        return add_sparse_dup()
    if "--c2-gen" in sys.argv:
        return add_c2_gen()
    if "--star" in sys.argv:
        return add_star()
    out = {"join": [], "gen": [], "prim": {}}
    cells = grid()
    cells.append(dict(r=1 << 20, s=1 << 22, match=1.0, zipf=0.0, key="u32", pay="u32", rpay=1,
                      spay=1, seed=42, name="C1"))
    cells.append(dict(r=4096, s=8192, match=0.5, zipf=0.0, key="u64", pay="u64", rpay=4, spay=4,
                      seed=42, widths="4,8,4,8", name="C3-shape"))
    for z in (0.5, 1.0, 1.5):
        cells.append(dict(r=8192, s=16384, match=1.0, zipf=z, key="u32", pay="u32", rpay=2,
                          spay=2, seed=42, name=f"C4-shape-z{z}"))
    for seed, z in ((101, 1.0), (102, 2.0)):
        cells.append(dict(r=2048, s=4096, match=1.0, zipf=z, key="u32", pay="u32", rpay=1,
                          spay=2, seed=seed, swap=True, name=f"dup-build-z{z}"))
    cells += SPARSE_DUP_CELLS
    for c in cells:
        out["join"] += join_rows(c)
        print(c, file=sys.stderr)
    for c in (cells[0], cells[5], cells[-7], cells[-6], cells[-3]):
        out["gen"].append(dict(cell=c, digests=O.refjoin("gen", *wl_args(c))))
    if os.environ.get("GOLDEN_C2"):
        out["gen"].append(dict(cell=C2, digests=O.refjoin("gen", *wl_args(C2))))
    for n, seed in ((5000, 2), (100000, 1)):
        out["prim"][f"{n}:{seed}"] = O.refjoin("prim", "--n", str(n), "--seed", str(seed))
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
