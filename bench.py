#!/usr/bin/env python
"""bench.py — end-to-end equi-join throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one run_join of the headline workload (BASELINE.json configs[1],
"C2"): PK-FK |R| = 2^27, |S| = 2^28, 4-byte key + 2 x 4-byte payload columns
per relation, uniform foreign keys, match ratio 1, GFTR partitioned hash join
(PHJ-OM).  Inputs are bit-identical to the reference's workloads::gen_pk_fk
(seed 42), generated on the device.  value = (|R|+|S|) / step time with inputs
resident in HBM (transform + find + materialise, the reference's PhaseReport
scope, mem_ledger.hpp:231-246); e2e = the same through the host-buffer C-ABI
(cj_run_join_host) with pinned host inputs and outputs, copies included.

Under torchrun (N>1) every rank joins its own C2-sized shard (weak scaling);
the step time is the max over ranks.  --impl reference times the reference's
own CPU engine (oracle/_ref/refjoin, compiled from the reference sources) on
the host cores, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "end-to-end join throughput (|R|+|S| tuples/s incl. materialisation) vs HBM roofline"
R_ROWS, S_ROWS, NPAY, SEED = 1 << 27, 1 << 28, 2, 42
WORKLOAD = ("C2: PK-FK |R|=2^27, |S|=2^28, 4-byte key + 2 x 4-byte payloads per relation, "
            "uniform FKs, match ratio 1, seed 42")
# BASELINE.json configs (C1 is the CPU-sized case, C5 the multi-GPU one)
CONFIGS = {
    "C1": dict(r=1 << 20, s=1 << 22, key=4, widths=(4,), match=1.0, zipf=0.0,
               desc="C1: PK-FK |R|=2^20, |S|=2^22, 4-byte key + 1 x 4-byte payload, uniform, match 1"),
    "C2": dict(r=R_ROWS, s=S_ROWS, key=4, widths=(4, 4), match=1.0, zipf=0.0, desc=WORKLOAD),
    "C3": dict(r=R_ROWS, s=S_ROWS, key=8, widths=(4, 8, 4, 8), match=0.5, zipf=0.0,
               desc="C3: |R|=2^27, |S|=2^28, 8-byte keys + payloads [4,8,4,8] B per relation, "
                    "match ratio 0.5, seed 42"),
    "C4z0.5": dict(r=R_ROWS, s=S_ROWS, key=4, widths=(4, 4), match=1.0, zipf=0.5,
                   desc="C4: C2 with Zipf(0.5) foreign keys"),
    "C4z1.0": dict(r=R_ROWS, s=S_ROWS, key=4, widths=(4, 4), match=1.0, zipf=1.0,
                   desc="C4: C2 with Zipf(1.0) foreign keys"),
    "C4z1.5": dict(r=R_ROWS, s=S_ROWS, key=4, widths=(4, 4), match=1.0, zipf=1.5,
                   desc="C4: C2 with Zipf(1.5) foreign keys"),
    # configs[4]'s "3-way star join chain" at the paper's sequence shape
    # (|F|=2^27, |D|=2^25): run_join_sequence, device-resident
    "STAR3": dict(r=1 << 25, s=1 << 27, key=4, widths=(4,), match=1.0, zipf=0.0, dims=3,
                  desc="STAR3: run_join_sequence of 3 PK-FK joins, |F|=2^27 fact rows, "
                       "3 dimensions of 2^25 rows (gen_star, seed 42), one 4-byte payload each"),
}


def b_alg_star(algo, pattern, nf, nd, dims):
    """Sum over the chain (SURVEY.md §8d formula per join) plus the FK gathers
    between joins: join i probes (FK_i, ID, P_1..P_{i-1}) — i + 1 payload
    columns — against a dimension (key + one payload); the probe's columns
    beyond the first cost what the formula charges any further payload column."""
    kbits = max(1, (nd - 1).bit_length())
    P = 2 if algo == "phj" else (kbits + 7) // 8
    tot = 0.0
    for i in range(dims):
        tot += b_alg(algo, pattern, nd, nf, nf, 4, (4,), kbits)
        per_col = (P * 2 * (4 + 4) + (4 + 2 * 4)) if pattern == "gftr" else (4 + 2 * 4)
        tot += i * per_col * nf
        if i + 1 < dims:
            tot += (4 + 2 * 4) * nf  # FK fetch: map read + gather
    return float(tot)


def gen_config(ctx, cfg, nr, ns):
    """Device generation bit-identical to gen_pk_fk (seed 42); mixed widths are
    generated as u64 and the 4-byte columns truncated."""
    import paper_2312_00720_b200 as cj
    ws = cfg["widths"]
    pb = 8 if 8 in ws else 4
    R, S = cj.gen_pk_fk(ctx, nr, ns, len(ws), len(ws), cfg["key"], pb, cfg["match"], cfg["zipf"],
                        SEED)
    if pb == 8:
        import torch

        def narrow(cols):
            return [c if w == 8 else c.view(torch.int32)[::2].contiguous() for c, w in zip(cols, ws)]
        R = cj.Relation(R.key, narrow(R.payloads), "R", True)
        S = cj.Relation(S.key, narrow(S.payloads), "S", False)
        torch.cuda.synchronize()  # the narrowing copies ran on torch's stream
    return R, S


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--variant", default="phj-gftr")
    p.add_argument("--config", default="C2", choices=sorted(CONFIGS),
                   help="BASELINE.json workload (the headline line uses C2)")
    p.add_argument("--scale-log2", type=int, default=0,
                   help="shrink |R|,|S| by 2^k (debug only; the headline uses 0)")
    p.add_argument("--no-extras", action="store_true", help="skip variants/e2e/cpu legs")
    p.add_argument("--sharded", action="store_true",
                   help="run the radix-sharded multi-GPU path even on one rank (exercises the "
                        "shard partition, the NCCL exchange and the per-rank join)")
    p.add_argument("--no-configs", action="store_true",
                   help="skip the C3/C4 records (PHJ/SMJ-GFTR, 3 timed steps each)")
    p.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                   help="weak: every rank joins a C2-sized shard (the default line); strong: "
                        "a fixed C2 x 2^strong-log2 join split over the ranks (sharded path)")
    p.add_argument("--strong-log2", type=int, default=2,
                   help="strong scaling total = C2 x 2^k (k=2: 2^29 x 2^30, fits one GPU)")
    p.add_argument("--e2e-steps", type=int, default=32,
                   help="end-to-end steps (two lanes; more steps amortise the lanes' ramp)")
    return p.parse_args()


def b_alg(algo: str, pattern: str, nr: int, ns: int, nt: int, k=4, w=(4, 4), key_bits=28) -> float:
    """Algorithmic bytes of one join: PHJ P=2 passes, SMJ P =
    live 8-bit digits (4 for keys < 2^28), tuple ids 4 B; gathers count 4 + 2w
    per output element."""
    P = 2 if algo == "phj" else (key_bits + 7) // 8
    if pattern == "gftr":
        t = sum(k * n + P * 2 * (k + w[0]) * n for n in (nr, ns))
        f = k * (nr + ns) + (k + 8) * nt
        m = 0
        for n in (nr, ns):
            m += (4 + 2 * w[0]) * nt
            for wc in w[1:]:
                m += P * 2 * (k + wc) * n + (4 + 2 * wc) * nt
    else:
        t = sum(k * n + P * 2 * (k + 4) * n for n in (nr, ns))
        f = k * (nr + ns) + (k + 16) * nt
        m = 2 * sum((4 + 2 * wc) * nt for wc in w)
    return float(t + f + m)


def b_min(nr, ns, nt, k=4, w=(4, 4)):
    return float((k + sum(w)) * (nr + ns) + (k + 2 * sum(w)) * nt)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.strip()]
        note = None
        if not rows:
            # a timed region shorter than nvidia-smi's start-up (C1): one
            # sample right after it, while the clocks still reflect the load
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=30).stdout
                rows = [r.split(", ") for r in out.strip().splitlines() if r.strip()]
                note = "timed region shorter than the sampler's start-up: one sample right after it"
            except Exception:
                rows = []
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].strip() == "Active"})
        busy = [x for x in sm if x > 600] or sm
        out = {"sm_mhz": statistics.median(busy) if busy else None,
               "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
               "samples": len(rows)}
        if note:
            out["note"] = note
        return out


def config_dict(cfg, a, nr, ns, world):
    """The `config` object of the JSON line; both arms print the same one."""
    sharded = world > 1 or a.sharded or a.scaling == "strong"
    if sharded and a.scaling == "strong":
        wl = (f"C5-shaped strong scaling: |R|=2^{27 + a.strong_log2}, |S|=2^{28 + a.strong_log2} "
              f"total over {world} GPU(s), 4-byte key + 2 x 4-byte payloads, cj_gen_shard")
    elif sharded:
        wl = (f"C5-shaped weak scaling: |R|={world}x2^27, |S|={world}x2^28 total, 4-byte key + "
              "2 x 4-byte payloads, cj_gen_shard")
    else:
        wl = cfg["desc"] if a.scale_log2 == 0 else f"{a.config}/2^{a.scale_log2}"
    return {"workload": wl, "variant": a.variant.upper(), "r_rows": nr, "s_rows": ns,
            "l2": "inputs >> 126 MB L2 (no flush needed)" if nr >= 1 << 24
            else "inputs partly L2-resident (small config)",
            "parallelism": f"radix-sharded x{world}" if sharded else "single GPU"}


def ref_workload_args(cfg, nr, ns):
    """refjoin workload flags for a CONFIGS entry (the reference's WorkloadSpec)."""
    ws = cfg["widths"]
    args = ["--r", str(nr), "--s", str(ns), "--rpay", str(len(ws)), "--spay", str(len(ws)),
            "--key", "u64" if cfg["key"] == 8 else "u32", "--pay", "u64" if 8 in ws else "u32",
            "--match", str(cfg["match"]), "--zipf", str(cfg["zipf"]), "--seed", str(SEED)]
    if 8 in ws:
        args += ["--widths", ",".join(str(w) for w in ws)]
    return args


def self_launch(a):
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run
    with N ranks on this node (fails loudly when fewer GPUs are visible)."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < a.gpus:
        sys.exit(f"bench.py: --gpus {a.gpus} but only {have} CUDA device(s) are visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def reference_arm(a):
    """Reference CPU engine on the host cores (rank 0 only), same config."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    if not O.refjoin_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/refjoin not built (needs /root/reference)"}))
        return
    algo, pattern = a.variant.split("-")
    if algo == "nphj":
        print(json.dumps({"impl": "reference", "unavailable":
                          "the reference has no non-partitioned hash join (SPEC.md)"}))
        return
    cfg = CONFIGS[a.config]
    world = max(world, a.gpus)
    # the whole job: under N ranks our arm joins N C2-sized shards (weak scaling)
    nr, ns = (cfg["r"] >> a.scale_log2) * world, (cfg["s"] >> a.scale_log2) * world
    if a.scaling == "strong":  # the same fixed total as our strong-scaling line
        nr, ns = (cfg["r"] >> a.scale_log2) << a.strong_log2, (cfg["s"] >> a.scale_log2) << a.strong_log2
    cores = os.cpu_count() or 1
    env = dict(os.environ, OMP_NUM_THREADS=str(cores))

    def run(shift, reps, warmup):
        return O.refjoin("join", *ref_workload_args(cfg, nr >> shift, ns >> shift), "--algo", algo,
                         "--pattern", pattern, "--prealloc", "--threads", str(cores), "--reps",
                         str(reps), "--warmup", str(warmup), env=env)

    # The full workload whenever its K+W run_join calls fit the budget (C2 on
    # 16 cores: ~4.6 s per call, ~2 min for 20+5); otherwise the largest
    # same-shape power-of-two sample that does, probed at 1/64 first.
    budget_s = float(os.environ.get("CJ_REF_BUDGET_S", "600"))
    probe = run(6, 1, 0)
    ns_per_tuple = probe["total_ns_mean"] / ((nr >> 6) + (ns >> 6))
    shift = 0
    while shift < 6 and ns_per_tuple * ((nr >> shift) + (ns >> shift)) * (a.steps + a.warmup) \
            > budget_s * 1e9:
        shift += 1
    r = probe if (shift == 6 and a.steps == 1 and a.warmup == 0) else run(shift, a.steps, a.warmup)
    snr, sns = nr >> shift, ns >> shift
    ms = r["total_ns_mean"] / 1e6
    v = (snr + sns) / (ms / 1e3)
    sample = (f"|R|={snr}, |S|={sns} ("
              + ("the whole workload" if shift == 0 else f"1/2^{shift} of the workload, same shape")
              + f"), mean of {a.steps} timed run_join calls after {a.warmup} warm-up "
              f"(preallocate=true, {cores} OpenMP threads)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tuples/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": a.scaling, "vs_baseline": None, "dtype": "u64" if cfg["key"] == 8 else "u32",
        "data": "synthetic: the reference's workloads::gen_pk_fk (seed 42), on the host",
        "config": config_dict(cfg, a, cfg["r"] >> a.scale_log2, cfg["s"] >> a.scale_log2, world),
        "same_workload": shift == 0,
        "cpu_baseline": {"value": v, "unit": "tuples/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phases_ms": {"transform": r["transform_ns"] / 1e6, "find": r["find_ns"] / 1e6,
                      "materialize": r["materialize_ns"] / 1e6},
    }))


def cpu_baseline(nr, ns, variant):
    """oracle/_ref (the reference compiled from its sources) on this host."""
    from oracle import oracle as O
    if not O.refjoin_available():
        return None
    algo, pattern = variant.split("-")
    cores = os.cpu_count() or 1
    # bounded sample: the whole workload, one warm-up + two timed run_join
    # calls (~10-15 s of CPU work at C2 on 16 cores, plus host generation)
    snr, sns = nr, ns
    try:
        r = O.refjoin("join", "--r", str(snr), "--s", str(sns), "--rpay", str(NPAY), "--spay",
                      str(NPAY), "--seed", str(SEED), "--algo", algo, "--pattern", pattern,
                      "--prealloc", "--threads", str(cores), "--reps", "2", "--warmup", "1",
                      env=dict(os.environ, OMP_NUM_THREADS=str(cores)), timeout=900)
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": "tuples/s", "cores": cores, "kind": "reference",
                "sample": f"failed: {e}"}
    v = (snr + sns) / (r["total_ns_mean"] / 1e9)
    return {"value": v, "unit": "tuples/s", "cores": cores, "kind": "reference",
            "sample": f"|R|=2^{snr.bit_length()-1}, |S|=2^{sns.bit_length()-1} (the whole "
                      f"workload), mean of 2 timed run_join calls after 1 warm-up, {cores} "
                      f"threads, preallocate=true",
            "ms": r["total_ns_mean"] / 1e6}


def main():
    a = parse()
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is not None and int(ws_env) != a.gpus and not (a.gpus == 1 and int(ws_env) > 1):
        sys.exit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={ws_env}")
    if a.impl == "reference":
        return reference_arm(a)
    if a.gpus > 1 and ws_env is None:
        return self_launch(a)
    import torch
    import torch.distributed as dist
    import paper_2312_00720_b200 as cj
    from paper_2312_00720_b200 import _capi as A
    import ctypes as C

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    sharded = world > 1 or a.sharded or a.scaling == "strong"
    out_fd = None
    if sharded:
        # rank 0 prints exactly one JSON line: NCCL's banner and anything else a
        # library writes to stdout goes to stderr; the JSON line to the saved fd
        sys.stdout.flush()
        out_fd = os.dup(1)
        os.dup2(2, 1)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = cj.Context(local)
    algo, pattern = a.variant.split("-")
    cfg = CONFIGS[a.config]
    nr, ns = cfg["r"] >> a.scale_log2, cfg["s"] >> a.scale_log2
    res = A.JoinResult()
    L = A.lib()
    opt = cj.options(algo, pattern)
    shuffle = {"exchange_ms": 0.0, "bytes": 0}
    if not sharded:
        # headline config: inputs bit-identical to the reference generator
        if "dims" in cfg:
            fact, dims = cj.gen_star(ctx, ns, cfg["dims"], nr, SEED)
            Fc = cj.coljoin.c_relation(fact)
            Dc = (A.Relation * cfg["dims"])(*[cj.coljoin.c_relation(d) for d in dims])
            st = (A.SequenceStep * cfg["dims"])()
            R, S = dims[0], fact

            def step():
                A.check(L.cj_run_join_sequence(ctx.h, C.byref(Fc), Dc, cfg["dims"], C.byref(opt),
                                               st, C.byref(res)), ctx.h, "run_join_sequence")
                rows = res.rows
                phases = tuple(sum(getattr(st[i], f) for i in range(cfg["dims"]))
                               for f in ("transform_ns", "find_ns", "materialize_ns"))
                A.check(L.cj_result_free(ctx.h, C.byref(res)), ctx.h, "free")
                return rows, phases
        else:
            R, S = gen_config(ctx, cfg, nr, ns)
        Rc, Sc = cj.coljoin.c_relation(R), cj.coljoin.c_relation(S)

        def step_join():
            A.check(L.cj_run_join(ctx.h, C.byref(Rc), C.byref(Sc), C.byref(opt), C.byref(res)),
                    ctx.h, "run_join")
            rows = res.rows
            phases = (res.transform_ns, res.find_ns, res.materialize_ns)
            A.check(L.cj_result_free(ctx.h, C.byref(res)), ctx.h, "free")
            return rows, phases
        if "dims" not in cfg:
            step = step_join
    else:
        # weak scaling: every rank owns a C2-sized slice of a world-times larger
        # PK-FK join; rows are shuffled to their key's shard over NCCL
        from paper_2312_00720_b200 import distributed as D
        if a.scaling == "strong":  # a fixed total split over the ranks
            tot_r, tot_s = nr << a.strong_log2, ns << a.strong_log2
            nr, ns = tot_r // world, tot_s // world
        else:
            tot_r, tot_s = nr * world, ns * world
        R, S = D.gen_shard(ctx, tot_r, tot_s, rank, world, NPAY, NPAY, SEED)
        comm = D.Comm.from_group(ctx)

        def step():
            t = {}
            out = D.distributed_join(ctx, R, S, algo, pattern, comm=comm, timings=t)
            shuffle["exchange_ms"] += (t["exchange_r_ns"] + t["exchange_s_ns"]) / 1e6
            shuffle["shard_ms"] = shuffle.get("shard_ms", 0.0) + t["shard_ns"] / 1e6
            shuffle["bytes"] += t["bytes_sent_peers"]
            shuffle["first_bits"] = t["first_bits"]
            rows = out.matches
            phases = (out.report.transform_ns, out.report.find_ns, out.report.materialize_ns)
            del out
            return rows, phases

    for _ in range(a.warmup):
        rows, _ = step()
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    clocks = Clocks(local)
    l0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(ctx.stream)
    phase_sum = [0, 0, 0]
    for _ in range(a.steps):
        rows, ph = step()
        for i in range(3):
            phase_sum[i] += ph[i]
    ev1.record(ctx.stream)
    torch.cuda.synchronize()
    launches = ctx.launches - l0
    ms = ev0.elapsed_time(ev1) / a.steps
    if sharded:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    clk = clocks.stop()
    shuffle_info = None
    if sharded:
        nsteps = max(a.steps + a.warmup, 1)
        ex = torch.tensor([shuffle["exchange_ms"] / nsteps, shuffle.get("shard_ms", 0.0) / nsteps],
                          device="cuda")
        dist.all_reduce(ex, op=dist.ReduceOp.MAX)
        per_step_bytes = shuffle["bytes"] / nsteps
        ex_ms, sh_ms = float(ex[0].item()), float(ex[1].item())
        shuffle_info = {"bytes_sent_to_peers_per_gpu_per_step": per_step_bytes,
                        "exchange_ms_max_over_ranks": ex_ms,
                        "shard_pass_ms_max_over_ranks": sh_ms,
                        "first_lsd_bits_in_shard_pass": shuffle.get("first_bits"),
                        "nvlink_gbs_per_gpu": per_step_bytes / 1e9 / (ex_ms / 1e3)
                        if ex_ms > 0 and per_step_bytes > 0 else None,
                        "nvlink_peak_gbs_per_dir": 770.0,
                        "how": "device time of the R and S data exchanges (CUDA events on the "
                               "library's NCCL stream), bytes to other ranks only",
                        "transport": "cj_run_join_sharded: grouped ncclSend/ncclRecv per (peer, "
                                     "first-digit run), NCCL over NVLink/NVSwitch"}
    # Per-kernel CUDA-event records: the same K steps again, each kernel
    # bracketed by events on the ctx stream (the launching stream).  Kept out of
    # the headline region above; the event pool is reset per step so no event
    # is created while timing.
    names = (C.c_char_p * 4096)()
    kms = (C.c_float * 4096)()
    kby = (C.c_uint64 * 4096)()
    cnt = C.c_int()
    agg = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    inst_ms = 0.0
    for _ in range(a.steps):
        A.check(L.cj_set_kernel_timing(ctx.h, 1), ctx.h, "timing")
        e0.record(ctx.stream)
        step()
        e1.record(ctx.stream)
        A.check(L.cj_kernel_records(ctx.h, 4096, names, kms, kby, C.byref(cnt)), ctx.h, "records")
        torch.cuda.synchronize()
        inst_ms += e0.elapsed_time(e1)
        for i in range(min(cnt.value, 4096)):
            e = agg.setdefault(names[i].decode(), [0, 0.0, 0])
            e[0] += 1
            e[1] += kms[i]
            e[2] += kby[i]
    A.check(L.cj_set_kernel_timing(ctx.h, 0), ctx.h, "timing")
    inst_ms /= a.steps
    peak, peak_src = peaks()
    kernels = sorted(({"kernel": n, "launches": c, "ms_per_step": t / a.steps,
                       "share": t / (inst_ms * a.steps) if inst_ms else None,
                       "alg_gbs": (b / 1e9) / (t / 1e3) if t else None}
                      for n, (c, t, b) in agg.items()), key=lambda d: -d["ms_per_step"])
    dom = kernels[0] if kernels else None
    # DRAM traffic per launch of the dominant kernel: not measurable inside a
    # timed run (ncu replays kernels), so it comes from the committed ncu
    # capture of the same kernel, labelled with its source; null when the
    # capture does not cover this kernel/config
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        ent = tj.get(f"{a.config}/{a.variant}/{dom['kernel']}") if dom else None
        if isinstance(ent, dict):
            traffic, traffic_src = ent.get("bytes_per_launch"), ent.get("source")
    except Exception:
        pass
    roofline = None
    if dom:
        c, t, b = agg[dom["kernel"]]
        achieved = (b / c) / 1e9 / ((t / c) / 1e3)
        roofline = {"bound": "hbm", "kernel": dom["kernel"], "achieved": achieved, "peak": peak,
                    "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                    "traffic_source": traffic_src,
                    "alg_bytes_per_launch": b / c, "peak_source": peak_src}
    tuples = (nr + ns) * world * cfg.get("dims", 1)
    value = tuples / (ms / 1e3)
    kb, ws = cfg["key"], cfg["widths"]
    key_bits = max(1, (2 * cfg["r"] - 1).bit_length() if cfg["match"] < 1 else (cfg["r"] - 1).bit_length())
    balg = b_alg(algo, pattern, nr, ns, rows, kb, ws, key_bits)
    if "dims" in cfg:
        balg = b_alg_star(algo, pattern, ns, nr, cfg["dims"])
    out = {
        "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": a.scaling,
        "vs_baseline": None, "dtype": "u64" if cfg["key"] == 8 else "u32",
        "data": "synthetic: bit-identical to the reference's workloads::gen_pk_fk "
                "(seed 42 + rank), generated on the device",
        "config": config_dict(cfg, a, nr, ns, world), "out_rows": rows,
        "roofline": roofline,
        "join_roofline": {"b_alg_bytes": balg, "b_min_bytes": b_min(nr, ns, rows, kb, ws),
                          "frac_b_alg": balg / (ms / 1e3) / (peak * 1e9),
                          "frac_b_min": b_min(nr, ns, rows, kb, ws) / (ms / 1e3) / (peak * 1e9)},
        "phases_ms": {"transform": phase_sum[0] / 1e6 / a.steps,
                      "find_and_fused_materialize": phase_sum[1] / 1e6 / a.steps,
                      "materialize": phase_sum[2] / 1e6 / a.steps},
        "gpu_launches": launches, "clocks": clk,
        "kernel_timing": {"ms_per_step_instrumented": inst_ms,
                          "kernel_sum_ms_per_step": sum(k["ms_per_step"] for k in kernels),
                          "how": "second pass of K steps, CUDA events around every launch on "
                                 "the ctx stream"},
        "kernels": kernels,
    }
    if shuffle_info:
        out["shuffle"] = shuffle_info
    if rank == 0 and not sharded and not a.no_extras and a.config == "C2":
        # the other variants (3 timed steps each)
        var = {}
        for v in ("phj-gftr", "smj-gftr", "phj-gfur", "smj-gfur", "nphj-gftr", "nphj-gfur"):
            o = cj.options(*v.split("-"))
            step_opt = o

            def vstep():
                A.check(L.cj_run_join(ctx.h, C.byref(Rc), C.byref(Sc), C.byref(step_opt),
                                      C.byref(res)), ctx.h, "run_join")
                A.check(L.cj_result_free(ctx.h, C.byref(res)), ctx.h, "free")
            vstep()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            for _ in range(3):
                vstep()
            e1.record(ctx.stream)
            torch.cuda.synchronize()
            vms = e0.elapsed_time(e1) / 3
            va, vp = v.split("-")
            var[v] = {"ms": vms, "tuples_per_s": (nr + ns) / (vms / 1e3),
                      "frac_b_alg": (b_alg(va, vp, nr, ns, rows, kb, ws, key_bits) / (vms / 1e3) / (peak * 1e9)
                                     if va != "nphj" else None)}
        out["variants"] = var
        # end to end through the host-buffer C-ABI (pinned host in/out)
        out["e2e"] = e2e_leg(ctx, R, S, opt, steps=a.e2e_steps)
        out["cpu_baseline"] = cpu_baseline(nr, ns, a.variant)
        if not a.no_configs:
            del Rc, Sc, R, S
            torch.cuda.empty_cache()
            out["configs"] = configs_leg(ctx, peak)
    if rank == 0:
        if out_fd is not None:
            sys.stdout.flush()
            os.write(out_fd, (json.dumps(out) + "\n").encode())
        else:
            print(json.dumps(out))
    if sharded:
        comm.close()
        dist.destroy_process_group()


def configs_leg(ctx, peak, names=("C3", "C4z0.5", "C4z1.0", "C4z1.5"), steps=3):
    """The other full-size BASELINE.json configs (C3, C4 at three skews): PHJ- and
    SMJ-GFTR, one warm-up + `steps` timed joins each, device-resident inputs
    generated bit-identically to the reference; ms and fraction of B_alg."""
    import ctypes as C
    import torch
    import paper_2312_00720_b200 as cj
    from paper_2312_00720_b200 import _capi as A
    L = A.lib()
    res = A.JoinResult()
    recs = {}
    # a fresh ctx (its own stream-ordered pool): the headline ctx's pool is
    # fragmented by the variants and the e2e lanes, and a C3-sized reservation
    # next to it can fall back to mapping memory mid-join
    ctx = cj.Context(ctx.device)
    for name in names:
        cfg = CONFIGS[name]
        nr, ns = cfg["r"], cfg["s"]
        R, S = gen_config(ctx, cfg, nr, ns)
        Rc, Sc = cj.coljoin.c_relation(R), cj.coljoin.c_relation(S)
        key_bits = max(1, (2 * nr - 1).bit_length() if cfg["match"] < 1 else (nr - 1).bit_length())
        rec = {}
        for v in ("phj-gftr", "smj-gftr"):
            o = cj.options(*v.split("-"))

            def one():
                A.check(L.cj_run_join(ctx.h, C.byref(Rc), C.byref(Sc), C.byref(o), C.byref(res)),
                        ctx.h, "run_join")
                rows = res.rows
                A.check(L.cj_result_free(ctx.h, C.byref(res)), ctx.h, "free")
                return rows
            rows = one()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            for _ in range(steps):
                one()
            e1.record(ctx.stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            va, vp = v.split("-")
            balg = b_alg(va, vp, nr, ns, rows, cfg["key"], cfg["widths"], key_bits)
            rec[v] = {"ms": ms, "tuples_per_s": (nr + ns) / (ms / 1e3), "out_rows": rows,
                      "frac_b_alg": balg / (ms / 1e3) / (peak * 1e9)}
        recs[name] = {"workload": cfg["desc"], **rec}
        del Rc, Sc, R, S
        torch.cuda.empty_cache()
    ctx.close()
    return recs


def e2e_leg(ctx, R, S, opt, steps=32, streams=2):
    """End to end through the host-buffer C-ABI (cj_run_join_host): every step
    uploads its pinned host input columns, joins, and downloads every output
    column into pinned host memory, all inside the timed region.  Steps run
    on `streams` contexts from as many host threads (the C-ABI allows one
    thread per ctx), so one step's download overlaps the next one's upload —
    PCIe is full duplex, and the library serialises same-direction copies of
    concurrent calls.  value = tuples of all timed steps / wall time."""
    import ctypes as C
    import threading
    import torch
    from paper_2312_00720_b200 import _capi as A
    import paper_2312_00720_b200 as cj
    L = A.lib()
    hk = [R.key.cpu().pin_memory()] + [p.cpu().pin_memory() for p in R.payloads]
    sk = [S.key.cpu().pin_memory()] + [p.cpu().pin_memory() for p in S.payloads]
    Rh = cj.Relation(hk[0], hk[1:], "R", True)
    Sh = cj.Relation(sk[0], sk[1:], "S", False)
    Rc, Sc = cj.coljoin.c_relation(Rh), cj.coljoin.c_relation(Sh)  # data_ptr() of pinned host
    row_out = R.key.element_size() + sum(p.element_size() for p in R.payloads + S.payloads)
    out_bytes = S.key.numel() * row_out

    class Lane:
        def __init__(self, c):
            self.ctx = c
            self.arena = torch.empty(out_bytes + 4096 * 8, dtype=torch.uint8).pin_memory()
            self.off = 0
            self.cb = A.HOST_ALLOC(self.alloc)
            self.res = A.JoinResult()
            self.h2d, self.d2h = C.c_uint64(), C.c_uint64()
            self.err = None

        def alloc(self, nbytes, _user):
            p = self.arena.data_ptr() + self.off
            self.off += (int(nbytes) + 255) & ~255
            return p

        def run(self, n, delay=0.0):
            try:
                if delay:
                    time.sleep(delay)
                for _ in range(n):
                    self.off = 0
                    A.check(L.cj_run_join_host(self.ctx.h, C.byref(Rc), C.byref(Sc), C.byref(opt),
                                               self.cb, None, C.byref(self.res), C.byref(self.h2d),
                                               C.byref(self.d2h)), self.ctx.h, "e2e")
            except Exception as e:  # noqa: BLE001
                self.err = e

    lanes = [Lane(ctx)] + [Lane(cj.Context(ctx.device)) for _ in range(streams - 1)]
    lanes[0].run(1)  # warm-up: module loading, this lane's pool
    warm = [threading.Thread(target=ln.run, args=(1,)) for ln in lanes[1:]]
    for t in warm:
        t.start()
    lanes[0].run(1)
    for t in warm:
        t.join()
    per = [steps // streams + (1 if i < steps % streams else 0) for i in range(streams)]
    # the library lets one host-buffer join per device upload (and one
    # download) at a time, so the lanes settle into one lane's download next
    # to the other's upload by themselves
    th = [threading.Thread(target=ln.run, args=(k,)) for ln, k in zip(lanes, per)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    for ln in lanes:
        if ln.err:
            raise ln.err
    n = R.key.numel() + S.key.numel()
    bi = sum(x.numel() * x.element_size() for x in hk + sk)
    bo = lanes[0].res.rows * row_out
    for ln in lanes[1:]:
        ln.ctx.close()
    return {"value": n * steps / wall, "unit": "tuples/s", "h2d_bytes_per_step": bi,
            "d2h_bytes_per_step": bo, "ms_per_step": wall * 1e3 / steps,
            "h2d_ms_per_call": lanes[0].h2d.value / 1e6, "d2h_ms_per_call": lanes[0].d2h.value / 1e6,
            "api": "cj_run_join_host (pinned host columns in, pinned host columns out)",
            "steps": steps, "concurrent_streams": streams,
            "how": "wall clock over all steps; one host thread + ctx per stream"}


if __name__ == "__main__":
    main()
