"""Radix-sharded multi-GPU join (the reference has no multi-GPU
path).

One process per GPU.  Every rank holds a horizontal slice of R and of S.  The
join shards by key: shard(key) = floor(mix64(key) * world / 2^64) (mix64 is the
reference's SplitMix64 finaliser, rng.hpp:8-12), which is deterministic in the
key, so every R row and every S row with the same key meet on one rank, and is
uncorrelated with the low key bits the local partitioning and hash slots use.

    1. cj_shard_partition: stable device partition of the local rows by shard
       (the send layout; one onesweep scatter pass with the shard as digit);
    2. exchange the world x world row counts (all_to_all_single of int64);
    3. shuffle every column with all_to_all_single (NCCL over NVLink/NVSwitch
       on B200; gloo on CPU for the tests);
    4. run the single-GPU join on the received rows.

The output is the union of the per-rank outputs; no gather step.  GFTR ships
full rows (key + payloads) so materialisation stays local.
"""
from __future__ import annotations

import ctypes as C
import time
from typing import Callable, Optional

import numpy as np

from . import _capi as A
from . import coljoin as cj


def shard_partition(ctx, rel, parts: int):
    """Device send layout: rows grouped by destination shard (stable)."""
    torch = cj._torch()
    cols = list(rel.payloads)
    n = rel.key.numel()
    ko = cj._empty(n, cj._nbytes(rel.key))
    vo = [cj._empty(n, cj._nbytes(p)) for p in cols]
    counts = (C.c_uint64 * parts)()
    A.check(A.lib().cj_shard_partition(ctx.h, rel.key.data_ptr(), ko.data_ptr(), n,
                                       cj._nbytes(rel.key), parts, cj._ptrs(cols), cj._ptrs(vo),
                                       cj._u32arr([cj._nbytes(p) for p in cols]), len(cols),
                                       counts), ctx.h, "shard_partition")
    del torch
    return cj.Relation(ko, vo, rel.name, rel.key_unique), [int(c) for c in counts]


def host_shard_of(keys: np.ndarray, parts: int) -> np.ndarray:
    """Host restatement of the device shard function (for CPU tests only)."""
    k = np.asarray(keys).astype(np.uint64)
    with np.errstate(over="ignore"):
        x = k.copy()
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return np.array([(int(v) * parts) >> 64 for v in x], dtype=np.int64)


def exchange(rel, counts, group=None, async_op=False):
    """all_to_all shuffle of a shard-grouped relation; returns the received
    rows, the received counts and (async_op) the pending column transfers,
    which the caller waits on before reading the rows."""
    import torch
    import torch.distributed as dist
    dev = rel.key.device
    send = torch.tensor(counts, dtype=torch.int64, device=dev)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    rc = [int(x) for x in recv.tolist()]
    out_cols, works = [], []
    for col in [rel.key] + list(rel.payloads):
        out = torch.empty(sum(rc), dtype=col.dtype, device=dev)
        w = dist.all_to_all_single(out, col, rc, counts, group=group, async_op=async_op)
        if async_op:
            works.append(w)
        out_cols.append(out)
    result = cj.Relation(out_cols[0], out_cols[1:], rel.name, rel.key_unique)
    return (result, rc, works) if async_op else (result, rc)


def distributed_join(ctx, build, probe, algo="phj", pattern="gftr", group=None,
                     partition: Optional[Callable] = None, timings: Optional[dict] = None, **kw):
    """Join this rank's slices of R and S across the group; returns this
    rank's share of the output (a cj.JoinOutput).  `partition(rel, parts)` may
    replace the device partitioner (CPU tests)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    part = partition or (lambda rel, p: shard_partition(ctx, rel, p))
    cuda = ctx is not None
    if cuda:
        import torch
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
    t0 = time.perf_counter()
    # R's columns travel while S is partitioned (the collectives run on the
    # process group's stream; the partition on the ctx stream)
    Rs, rcount = part(build, world)
    Rr, _, r_works = exchange(Rs, rcount, group, async_op=True)
    Ss, scount = part(probe, world)
    t1 = time.perf_counter()
    if cuda:
        ev[1].record()
    Sr, _ = exchange(Ss, scount, group)
    for w in r_works:
        w.wait()
    t2 = time.perf_counter()
    if cuda:
        ev[2].record()
        ev[2].synchronize()
    if timings is not None:
        timings["partition_s"] = t1 - t0
        timings["exchange_s"] = t2 - t1
        if cuda:
            # (R's exchange overlaps S's partition: partition_ms includes it)
            timings["partition_ms"] = ev[0].elapsed_time(ev[1])
            timings["exchange_ms"] = ev[1].elapsed_time(ev[2])
        sent = sum(c for d, c in enumerate(rcount) if d != dist.get_rank(group))
        sent_s = sum(c for d, c in enumerate(scount) if d != dist.get_rank(group))
        row_r = sum(x.element_size() for x in [build.key] + list(build.payloads))
        row_s = sum(x.element_size() for x in [probe.key] + list(probe.payloads))
        timings["bytes_sent"] = sent * row_r + sent_s * row_s
    if ctx is None:  # CPU test path: the caller joins the received rows
        return Rr, Sr
    return cj.run_join(ctx, Rr, Sr, algo, pattern, **kw)


def gen_shard(ctx, r_rows_total, s_rows_total, rank, ranks, r_payloads=2, s_payloads=2, seed=42):
    """This rank's slice of the weak-scaling workload (cj_gen_shard)."""
    rn, sn = r_rows_total // ranks, s_rows_total // ranks
    rk, sk = cj._empty(rn, 4), cj._empty(sn, 4)
    rp = [cj._empty(rn, 4) for _ in range(r_payloads)]
    sp = [cj._empty(sn, 4) for _ in range(s_payloads)]
    A.check(A.lib().cj_gen_shard(ctx.h, r_rows_total, s_rows_total, rank, ranks, r_payloads,
                                 s_payloads, seed, rk.data_ptr(), cj._ptrs(rp), sk.data_ptr(),
                                 cj._ptrs(sp)), ctx.h, "gen_shard")
    return cj.Relation(rk, rp, "R", True), cj.Relation(sk, sp, "S", False)
