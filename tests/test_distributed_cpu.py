"""The multi-GPU sharding logic on CPU: world_size 2 over gloo.

The device data path (shard pass, NCCL exchange, presorted local join) needs
GPUs; what runs here is everything around it, in two real processes:
  - the send layout the device shard pass produces (rows stably grouped by
    (shard, low f key bits), restated on the host with the same mix64 shard
    function),
  - the library's own exchange placement (cj_exchange_plan, host-only C-ABI)
    applied to the runs each rank receives over gloo,
  - the receiver's invariant that makes the local first LSD pass redundant:
    the received relation equals the stable sort, by the low f bits, of the
    sources' rows concatenated in rank order,
  - co-partitioning, and that the union of the per-rank joins (oracle) is the
    single-process join of the whole input."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _send_layout(rel, world, f):
    """Host restatement of cj_shard_partition_ex: stable by shard << f | low f bits."""
    from paper_2312_00720_b200.distributed import host_shard_of
    keys = rel["key"]
    digit = (host_shard_of(keys, world) << f) | (keys.astype(np.int64) & ((1 << f) - 1))
    order = np.argsort(digit, kind="stable")
    counts = np.bincount(digit, minlength=world << f).reshape(world, 1 << f)
    return {"key": keys[order], "payloads": [p[order] for p in rel["payloads"]]}, counts


def _worker(rank, world, port, f, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2312_00720_b200.distributed import exchange_plan, host_shard_of
        R, S = O.gen_pk_fk(4096, 8192, 2, 1, match=0.75, zipf=1.0, seed=9)

        def slice_rel(X):
            n = len(X["key"])
            lo, hi = n * rank // world, n * (rank + 1) // world
            return {"key": X["key"][lo:hi], "payloads": [p[lo:hi] for p in X["payloads"]]}

        got = {}
        for name, X in (("R", R), ("S", S)):
            send, sc = _send_layout(slice_rel(X), world, f)
            # every rank's counts and send layout travel over gloo
            allc, alls = [None] * world, [None] * world
            dist.all_gather_object(allc, sc)
            dist.all_gather_object(alls, send)
            rc = np.stack([allc[src][rank] for src in range(world)])
            so, ro, total = exchange_plan(sc, rc)
            # the send offsets address this rank's own layout run by run
            assert np.array_equal(so.ravel(), np.concatenate([[0], np.cumsum(sc.ravel())[:-1]]))
            cols = [np.zeros(total, np.uint64) for _ in range(1 + len(send["payloads"]))]
            for src in range(world):
                s_sc = allc[src]
                s_so, _, _ = exchange_plan(s_sc, rc)  # src's own send offsets for its counts
                s_off = np.concatenate([[0], np.cumsum(s_sc.ravel())[:-1]]).reshape(s_sc.shape)
                assert np.array_equal(s_so, s_off)
                for d in range(1 << f):
                    n = int(rc[src, d])
                    lo = int(s_off[rank, d])
                    for c, col in enumerate([alls[src]["key"]] + alls[src]["payloads"]):
                        cols[c][ro[src, d]:ro[src, d] + n] = col[lo:lo + n]
            # the invariant: stable sort by the low f bits of the sources' rows in rank order
            cat = [np.concatenate([
                ([alls[src]["key"]] + alls[src]["payloads"])[c][host_shard_of(
                    alls[src]["key"], world) == rank] for src in range(world)])
                for c in range(len(cols))]
            order = np.argsort(cat[0].astype(np.int64) & ((1 << f) - 1), kind="stable")
            for c in range(len(cols)):
                assert np.array_equal(cols[c], cat[c][order].astype(np.uint64))
            assert (host_shard_of(cols[0], world) == rank).all()  # co-partitioned
            got[name] = {"key": cols[0].astype(np.uint32),
                         "payloads": [c.astype(np.uint32) for c in cols[1:]]}
        local = O.run_join(got["R"], got["S"], "phj", "gftr")
        rows = np.stack([local["key"]] + local["payloads"], axis=1) if len(local["key"]) else \
            np.zeros((0, 4), np.uint64)
        gathered = [None] * world
        dist.all_gather_object(gathered, rows)
        if rank == 0:
            allrows = np.concatenate(gathered)
            ref = O.run_join(R, S, "phj", "gftr")
            q.put((O.canonical_digest([allrows[:, c] for c in range(allrows.shape[1])]),
                   O.canonical_digest([ref["key"]] + ref["payloads"]), len(allrows),
                   len(ref["key"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("f", [0, 3, 6])
def test_two_rank_shuffle_join_equals_single_join(f):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, f, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got, want, n_got, n_want = q.get(timeout=10)
    assert n_got == n_want and got == want


def test_exchange_plan_places_runs_digit_major():
    """cj_exchange_plan on a 3-rank, 4-digit shape: send offsets are the
    row-major prefix of the send counts; receive offsets put every source's
    digit-d run after all smaller digits and after earlier sources' digit-d runs."""
    from paper_2312_00720_b200.distributed import exchange_plan
    g = np.random.default_rng(3)
    sc = g.integers(0, 50, (3, 4))
    rc = g.integers(0, 50, (3, 4))
    so, ro, total = exchange_plan(sc, rc)
    assert total == rc.sum()
    assert np.array_equal(so.ravel(), np.concatenate([[0], np.cumsum(sc.ravel())[:-1]]))
    flat = rc.T.ravel()  # (digit, source) order
    want = np.concatenate([[0], np.cumsum(flat)[:-1]]).reshape(4, 3).T
    assert np.array_equal(ro, want)
