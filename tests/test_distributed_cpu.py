"""The multi-GPU sharding logic (paper_2312_00720_b200/distributed.py) on CPU:
world_size 2 over gloo.  The device partitioner is replaced by a host
restatement of the same shard function (test double); the exchange, the
co-partitioning guarantee and the union of per-rank joins are checked against
the oracle's single-process join of the whole input."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _host_partition(rel, parts):
    from paper_2312_00720_b200 import coljoin as cjm
    from paper_2312_00720_b200.distributed import host_shard_of
    keys = rel.key.numpy().view(np.uint32 if rel.key.element_size() == 4 else np.uint64)
    shard = host_shard_of(keys, parts)
    order = np.argsort(shard, kind="stable")
    counts = np.bincount(shard, minlength=parts).tolist()
    take = lambda t: torch.from_numpy(t.numpy()[order].copy())
    return cjm.Relation(take(rel.key), [take(p) for p in rel.payloads], rel.name,
                        rel.key_unique), counts


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2312_00720_b200 import coljoin as cjm
    from paper_2312_00720_b200.distributed import distributed_join, host_shard_of
    R, S = O.gen_pk_fk(4096, 8192, 2, 1, match=0.75, zipf=1.0, seed=9)

    def slice_rel(X, uniq):
        n = len(X["key"])
        lo, hi = n * rank // world, n * (rank + 1) // world
        t = lambda a: torch.from_numpy(a[lo:hi].view(np.int32).copy())
        return cjm.Relation(t(X["key"]), [t(p) for p in X["payloads"]], "", uniq)

    Rr, Sr = distributed_join(None, slice_rel(R, True), slice_rel(S, False),
                              partition=_host_partition)
    rk = Rr.key.numpy().view(np.uint32)
    sk = Sr.key.numpy().view(np.uint32)
    # co-partitioning: every received key belongs to this rank
    assert (host_shard_of(rk, world) == rank).all()
    assert (host_shard_of(sk, world) == rank).all()
    local = O.run_join({"key": rk, "payloads": [p.numpy().view(np.uint32) for p in Rr.payloads]},
                       {"key": sk, "payloads": [p.numpy().view(np.uint32) for p in Sr.payloads]},
                       "phj", "gftr")
    rows = np.stack([local["key"]] + local["payloads"], axis=1) if len(local["key"]) else \
        np.zeros((0, 4), np.uint64)
    gathered = [None] * world
    dist.all_gather_object(gathered, rows)
    if rank == 0:
        allrows = np.concatenate(gathered)
        ref = O.run_join(R, S, "phj", "gftr")
        q.put((O.canonical_digest([allrows[:, c] for c in range(allrows.shape[1])]),
               O.canonical_digest([ref["key"]] + ref["payloads"]), len(allrows), len(ref["key"])))
    dist.destroy_process_group()


def test_two_rank_shuffle_join_equals_single_join():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got, want, n_got, n_want = q.get(timeout=10)
    assert n_got == n_want and got == want
