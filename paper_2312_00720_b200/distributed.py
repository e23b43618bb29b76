"""Radix-sharded multi-GPU join (the reference has no
multi-GPU path) — a thin Python wrapper over the C-ABI
(cj_comm_*, cj_shuffle_relation, cj_run_join_sharded in include/cj_api.h;
implementation csrc/shard.cu).

One process per GPU.  Every rank holds a slice of R and of S.  A row belongs
to rank shard(key) = floor(mix64(key) * world / 2^64) (mix64 = the reference's
SplitMix64 finaliser, rng.hpp:8-12): deterministic in the key, so equal keys
of R and S meet on one rank, and uncorrelated with the low key bits the local
partitioning and hash slots use.  Per relation the library runs

    1. one stable scatter pass whose digit is (shard, low f key bits): the
       destination and the receiver's first LSD digit together;
    2. an exchange of the world x 2^f run lengths (NCCL, control communicator);
    3. grouped ncclSend/ncclRecv of every column, each (source, digit) run
       received at its cj_exchange_plan offset, so the received rows are
       already grouped by their low f bits;
    4. the local join without its first LSD pass.

The output is the union of the per-rank outputs.  This module only creates
the communicator (rank 0's NCCL unique id travels over the torch.distributed
group) and wraps results; there is no data path in Python.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _capi as A
from . import coljoin as cj


class Comm:
    """cj_comm: this rank's NCCL communicator on ctx's device.  from_group()
    builds it for a torch.distributed group (gloo or nccl: the unique id made
    on the group's rank 0 is broadcast through the group); single() is a
    one-rank communicator (the exchange is a self send/receive)."""

    def __init__(self, ctx, uid: bytes, world: int, rank: int):
        self.ctx, self.world, self.rank = ctx, world, rank
        self.h = None
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        A.check(A.lib().cj_comm_init(ctx.h, buf, world, rank, C.byref(h)), ctx.h, "comm_init")
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        uid = (C.c_uint8 * 128)()
        A.check(A.lib().cj_comm_unique_id(uid), None, "comm_unique_id")
        return bytes(uid)

    @classmethod
    def from_group(cls, ctx, group=None):
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        return cls(ctx, obj[0], world, rank)

    @classmethod
    def single(cls, ctx):
        return cls(ctx, cls.unique_id(), 1, 0)

    def close(self):
        if getattr(self, "h", None):
            A.lib().cj_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


@cj.fenced
def shard_partition(ctx, rel, parts: int, first_bits: int = 0):
    """Device send layout: rows stably grouped by (shard, low first_bits key
    bits); counts[dst][d] as a (parts, 2^first_bits) array."""
    cols = list(rel.payloads)
    n = rel.key.numel()
    ko = cj._empty(n, cj._nbytes(rel.key))
    vo = [cj._empty(n, cj._nbytes(p)) for p in cols]
    digits = parts << first_bits
    counts = (C.c_uint64 * digits)()
    A.check(A.lib().cj_shard_partition_ex(ctx.h, rel.key.data_ptr(), ko.data_ptr(), n,
                                          cj._nbytes(rel.key), parts, first_bits, cj._ptrs(cols),
                                          cj._ptrs(vo), cj._u32arr([cj._nbytes(p) for p in cols]),
                                          len(cols), counts), ctx.h, "shard_partition")
    c = np.frombuffer(counts, dtype=np.uint64).reshape(parts, 1 << first_bits).astype(np.int64)
    return cj.Relation(ko, vo, rel.name, rel.key_unique), c


def exchange_plan(send_counts: np.ndarray, recv_counts: np.ndarray):
    """cj_exchange_plan (host only): send_counts[dst][d] of this rank,
    recv_counts[src][d] of every source -> (send_off, recv_off, recv_total)."""
    sc = np.ascontiguousarray(send_counts, dtype=np.uint64)
    rc = np.ascontiguousarray(recv_counts, dtype=np.uint64)
    world, digits = sc.shape
    so, ro = np.zeros_like(sc), np.zeros_like(rc)
    tot = C.c_uint64()
    P = C.POINTER(C.c_uint64)
    A.check(A.lib().cj_exchange_plan(world, digits, sc.ctypes.data_as(P), rc.ctypes.data_as(P),
                                     so.ctypes.data_as(P), ro.ctypes.data_as(P), C.byref(tot)),
            None, "exchange_plan")
    return so.astype(np.int64), ro.astype(np.int64), int(tot.value)


def host_shard_of(keys: np.ndarray, parts: int) -> np.ndarray:
    """Host restatement of the device shard function (CPU tests only)."""
    with np.errstate(over="ignore"):
        x = np.asarray(keys).astype(np.uint64)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    # floor(x * parts / 2^64) without 128-bit numpy arithmetic
    hi, lo = x >> np.uint64(32), x & np.uint64(0xFFFFFFFF)
    p = np.uint64(parts)
    with np.errstate(over="ignore"):
        return ((hi * p + ((lo * p) >> np.uint64(32))) >> np.uint64(32)).astype(np.int64)


def stats_dict(st: A.ShuffleStats) -> dict:
    return {f: getattr(st, f) for f, _ in A.ShuffleStats._fields_}


@cj.fenced
def shuffle(ctx, comm: Comm, rel, first_bits: int = 0, stats: Optional[dict] = None):
    """This rank's shard of `rel` from every rank (cj_shuffle_relation), stably
    grouped by its low first_bits key bits."""
    Rc = cj.c_relation(rel)
    out = A.Relation()
    st = A.ShuffleStats()
    A.check(A.lib().cj_shuffle_relation(ctx.h, comm.h, C.byref(Rc), first_bits, C.byref(out),
                                        C.byref(st)), ctx.h, "shuffle_relation")
    n = out.rows
    key = cj._wrap(ctx, out.key, n, out.key_bytes)
    pays = [cj._wrap(ctx, out.pay[i], n, out.pay_bytes[i]) for i in range(out.npay)]
    if stats is not None:
        stats.update(stats_dict(st))
    return cj.Relation(key, pays, rel.name, rel.key_unique)


@cj.fenced
def distributed_join(ctx, build, probe, algo="phj", pattern="gftr", comm: Optional[Comm] = None,
                     timings: Optional[dict] = None, **kw):
    """Join this rank's slices of R and S across the communicator's ranks
    (cj_run_join_sharded); returns this rank's share of the output."""
    if comm is None:
        raise A.SpecInvalid("distributed_join needs a Comm")
    opt = cj.options(algo, pattern, **kw)
    R, S = cj.c_relation(build), cj.c_relation(probe)
    res = A.JoinResult()
    st = A.ShuffleStats()
    A.check(A.lib().cj_run_join_sharded(ctx.h, comm.h, C.byref(R), C.byref(S), C.byref(opt),
                                        C.byref(res), C.byref(st)), ctx.h, "run_join_sharded")
    if timings is not None:
        timings.update(stats_dict(st))
    return cj.join_output(ctx, res, R, S, build, probe, kw)


@cj.fenced
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
