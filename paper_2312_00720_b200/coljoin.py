"""Python mirror of the reference operator API for the join path, over the C-ABI.

Names, argument meaning and error behaviour follow the reference's C++ API
(paths relative to the reference's proj/): primitives.hpp:25-77,
hash_match.hpp:26-81, merge_match.hpp:25-52, join_engine.hpp:60-105,
task.hpp:24-41, workloads.hpp:11-33.  The C++ host library
(include/coljoin/*.hpp) is the same mirror for C++ callers.

Device columns are torch CUDA tensors used as raw storage: 4-byte columns are
torch.int32, 8-byte columns torch.int64 (bit patterns are unsigned; view the
host copies as np.uint32 / np.uint64).  torch supplies device memory and the
stream; every byte of join work runs in the hand-written sm_100a kernels of
libcoljoin_b200.so — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi as A
from ._capi import check

_ALGOS = {"smj": A.SMJ, "phj": A.PHJ, "nphj": A.NPHJ}
_PATTERNS = {"gfur": A.GFUR, "gftr": A.GFTR}


def _torch():
    import torch
    return torch


def _nbytes(t) -> int:
    return t.element_size()


def _tdtype(nbytes: int):
    torch = _torch()
    return torch.int32 if nbytes == 4 else torch.int64


def to_device(a, nbytes: Optional[int] = None):
    """Host numpy column -> device tensor (int32/int64 storage of the bits)."""
    torch = _torch()
    a = np.ascontiguousarray(a)
    nb = nbytes or a.dtype.itemsize
    a = a.astype(np.uint32 if nb == 4 else np.uint64, copy=False)
    return torch.from_numpy(a.view(np.int32 if nb == 4 else np.int64)).cuda()


def to_host(t) -> np.ndarray:
    """Device tensor -> numpy uint32/uint64."""
    a = t.detach().cpu().numpy()
    return a.view(np.uint32 if a.dtype.itemsize == 4 else np.uint64)


class Context:
    """One cj_ctx bound to a device and a stream (torch's current stream)."""

    def __init__(self, device: int = 0, stream=None):
        torch = _torch()
        torch.cuda.set_device(device)
        self.stream = stream or torch.cuda.current_stream(device)
        self.device = device
        h = C.c_void_p()
        st = A.lib().cj_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        if st != 0:
            raise A._BY_CODE.get(st, A.Error)(f"cj_ctx_create failed (status {st})")
        self.h = h
        # the library's own stream (a fresh non-blocking one unless a stream
        # was passed): torch work is ordered against it by `fenced`
        self.lib_stream = torch.cuda.ExternalStream(A.lib().cj_ctx_stream(h) or 0, device=device)

    @property
    def launches(self) -> int:
        return int(A.lib().cj_launch_count(self.h))

    def sync(self):
        check(A.lib().cj_sync(self.h), self.h, "sync")

    def close(self):
        if self.h:
            A.lib().cj_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def fenced(fn):
    """Entry points that take a Context first: the library's stream waits for
    the work torch queued on its current stream (the inputs), and torch's
    stream waits for the library's work (the outputs), without host syncs."""
    import functools

    @functools.wraps(fn)
    def wrapper(ctx, *args, **kw):
        torch = _torch()
        lib = getattr(ctx, "lib_stream", None)
        if lib is None:
            return fn(ctx, *args, **kw)
        cur = torch.cuda.current_stream(ctx.device)
        lib.wait_stream(cur)
        try:
            return fn(ctx, *args, **kw)
        finally:
            cur.wait_stream(lib)
    return wrapper


class DeviceBuffer:
    """A library-allocated device array exposed to torch via
    __cuda_array_interface__; released with cj_free when torch drops it."""

    def __init__(self, ctx: Context, ptr: int, n: int, nbytes: int):
        self.ctx, self.ptr, self.n, self.nbytes = ctx, ptr, n, nbytes

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.n,), "typestr": "<i4" if self.nbytes == 4 else "<i8",
                "data": (self.ptr or 0, False), "version": 2,
                "stream": None}

    def tensor(self):
        torch = _torch()
        if self.n == 0:
            return torch.empty(0, dtype=_tdtype(self.nbytes), device="cuda")
        return torch.as_tensor(self, device="cuda")

    def __del__(self):
        if self.ptr and self.ctx.h:
            try:
                A.lib().cj_free(self.ctx.h, C.c_void_p(self.ptr))
            except (TypeError, AttributeError):  # interpreter shutdown: modules torn down
                pass
            self.ptr = 0


def _wrap(ctx, ptr, n, nbytes):
    t = DeviceBuffer(ctx, ptr, n, nbytes).tensor()
    return t


def _ptrs(ts):
    arr = (C.c_void_p * max(len(ts), 1))(*[t.data_ptr() for t in ts])
    return arr


def _u32arr(vals):
    return (C.c_uint32 * max(len(vals), 1))(*vals)


def _empty(n, nbytes):
    return _torch().empty(max(n, 0), dtype=_tdtype(nbytes), device="cuda")


# ---- primitives (primitives.hpp:25-77) --------------------------------------

@fenced
def histogram(ctx: Context, keys, low_bit: int, high_bit: int) -> np.ndarray:
    fan = 1 << max(0, min(high_bit - low_bit, 8))
    out = (C.c_uint32 * fan)()
    check(A.lib().cj_histogram(ctx.h, keys.data_ptr(), keys.numel(), _nbytes(keys), low_bit,
                               high_bit, out), ctx.h, "histogram")
    return np.frombuffer(out, dtype=np.uint32).copy()


def exclusive_prefix_sum(counts) -> np.ndarray:
    """primitives.hpp:31-33 (host helper)."""
    c = np.asarray(counts, dtype=np.uint64)
    out = np.zeros(c.size + 1, np.uint64)
    np.cumsum(c, out=out[1:])
    return out


@fenced
def radix_partition(ctx: Context, keys, vals: Sequence, low_bit: int, high_bit: int):
    """One stable pass; returns (keys_out, [vals_out], offsets[np.uint64])."""
    n = keys.numel()
    for v in vals:
        if v.numel() != n:
            raise A.LengthMismatch("key and value columns differ in length")
    ko = _empty(n, _nbytes(keys))
    vo = [_empty(n, _nbytes(v)) for v in vals]
    fan = (1 << (high_bit - low_bit)) if 0 <= high_bit - low_bit <= 8 else 1
    off = (C.c_uint64 * (fan + 1))()
    check(A.lib().cj_radix_partition(ctx.h, keys.data_ptr(), ko.data_ptr(), n, _nbytes(keys),
                                     low_bit, high_bit, _ptrs(vals), _ptrs(vo),
                                     _u32arr([_nbytes(v) for v in vals]), len(vals), off),
          ctx.h, "radix_partition")
    return ko, vo, np.frombuffer(off, dtype=np.uint64).copy()


@fenced
def radix_partition_passes(ctx: Context, keys, vals: Sequence, plan, gen_ids: bool = False):
    n = keys.numel()
    ko = _empty(n, _nbytes(keys))
    widths = ([4] if gen_ids else []) + [_nbytes(v) for v in vals]
    vo = [_empty(n, w) for w in widths]
    vin = ([ko] if gen_ids else []) + list(vals)  # ids column input is ignored
    lo = _u32arr([p[0] for p in plan])
    hi = _u32arr([p[1] for p in plan])
    check(A.lib().cj_radix_partition_passes(ctx.h, keys.data_ptr(), ko.data_ptr(), n,
                                            _nbytes(keys), lo, hi, len(plan), _ptrs(vin),
                                            _ptrs(vo), _u32arr(widths), len(widths),
                                            int(gen_ids)), ctx.h, "radix_partition_passes")
    return ko, vo


@fenced
def sort_pairs(ctx: Context, keys, vals: Sequence = (), gen_ids: bool = False):
    n = keys.numel()
    ko = _empty(n, _nbytes(keys))
    widths = ([4] if gen_ids else []) + [_nbytes(v) for v in vals]
    vo = [_empty(n, w) for w in widths]
    vin = ([ko] if gen_ids else []) + list(vals)
    check(A.lib().cj_sort_pairs(ctx.h, keys.data_ptr(), ko.data_ptr(), n, _nbytes(keys),
                                _ptrs(vin), _ptrs(vo), _u32arr(widths), len(widths),
                                int(gen_ids)), ctx.h, "sort_pairs")
    return ko, vo


def sort_keys(ctx: Context, keys):
    return sort_pairs(ctx, keys, ())[0]


@fenced
def gather(ctx: Context, cols: Sequence, idx):
    """out[c][i] = cols[c][idx[i]]; idx int32 tensor of u32 ids."""
    m = idx.numel()
    n_in = cols[0].numel() if cols else 0
    outs = [_empty(m, _nbytes(c)) for c in cols]
    check(A.lib().cj_gather(ctx.h, _ptrs(cols), n_in, idx.data_ptr(), m, _ptrs(outs),
                            _u32arr([_nbytes(c) for c in cols]), len(cols)), ctx.h, "gather")
    return outs


def gather_clusteredness(ids: np.ndarray) -> float:
    """primitives.cpp:398-407 (host helper)."""
    ids = np.asarray(ids)
    if ids.size == 0:
        raise A.EmptyInput("clusteredness of an empty map")
    if ids.size == 1:
        return 1.0
    return float(np.abs(np.diff(ids.astype(np.int64))).sum()) / (ids.size - 1)


@fenced
def partition_relation(ctx: Context, keys, vals: Sequence, total_bits: int,
                       bits_per_pass: int = 8, gen_ids: bool = False):
    """hash_match.hpp:26-38; returns (keys_out, [vals_out], offsets device int64)."""
    torch = _torch()
    n = keys.numel()
    ko = _empty(n, _nbytes(keys))
    widths = ([4] if gen_ids else []) + [_nbytes(v) for v in vals]
    vo = [_empty(n, w) for w in widths]
    vin = ([ko] if gen_ids else []) + list(vals)
    off = torch.empty((1 << min(total_bits, 20)) + 1, dtype=torch.int64, device="cuda")
    check(A.lib().cj_partition_relation(ctx.h, keys.data_ptr(), ko.data_ptr(), n, _nbytes(keys),
                                        total_bits, bits_per_pass, _ptrs(vin), _ptrs(vo),
                                        _u32arr(widths), len(widths), int(gen_ids),
                                        off.data_ptr()), ctx.h, "partition_relation")
    return ko, vo, off


@fenced
def hash_find_matches(ctx: Context, bkeys, boff, pkeys, poff, limit: int = 4096,
                      id_mode: str = "virtual", bcarried=None, pcarried=None):
    """hash_match.hpp:73-81: returns (keys, ids_r, ids_s) device tensors."""
    if boff.numel() != poff.numel():
        raise A.FanoutMismatch("build and probe views disagree on fan-out")
    b = A.Partitioned(bkeys.data_ptr(), boff.data_ptr(),
                      bcarried.data_ptr() if bcarried is not None else None, bkeys.numel())
    p = A.Partitioned(pkeys.data_ptr(), poff.data_ptr(),
                      pcarried.data_ptr() if pcarried is not None else None, pkeys.numel())
    tot = C.c_uint64()
    k, ir, js = C.c_void_p(), C.c_void_p(), C.c_void_p()
    mode = A.IDS_VIRTUAL if id_mode == "virtual" else A.IDS_PHYSICAL
    check(A.lib().cj_hash_find_matches(ctx.h, C.byref(b), C.byref(p), boff.numel() - 1,
                                       _nbytes(bkeys), limit, mode, C.byref(tot), C.byref(k),
                                       C.byref(ir), C.byref(js)), ctx.h, "hash_find_matches")
    t = tot.value
    return (_wrap(ctx, k.value, t, _nbytes(bkeys)), _wrap(ctx, ir.value, t, 4),
            _wrap(ctx, js.value, t, 4))


@fenced
def merge_find_matches(ctx: Context, r_sorted, s_sorted, pk_fk: bool, validate: bool = False):
    """merge_match.hpp:49-52: returns (keys, ids_r, ids_s) device tensors."""
    if _nbytes(r_sorted) != _nbytes(s_sorted):
        raise A.KindError("merge inputs must share a value kind")
    tot = C.c_uint64()
    k, ir, js = C.c_void_p(), C.c_void_p(), C.c_void_p()
    check(A.lib().cj_merge_find_matches(ctx.h, r_sorted.data_ptr(), r_sorted.numel(),
                                        s_sorted.data_ptr(), s_sorted.numel(), _nbytes(r_sorted),
                                        int(pk_fk), int(validate), C.byref(tot), C.byref(k),
                                        C.byref(ir), C.byref(js)), ctx.h, "merge_find_matches")
    t = tot.value
    return (_wrap(ctx, k.value, t, _nbytes(r_sorted)), _wrap(ctx, ir.value, t, 4),
            _wrap(ctx, js.value, t, 4))


# ---- relations and the end-to-end join (join_engine.hpp:60-105) -------------

@dataclass
class Relation:
    """column.hpp:115-123: key + ordered payloads (+ key_unique)."""
    key: object
    payloads: list = field(default_factory=list)
    name: str = ""
    key_unique: bool = False

    def rows(self) -> int:
        return int(self.key.numel() if hasattr(self.key, "numel") else len(self.key))


@dataclass
class PhaseReport:
    """mem_ledger.hpp:231-246: phase times and, per phase, the device bytes the
    call held at its high-water mark (peak_by_phase)."""
    transform_ns: int = 0
    find_ns: int = 0
    materialize_ns: int = 0
    peak_by_phase: tuple = (0, 0, 0)
    # MemLedger view (mem_ledger.hpp:26-100) per phase: logical bytes of
    # column-sized working data and of scratch at the phase's high-water mark
    column_bytes: tuple = (0, 0, 0)
    scratch_bytes: tuple = (0, 0, 0)

    def total_ns(self) -> int:
        return self.transform_ns + self.find_ns + self.materialize_ns


@dataclass
class JoinOutput:
    relation: Relation
    report: PhaseReport
    matches: int
    clusteredness_r: float = 1.0
    clusteredness_s: float = 1.0
    ids_r: object = None
    ids_s: object = None


def options(algo="phj", pattern="gftr", radix_bits_per_pass=8, total_radix_bits=-1,
            sub_partition_limit=4096, validate=False, want_ids=False, want_stats=False):
    o = A.JoinOptions()
    A.lib().cj_default_options(C.byref(o))
    o.algo = _ALGOS[algo]
    o.pattern = _PATTERNS[pattern]
    o.radix_bits_per_pass = radix_bits_per_pass
    o.total_radix_bits = total_radix_bits
    o.sub_partition_limit = sub_partition_limit
    o.validate = int(validate)
    o.want_ids = int(want_ids)
    o.want_stats = int(want_stats)
    return o


def c_relation(rel: Relation, host: bool = False) -> A.Relation:
    if len(rel.payloads) > A.CJ_MAX_COLS:
        raise A.Unsupported("too many payload columns")
    r = A.Relation()
    if host:
        r.key = rel.key.ctypes.data
        r.key_bytes = rel.key.dtype.itemsize
        r.rows = rel.key.size
        for i, p in enumerate(rel.payloads):
            if p.size != rel.key.size:
                raise A.LengthMismatch("payload length differs from key length")
            r.pay[i] = p.ctypes.data
            r.pay_bytes[i] = p.dtype.itemsize
    else:
        r.key = rel.key.data_ptr()
        r.key_bytes = _nbytes(rel.key)
        r.rows = rel.key.numel()
        for i, p in enumerate(rel.payloads):
            if p.numel() != rel.key.numel():
                raise A.LengthMismatch("payload length differs from key length")
            r.pay[i] = p.data_ptr()
            r.pay_bytes[i] = _nbytes(p)
    r.npay = len(rel.payloads)
    r.key_unique = int(rel.key_unique)
    return r


def join_output(ctx: Context, res, R, S, build: Relation, probe: Relation, kw) -> JoinOutput:
    """Wrap a cj_join_result's library-owned columns as torch tensors."""
    t = res.rows
    key = _wrap(ctx, res.key, t, R.key_bytes)
    pays = [_wrap(ctx, res.pay[i], t, R.pay_bytes[i]) for i in range(R.npay)]
    pays += [_wrap(ctx, res.pay[R.npay + i], t, S.pay_bytes[i]) for i in range(S.npay)]
    ids_r = _wrap(ctx, res.ids_r, t, 4) if res.ids_r else None
    ids_s = _wrap(ctx, res.ids_s, t, 4) if res.ids_s else None
    rel = Relation(key, pays, name=(build.name + "_" + probe.name) or "join")
    return JoinOutput(rel, PhaseReport(res.transform_ns, res.find_ns, res.materialize_ns,
                                       (res.peak_transform_b, res.peak_find_b,
                                        res.peak_materialize_b),
                                       tuple(res.ledger_column_b), tuple(res.ledger_scratch_b)), t,
                      res.clusteredness_r if kw.get("want_stats") else 1.0,
                      res.clusteredness_s if kw.get("want_stats") else 1.0, ids_r, ids_s)


@fenced
def run_join(ctx: Context, build: Relation, probe: Relation, algo="phj", pattern="gftr",
             **kw) -> JoinOutput:
    """join_engine.hpp:68 run_join on device-resident relations."""
    opt = options(algo, pattern, **kw)
    R, S = c_relation(build), c_relation(probe)
    res = A.JoinResult()
    check(A.lib().cj_run_join(ctx.h, C.byref(R), C.byref(S), C.byref(opt), C.byref(res)),
          ctx.h, "run_join")
    return join_output(ctx, res, R, S, build, probe, kw)


@fenced
def run_join_presorted(ctx: Context, build: Relation, probe: Relation, presorted_bits: int,
                       algo="phj", pattern="gftr", **kw) -> JoinOutput:
    """run_join on relations already stably grouped by their low
    `presorted_bits` key bits (what the sharded join's exchange delivers): the
    transform skips its first LSD pass; the output multiset is run_join's."""
    opt = options(algo, pattern, **kw)
    R, S = c_relation(build), c_relation(probe)
    res = A.JoinResult()
    check(A.lib().cj_run_join_presorted(ctx.h, C.byref(R), C.byref(S), C.byref(opt),
                                        presorted_bits, C.byref(res)), ctx.h, "run_join_presorted")
    return join_output(ctx, res, R, S, build, probe, kw)


class _HostArena:
    """Host output allocator for cj_run_join_host (numpy-owned buffers)."""

    def __init__(self):
        self.bufs = []
        self.cb = A.HOST_ALLOC(self._alloc)

    def _alloc(self, nbytes, _user):
        b = np.empty(int(nbytes), np.uint8)
        self.bufs.append(b)
        return b.ctypes.data

    def take(self, ptr, n, nbytes):
        for b in self.bufs:
            if b.ctypes.data == ptr:
                return b[: n * nbytes].view(np.uint32 if nbytes == 4 else np.uint64)
        raise KeyError(ptr)


@fenced
def run_join_host(ctx: Context, build: Relation, probe: Relation, algo="phj", pattern="gftr",
                  **kw):
    """The drop-in for coljoin::run_join(const JoinTask&) with host columns:
    returns (JoinOutput with numpy columns, h2d_ns, d2h_ns)."""
    opt = options(algo, pattern, **kw)
    R, S = c_relation(build, host=True), c_relation(probe, host=True)
    res = A.JoinResult()
    arena = _HostArena()
    h2d, d2h = C.c_uint64(), C.c_uint64()
    check(A.lib().cj_run_join_host(ctx.h, C.byref(R), C.byref(S), C.byref(opt), arena.cb, None,
                                   C.byref(res), C.byref(h2d), C.byref(d2h)), ctx.h,
          "run_join_host")
    t = res.rows
    key = arena.take(res.key, t, R.key_bytes)
    pays = [arena.take(res.pay[i], t, R.pay_bytes[i]) for i in range(R.npay)]
    pays += [arena.take(res.pay[R.npay + i], t, S.pay_bytes[i]) for i in range(S.npay)]
    ids_r = arena.take(res.ids_r, t, 4) if res.ids_r else None
    ids_s = arena.take(res.ids_s, t, 4) if res.ids_s else None
    out = JoinOutput(Relation(key, pays),
                     PhaseReport(res.transform_ns, res.find_ns, res.materialize_ns,
                                 (res.peak_transform_b, res.peak_find_b, res.peak_materialize_b),
                                 tuple(res.ledger_column_b), tuple(res.ledger_scratch_b)),
                     t,
                     res.clusteredness_r, res.clusteredness_s, ids_r, ids_s)
    return out, h2d.value, d2h.value


# ---- workloads (workloads.hpp:11-33) ------------------------------------------

@fenced
def gen_pk_fk(ctx: Context, r_rows, s_rows, r_payloads=1, s_payloads=1, key_bytes=4,
              pay_bytes=4, match_ratio=1.0, zipf_factor=0.0, seed=0):
    """Device-resident inputs bit-identical to workloads::gen_pk_fk."""
    rk = _empty(r_rows, key_bytes)
    sk = _empty(s_rows, key_bytes)
    rp = [_empty(r_rows, pay_bytes) for _ in range(r_payloads)]
    sp = [_empty(s_rows, pay_bytes) for _ in range(s_payloads)]
    check(A.lib().cj_gen_pk_fk(ctx.h, r_rows, s_rows, r_payloads, s_payloads, key_bytes,
                               pay_bytes, match_ratio, zipf_factor, seed, rk.data_ptr(),
                               _ptrs(rp), sk.data_ptr(), _ptrs(sp)), ctx.h, "gen_pk_fk")
    return (Relation(rk, rp, "R", True), Relation(sk, sp, "S", False))


@dataclass
class SequenceStep:
    """sequence.hpp:10-15."""
    rows: int
    output_columns: int
    report: PhaseReport
    fk_fetch_ns: int


@fenced
def run_join_sequence(ctx: Context, fact: Relation, dims: Sequence, algo="phj", pattern="gftr",
                      **kw):
    """sequence.hpp:21-24 run_join_sequence, device-resident (no host copy
    between the joins).  Returns (steps, final JoinOutput)."""
    opt = options(algo, pattern, **kw)
    F = c_relation(fact)
    D = (A.Relation * max(len(dims), 1))(*[c_relation(d) for d in dims])
    st = (A.SequenceStep * max(len(dims), 1))()
    res = A.JoinResult()
    check(A.lib().cj_run_join_sequence(ctx.h, C.byref(F), D, len(dims), C.byref(opt), st,
                                       C.byref(res)), ctx.h, "run_join_sequence")
    steps = [SequenceStep(st[i].rows, st[i].output_columns,
                          PhaseReport(st[i].transform_ns, st[i].find_ns, st[i].materialize_ns),
                          st[i].fk_fetch_ns) for i in range(len(dims))]
    if not dims:
        return steps, None
    t = res.rows
    last = dims[-1]
    nr = len(last.payloads)
    key = _wrap(ctx, res.key, t, _nbytes(last.key))
    pays = [_wrap(ctx, res.pay[i], t, _nbytes(last.payloads[i])) for i in range(nr)]
    # carried probe columns: (ID, payloads of dims 1..n-1)  (sequence.cpp:56-62)
    widths = [4] + [_nbytes(p) for d in dims[:-1] for p in d.payloads]
    pays += [_wrap(ctx, res.pay[nr + i], t, w) for i, w in enumerate(widths)]
    return steps, JoinOutput(Relation(key, pays, "sequence"),
                             PhaseReport(res.transform_ns, res.find_ns, res.materialize_ns), t)


@fenced
def gen_star(ctx: Context, fact_rows: int, dims: int, dim_rows: int, seed: int = 0,
             key_bytes: int = 4, pay_bytes: int = 4):
    """workloads.hpp:47-61 gen_star, bit-identical, on the device."""
    ids = _empty(fact_rows, 4)
    fks = [_empty(fact_rows, key_bytes) for _ in range(dims)]
    dk = [_empty(dim_rows, key_bytes) for _ in range(dims)]
    dp = [_empty(dim_rows, pay_bytes) for _ in range(dims)]
    check(A.lib().cj_gen_star(ctx.h, fact_rows, dims, dim_rows, seed, key_bytes, pay_bytes,
                              ids.data_ptr(), _ptrs(fks), _ptrs(dk), _ptrs(dp)), ctx.h, "gen_star")
    fact = Relation(ids, fks, "fact", True)
    return fact, [Relation(dk[d], [dp[d]], f"dim{d + 1}", True) for d in range(dims)]


# ---- relation manifests (relation_io.hpp:7-15, relation_io.cpp:48-103) -------

def export_relation(rel: Relation, path) -> None:
    """workloads::export_relation: manifest.txt + one raw little-endian file per
    column (key.bin, payload<c>.bin).  Device columns are downloaded; numpy
    columns are written as they are.  Readable by the reference's
    import_relation and by import_relation below."""
    import os
    os.makedirs(path, exist_ok=True)

    def host(c):
        return np.ascontiguousarray(c) if isinstance(c, np.ndarray) else to_host(c)

    cols = [("key", "key.bin", host(rel.key))] + \
        [(f"payload{i}", f"payload{i}.bin", host(p)) for i, p in enumerate(rel.payloads)]
    lines = [f"name {rel.name or 'relation'}", f"rows {len(cols[0][2])}",
             f"key_unique {1 if rel.key_unique else 0}"]
    for label, fname, a in cols:
        if a.dtype.itemsize not in (4, 8):
            raise A.SchemaError("columns are u32 or u64")
        a.astype("<u4" if a.dtype.itemsize == 4 else "<u8", copy=False).tofile(
            os.path.join(path, fname))
        lines.append(f"column {label} {'u32' if a.dtype.itemsize == 4 else 'u64'} {fname}")
    with open(os.path.join(path, "manifest.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")


def import_relation(path, ctx: Optional[Context] = None) -> Relation:
    """workloads::import_relation.  With a ctx the columns go straight to the
    device (int32/int64 tensors holding the bits), else they stay numpy.
    SchemaError on a missing/malformed manifest or a short column file."""
    import os
    mf = os.path.join(path, "manifest.txt")
    if not os.path.exists(mf):
        raise A.SchemaError(f"no manifest.txt in {path}")
    name, rows, unique, key, pays = "", 0, False, None, []
    with open(mf) as f:
        for line in f:
            line = line.rstrip("\n")
            if not line or line.startswith("#"):
                continue
            tok = line.split()
            if tok[0] == "name":
                name = tok[1] if len(tok) > 1 else ""
            elif tok[0] == "rows":
                rows = int(tok[1])
            elif tok[0] == "key_unique":
                unique = int(tok[1]) != 0
            elif tok[0] == "column":
                if len(tok) < 4:
                    raise A.SchemaError(f"malformed column line: {line}")
                if tok[2] not in ("u32", "u64"):
                    raise A.SchemaError(f"unknown column kind in manifest: {tok[2]}")
                dt = np.dtype("<u4" if tok[2] == "u32" else "<u8")
                a = np.fromfile(os.path.join(path, tok[3]), dtype=dt, count=rows)
                if len(a) != rows:
                    raise A.SchemaError(f"column file shorter than the manifest row count: {tok[3]}")
                if tok[1] == "key":
                    key = a
                else:
                    pays.append(a)
            else:
                raise A.SchemaError(f"unknown manifest field: {tok[0]}")
    if key is None:
        raise A.SchemaError("manifest lists no key column")
    if ctx is not None:
        key, pays = to_device(key), [to_device(p) for p in pays]
    return Relation(key, pays, name, unique)
