"""ctypes front-end of the C restatement (oracle/cj_oracle.c) and of the
reference driver (oracle/_ref/refjoin).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference leg may import this module, and only as the checker.
Every column crosses this boundary widened to uint64 (see cj_oracle.h).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libcjoracle.so")
REFJOIN = os.path.join(HERE, "_ref", "refjoin")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_lib = None


def build() -> None:
    """Compile the C port (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)
        if os.path.exists(os.path.join(HERE, "..", "paper_2312_00720_b200", "libcoljoin_host.so")):
            subprocess.run(["make", "-s", "-j8", "-C", HERE, "dropin"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.cjo_mix64.restype = C.c_uint64
        L.cjo_mix64.argtypes = [C.c_uint64]
        L.cjo_digest.restype = C.c_uint64
        L.cjo_digest.argtypes = [_u64p, C.c_uint64]
        L.cjo_digest_continue.restype = C.c_uint64
        L.cjo_digest_continue.argtypes = [C.c_uint64, _u64p, C.c_uint64, C.c_uint64]
        L.cjo_gen_pk_fk.argtypes = [C.c_uint64, C.c_uint64, C.c_uint, C.c_uint, C.c_double,
                                    C.c_double, C.c_uint64, C.c_uint, _u64p, _u64p, _u64p, _u64p]
        L.cjo_default_total_radix_bits.restype = C.c_uint
        L.cjo_default_total_radix_bits.argtypes = [C.c_uint64]
        L.cjo_radix_partition.argtypes = [_u64p, _u64p, C.c_uint, C.c_uint64, C.c_uint, C.c_uint,
                                          C.c_uint, _u64p, _u64p, _u64p]
        L.cjo_sort_pairs.argtypes = [_u64p, _u64p, C.c_uint, C.c_uint64, C.c_uint, _u64p, _u64p]
        L.cjo_partition_relation.argtypes = [_u64p, _u64p, C.c_uint, C.c_uint64, C.c_uint,
                                             C.c_uint, C.c_uint, _u64p, _u64p, _u64p]
        L.cjo_gather.argtypes = [_u64p, C.c_uint64, _u32p, C.c_uint64, _u64p]
        L.cjo_hash_find_matches.argtypes = [_u64p, _u64p, C.c_uint64, _u64p, _u64p, C.c_uint64,
                                            C.c_uint, C.c_uint32, C.POINTER(C.c_uint64),
                                            C.c_void_p, C.c_void_p, C.c_void_p]
        L.cjo_merge_find_matches.argtypes = [_u64p, C.c_uint64, _u64p, C.c_uint64, C.c_int,
                                             C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p,
                                             C.c_void_p]
        L.cjo_run_join.argtypes = [C.c_int, C.c_int, _u64p, _u64p, C.c_uint, C.c_uint64, C.c_int,
                                   _u64p, _u64p, C.c_uint, C.c_uint64, C.c_uint, C.c_int,
                                   C.c_uint32, C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
        L.cjo_canonical_digest.restype = C.c_uint64
        L.cjo_canonical_digest.argtypes = [C.POINTER(C.c_void_p), C.c_uint, C.c_uint64]
        L.cjo_nested_loop_join.argtypes = [_u64p, _u64p, C.c_uint, C.c_uint64, _u64p, _u64p,
                                           C.c_uint, C.c_uint64, C.POINTER(C.c_uint64),
                                           C.c_void_p]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


def _chk(code: int, what: str) -> None:
    if code != 0:
        raise OracleError(code, what)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a).astype(np.uint64, copy=False))


def _cols(cols, n) -> np.ndarray:
    """Column-major block (ncols * n) of widened columns."""
    if not cols:
        return np.zeros(1, np.uint64)
    return np.ascontiguousarray(np.concatenate([_u64(c) for c in cols]))


def mix64(x: int) -> int:
    return int(lib().cjo_mix64(x))


def digest(words) -> int:
    w = _u64(words).ravel()
    return int(lib().cjo_digest(w if w.size else np.zeros(1, np.uint64), w.size))


class DigestStream:
    """digest() of a long word sequence fed in pieces (BASELINE.md §2 formula)."""

    def __init__(self):
        self.h, self.i = 0x12345678, 0

    def update(self, words):
        w = np.ascontiguousarray(_u64(words).ravel())
        if w.size:
            self.h = int(lib().cjo_digest_continue(self.h, w, w.size, self.i))
            self.i += w.size
        return self


def default_total_radix_bits(build_rows: int) -> int:
    return int(lib().cjo_default_total_radix_bits(build_rows))


def gen_pk_fk(r_rows, s_rows, r_pay=1, s_pay=1, match=1.0, zipf=0.0, seed=42, pay_bytes=4,
              key_bytes=4):
    """workloads.cpp:89-133.  Returns (R, S) as dicts of numpy columns whose
    dtypes follow the key/payload kinds."""
    rk = np.empty(max(r_rows, 1), np.uint64)
    sk = np.empty(max(s_rows, 1), np.uint64)
    rp = np.empty(max(r_rows * r_pay, 1), np.uint64)
    sp = np.empty(max(s_rows * s_pay, 1), np.uint64)
    _chk(lib().cjo_gen_pk_fk(r_rows, s_rows, r_pay, s_pay, match, zipf, seed, pay_bytes,
                             rk, rp, sk, sp), "gen_pk_fk")
    kt = np.uint32 if key_bytes == 4 else np.uint64
    pt = np.uint32 if pay_bytes == 4 else np.uint64
    R = {"key": rk[:r_rows].astype(kt),
         "payloads": [rp[c * r_rows:(c + 1) * r_rows].astype(pt) for c in range(r_pay)]}
    S = {"key": sk[:s_rows].astype(kt),
         "payloads": [sp[c * s_rows:(c + 1) * s_rows].astype(pt) for c in range(s_pay)]}
    return R, S


def radix_partition(keys, vals, lo, hi, key_bytes=4):
    k = _u64(keys)
    n = k.size
    v = _cols(vals, n)
    ko = np.empty(max(n, 1), np.uint64)
    vo = np.empty(max(n * len(vals), 1), np.uint64)
    off = np.empty((1 << (hi - lo)) + 1 if hi >= lo and hi - lo <= 8 else 2, np.uint64)
    _chk(lib().cjo_radix_partition(k if n else np.zeros(1, np.uint64), v, len(vals), n,
                                   key_bytes, lo, hi, ko, vo, off), "radix_partition")
    return ko[:n], [vo[c * n:(c + 1) * n] for c in range(len(vals))], off


def sort_pairs(keys, vals, key_bytes=4):
    k = _u64(keys)
    n = k.size
    v = _cols(vals, n)
    ko = np.empty(max(n, 1), np.uint64)
    vo = np.empty(max(n * len(vals), 1), np.uint64)
    _chk(lib().cjo_sort_pairs(k if n else np.zeros(1, np.uint64), v, len(vals), n, key_bytes,
                              ko, vo), "sort_pairs")
    return ko[:n], [vo[c * n:(c + 1) * n] for c in range(len(vals))]


def partition_relation(keys, vals, total_bits, bits_per_pass=8, key_bytes=4):
    k = _u64(keys)
    n = k.size
    v = _cols(vals, n)
    ko = np.empty(max(n, 1), np.uint64)
    vo = np.empty(max(n * len(vals), 1), np.uint64)
    off = np.empty((1 << total_bits) + 1 if total_bits <= 20 else 2, np.uint64)
    _chk(lib().cjo_partition_relation(k if n else np.zeros(1, np.uint64), v, len(vals), n,
                                      key_bytes, total_bits, bits_per_pass, ko, vo, off),
         "partition_relation")
    if total_bits == 0:
        off = off[:2]
    return ko[:n], [vo[c * n:(c + 1) * n] for c in range(len(vals))], off


def gather(col, idx):
    c = _u64(col)
    m = np.ascontiguousarray(np.asarray(idx, np.uint32))
    out = np.empty(max(m.size, 1), np.uint64)
    _chk(lib().cjo_gather(c if c.size else np.zeros(1, np.uint64), c.size,
                          m if m.size else np.zeros(1, np.uint32), m.size, out), "gather")
    return out[:m.size]


def hash_find_matches(bkeys, boff, pkeys, poff, limit=4096):
    bk, bo, pk, po = _u64(bkeys), _u64(boff), _u64(pkeys), _u64(poff)
    fan = bo.size - 1
    tot = C.c_uint64(0)
    z = np.zeros(1, np.uint64)
    bk_ = bk if bk.size else z
    pk_ = pk if pk.size else z
    _chk(lib().cjo_hash_find_matches(bk_, bo, bk.size, pk_, po, pk.size, fan, limit,
                                     C.byref(tot), None, None, None), "hash count")
    t = tot.value
    keys = np.empty(max(t, 1), np.uint64)
    ir = np.empty(max(t, 1), np.uint32)
    js = np.empty(max(t, 1), np.uint32)
    _chk(lib().cjo_hash_find_matches(bk_, bo, bk.size, pk_, po, pk.size, fan, limit,
                                     C.byref(tot), keys.ctypes.data, ir.ctypes.data,
                                     js.ctypes.data), "hash fill")
    return keys[:t], ir[:t], js[:t]


def merge_find_matches(r_sorted, s_sorted, pk_fk):
    r, s = _u64(r_sorted), _u64(s_sorted)
    z = np.zeros(1, np.uint64)
    tot = C.c_uint64(0)
    _chk(lib().cjo_merge_find_matches(r if r.size else z, r.size, s if s.size else z, s.size,
                                      int(pk_fk), C.byref(tot), None, None, None), "merge count")
    t = tot.value
    keys = np.empty(max(t, 1), np.uint64)
    ir = np.empty(max(t, 1), np.uint32)
    js = np.empty(max(t, 1), np.uint32)
    _chk(lib().cjo_merge_find_matches(r if r.size else z, r.size, s if s.size else z, s.size,
                                      int(pk_fk), C.byref(tot), keys.ctypes.data,
                                      ir.ctypes.data, js.ctypes.data), "merge fill")
    return keys[:t], ir[:t], js[:t]


ALGOS = {"smj": 0, "phj": 1}
PATTERNS = {"gfur": 0, "gftr": 1}


def run_join(R, S, algo="phj", pattern="gftr", key_bytes=None, total_bits=-1, limit=4096,
             r_key_unique=True):
    """join_engine.cpp:255-361.  Returns dict(key, payloads, ids_r, ids_s)."""
    rk, sk = _u64(R["key"]), _u64(S["key"])
    if key_bytes is None:
        key_bytes = np.asarray(R["key"]).dtype.itemsize
    nr, ns = rk.size, sk.size
    rp, sp = _cols(R["payloads"], nr), _cols(S["payloads"], ns)
    z = np.zeros(1, np.uint64)
    rows = C.c_uint64(0)
    args = (ALGOS[algo], PATTERNS[pattern], rk if nr else z, rp, len(R["payloads"]), nr,
            int(r_key_unique), sk if ns else z, sp, len(S["payloads"]), ns, key_bytes,
            total_bits, limit, C.byref(rows))
    _chk(lib().cjo_run_join(*args, None, None, None, None), "run_join count")
    t = rows.value
    npay = len(R["payloads"]) + len(S["payloads"])
    okey = np.empty(max(t, 1), np.uint64)
    opay = np.empty(max(t * npay, 1), np.uint64)
    ir = np.empty(max(t, 1), np.uint32)
    js = np.empty(max(t, 1), np.uint32)
    _chk(lib().cjo_run_join(*args, okey.ctypes.data, opay.ctypes.data, ir.ctypes.data,
                            js.ctypes.data), "run_join fill")
    return {"key": okey[:t], "payloads": [opay[c * t:(c + 1) * t] for c in range(npay)],
            "ids_r": ir[:t], "ids_s": js[:t]}


def canonical_digest(cols) -> int:
    """oracle.cpp:77-88 canonical rows + BASELINE.md §2 digest."""
    arrs = [_u64(c) for c in cols]
    n = arrs[0].size if arrs else 0
    ptrs = (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])
    return int(lib().cjo_canonical_digest(ptrs, len(arrs), n))


def nested_loop_join(R, S):
    rk, sk = _u64(R["key"]), _u64(S["key"])
    nr, ns = rk.size, sk.size
    rp, sp = _cols(R["payloads"], nr), _cols(S["payloads"], ns)
    z = np.zeros(1, np.uint64)
    rows = C.c_uint64(0)
    a = (rk if nr else z, rp, len(R["payloads"]), nr, sk if ns else z, sp, len(S["payloads"]), ns,
         C.byref(rows))
    _chk(lib().cjo_nested_loop_join(*a, None), "nested_loop count")
    w = 1 + len(R["payloads"]) + len(S["payloads"])
    out = np.empty(max(rows.value * w, 1), np.uint64)
    _chk(lib().cjo_nested_loop_join(*a, out.ctypes.data), "nested_loop fill")
    return out[:rows.value * w].reshape(rows.value, w)


# ---- reference driver (oracle/_ref/refjoin) --------------------------------

def refjoin_available() -> bool:
    return os.access(REFJOIN, os.X_OK)


def refjoin(*args: str, env=None, timeout=None) -> dict:
    out = subprocess.run([REFJOIN, *args], check=True, capture_output=True, text=True,
                         env=env, timeout=timeout)
    return json.loads(out.stdout.strip().splitlines()[-1])
