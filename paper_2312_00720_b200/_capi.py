"""ctypes binding of the C-ABI (include/cj_api.h) exported by libcoljoin_b200.so.

There is no fallback: if the shared library is missing or no CUDA device is
present, every entry point raises.  Status codes map 1:1 to exception classes
named after the reference's (include/coljoin/errors.hpp:19-33).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcoljoin_b200.so")
CSRC = os.path.join(HERE, "csrc")

CJ_MAX_COLS = 16
CJ_MAX_PASSES = 8
SMJ, PHJ, NPHJ = 0, 1, 2
GFUR, GFTR = 0, 1
IDS_PHYSICAL, IDS_VIRTUAL = 0, 1


class Error(RuntimeError):
    """coljoin::Error (errors.hpp:8-10)."""
    code = -1


def _mk(name, code):
    return type(name, (Error,), {"code": code})


LengthMismatch = _mk("LengthMismatch", 1)
KindError = _mk("KindError", 2)
FanoutTooLarge = _mk("FanoutTooLarge", 3)
IndexOutOfBounds = _mk("IndexOutOfBounds", 4)
EmptyInput = _mk("EmptyInput", 5)
NotSorted = _mk("NotSorted", 6)
DuplicateBuildKeys = _mk("DuplicateBuildKeys", 7)
FanoutMismatch = _mk("FanoutMismatch", 8)
CapacityExceeded = _mk("CapacityExceeded", 9)
TransformMismatch = _mk("TransformMismatch", 10)
PhaseOrderViolation = _mk("PhaseOrderViolation", 11)
SpecInvalid = _mk("SpecInvalid", 12)
UnknownShape = _mk("UnknownShape", 13)
SchemaError = _mk("SchemaError", 14)
Unsupported = _mk("Unsupported", 15)
CudaError = _mk("CudaError", 100)
NcclError = _mk("NcclError", 101)
DeviceOutOfMemory = _mk("DeviceOutOfMemory", 102)
_BY_CODE = {c.code: c for c in (LengthMismatch, KindError, FanoutTooLarge, IndexOutOfBounds,
                                EmptyInput, NotSorted, DuplicateBuildKeys, FanoutMismatch,
                                CapacityExceeded, TransformMismatch, PhaseOrderViolation,
                                SpecInvalid, UnknownShape, SchemaError, Unsupported, CudaError,
                                NcclError, DeviceOutOfMemory)}


class Relation(C.Structure):
    _fields_ = [("key", C.c_void_p), ("key_bytes", C.c_uint32), ("rows", C.c_uint64),
                ("npay", C.c_uint32), ("pay", C.c_void_p * CJ_MAX_COLS),
                ("pay_bytes", C.c_uint32 * CJ_MAX_COLS), ("key_unique", C.c_int)]


class JoinOptions(C.Structure):
    _fields_ = [("algo", C.c_int), ("pattern", C.c_int), ("radix_bits_per_pass", C.c_uint32),
                ("total_radix_bits", C.c_int), ("sub_partition_limit", C.c_uint32),
                ("validate", C.c_int), ("want_ids", C.c_int), ("want_stats", C.c_int)]


class JoinResult(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("key", C.c_void_p), ("pay", C.c_void_p * (2 * CJ_MAX_COLS)),
                ("ids_r", C.c_void_p), ("ids_s", C.c_void_p), ("transform_ns", C.c_uint64),
                ("find_ns", C.c_uint64), ("materialize_ns", C.c_uint64),
                ("clusteredness_r", C.c_double), ("clusteredness_s", C.c_double),
                ("device_bytes_peak", C.c_uint64), ("peak_transform_b", C.c_uint64),
                ("peak_find_b", C.c_uint64), ("peak_materialize_b", C.c_uint64),
                ("ledger_column_b", C.c_uint64 * 3), ("ledger_scratch_b", C.c_uint64 * 3)]


class SequenceStep(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("output_columns", C.c_uint32),
                ("transform_ns", C.c_uint64), ("find_ns", C.c_uint64),
                ("materialize_ns", C.c_uint64), ("fk_fetch_ns", C.c_uint64)]


class ShuffleStats(C.Structure):
    _fields_ = [("first_bits", C.c_uint32), ("r_rows_received", C.c_uint64),
                ("s_rows_received", C.c_uint64), ("bytes_sent_peers", C.c_uint64),
                ("bytes_received_peers", C.c_uint64), ("shard_ns", C.c_uint64),
                ("exchange_r_ns", C.c_uint64), ("exchange_s_ns", C.c_uint64),
                ("wall_ns", C.c_uint64)]


class Partitioned(C.Structure):
    _fields_ = [("keys", C.c_void_p), ("offsets", C.c_void_p), ("carried", C.c_void_p),
                ("rows", C.c_uint64)]


HOST_ALLOC = C.CFUNCTYPE(C.c_void_p, C.c_uint64, C.c_void_p)

_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_U32P = C.POINTER(C.c_uint32)
_U64P = C.POINTER(C.c_uint64)

PROTOS = {
    "cj_ctx_create": (C.c_int, [C.c_int, _P, C.POINTER(_P)]),
    "cj_ctx_destroy": (C.c_int, [_P]),
    "cj_ctx_stream": (_P, [_P]),
    "cj_last_error": (C.c_char_p, [_P]),
    "cj_sync": (C.c_int, [_P]),
    "cj_free": (C.c_int, [_P, _P]),
    "cj_alloc": (C.c_int, [_P, C.c_uint64, C.POINTER(_P)]),
    "cj_launch_count": (C.c_uint64, [_P]),
    "cj_mark": (C.c_int, [_P, C.c_int]),
    "cj_elapsed_ms": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "cj_histogram": (C.c_int, [_P, _P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, _U32P]),
    "cj_radix_partition": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                     _PP, _PP, _U32P, C.c_uint32, _U64P]),
    "cj_radix_partition_passes": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, _U32P, _U32P,
                                            C.c_uint32, _PP, _PP, _U32P, C.c_uint32, C.c_int]),
    "cj_sort_pairs": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, _PP, _PP, _U32P, C.c_uint32,
                                C.c_int]),
    "cj_gather": (C.c_int, [_P, _PP, C.c_uint64, _P, C.c_uint64, _PP, _U32P, C.c_uint32]),
    "cj_partition_relation": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, C.c_uint32,
                                        C.c_uint32, _PP, _PP, _U32P, C.c_uint32, C.c_int, _P]),
    "cj_hash_find_matches": (C.c_int, [_P, C.POINTER(Partitioned), C.POINTER(Partitioned),
                                       C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _U64P,
                                       C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "cj_merge_find_matches": (C.c_int, [_P, _P, C.c_uint64, _P, C.c_uint64, C.c_uint32, C.c_int,
                                        C.c_int, _U64P, C.POINTER(_P), C.POINTER(_P),
                                        C.POINTER(_P)]),
    "cj_default_options": (None, [C.POINTER(JoinOptions)]),
    "cj_run_join": (C.c_int, [_P, C.POINTER(Relation), C.POINTER(Relation),
                              C.POINTER(JoinOptions), C.POINTER(JoinResult)]),
    "cj_result_free": (C.c_int, [_P, C.POINTER(JoinResult)]),
    "cj_run_join_host": (C.c_int, [_P, C.POINTER(Relation), C.POINTER(Relation),
                                   C.POINTER(JoinOptions), HOST_ALLOC, _P,
                                   C.POINTER(JoinResult), _U64P, _U64P]),
    "cj_shard_partition": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, C.c_uint32, _PP, _PP,
                                     _U32P, C.c_uint32, _U64P]),
    "cj_shard_partition_ex": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, C.c_uint32,
                                        C.c_uint32, _PP, _PP, _U32P, C.c_uint32, _U64P]),
    "cj_exchange_plan": (C.c_int, [C.c_uint32, C.c_uint32, _U64P, _U64P, _U64P, _U64P, _U64P]),
    "cj_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "cj_comm_init": (C.c_int, [_P, C.POINTER(C.c_uint8), C.c_int, C.c_int, C.POINTER(_P)]),
    "cj_comm_destroy": (C.c_int, [_P]),
    "cj_comm_size": (C.c_int, [_P]),
    "cj_comm_rank": (C.c_int, [_P]),
    "cj_shuffle_relation": (C.c_int, [_P, _P, C.POINTER(Relation), C.c_uint32,
                                      C.POINTER(Relation), C.POINTER(ShuffleStats)]),
    "cj_relation_free": (C.c_int, [_P, C.POINTER(Relation)]),
    "cj_run_join_presorted": (C.c_int, [_P, C.POINTER(Relation), C.POINTER(Relation),
                                        C.POINTER(JoinOptions), C.c_uint32,
                                        C.POINTER(JoinResult)]),
    "cj_run_join_sharded": (C.c_int, [_P, _P, C.POINTER(Relation), C.POINTER(Relation),
                                      C.POINTER(JoinOptions), C.POINTER(JoinResult),
                                      C.POINTER(ShuffleStats)]),
    "cj_gen_shard": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                               C.c_uint32, C.c_uint64, _P, _PP, _P, _PP]),
    "cj_set_kernel_timing": (C.c_int, [_P, C.c_int]),
    "cj_kernel_records": (C.c_int, [_P, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_float),
                                    _U64P, C.POINTER(C.c_int)]),
    "cj_copy": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_int]),
    "cj_scratch_peak": (C.c_uint64, [_P, C.c_int]),
    "cj_gen_pk_fk": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                               C.c_uint32, C.c_double, C.c_double, C.c_uint64, _P, _PP, _P, _PP]),
    "cj_run_join_sequence": (C.c_int, [_P, C.POINTER(Relation), C.POINTER(Relation), C.c_uint32,
                                       C.POINTER(JoinOptions), C.POINTER(SequenceStep),
                                       C.POINTER(JoinResult)]),
    "cj_gen_star": (C.c_int, [_P, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32,
                              C.c_uint32, _P, _PP, _PP, _PP]),
}

_lib = None


def build(force: bool = False) -> None:
    """Compile the CUDA sources for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-j8", "-C", CSRC] + (["-B"] if force else []), check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2312_00720_b200.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int, ctx=None, what: str = "") -> None:
    if status != 0:
        msg = lib().cj_last_error(ctx).decode() if ctx else ""
        raise _BY_CODE.get(status, Error)(f"{what}: {msg} (status {status})")


def exported_symbols() -> list[str]:
    return list(PROTOS)
