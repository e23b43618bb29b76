"""B200-native equi-join path of arXiv 2312.00720 (PHJ / SMJ / NPHJ x GFUR / GFTR).

The compute path is libcoljoin_b200.so (hand-written sm_100a kernels behind the
C-ABI in include/cj_api.h).  This package is the Python host mirror of the
reference operator API; see DESIGN.md.
"""
from ._capi import (CJ_MAX_COLS, Error, LengthMismatch, KindError, FanoutTooLarge,  # noqa: F401
                    IndexOutOfBounds, EmptyInput, NotSorted, DuplicateBuildKeys,
                    FanoutMismatch, CapacityExceeded, TransformMismatch, SpecInvalid,
                    Unsupported, UnknownShape, SchemaError, build, lib, exported_symbols)
from .coljoin import (Context, Relation, JoinOutput, PhaseReport, histogram,  # noqa: F401
                      exclusive_prefix_sum, radix_partition, radix_partition_passes, sort_pairs,
                      sort_keys, gather, gather_clusteredness, partition_relation,
                      hash_find_matches, merge_find_matches, run_join, run_join_host,
                      run_join_presorted, gen_pk_fk, to_device, to_host, options, run_join_sequence, gen_star,
                      SequenceStep, export_relation, import_relation)

__all__ = [n for n in dir() if not n.startswith("_")]
