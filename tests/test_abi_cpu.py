"""CPU checks of the drop-in boundary: the C-ABI library and the C++ host
library load and export every symbol include/cj_api.h declares; the headers
compile as C and as C++; status codes mirror the reference's error classes."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "cj_api.h")
LIB = os.path.join(ROOT, "paper_2312_00720_b200", "libcoljoin_b200.so")
HOST = os.path.join(ROOT, "paper_2312_00720_b200", "libcoljoin_host.so")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cj_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("cj_run_join", "cj_run_join_host", "cj_radix_partition", "cj_sort_pairs",
                 "cj_gather", "cj_partition_relation", "cj_hash_find_matches",
                 "cj_merge_find_matches", "cj_shard_partition", "cj_gen_pk_fk"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2312_00720_b200 import _capi
    assert set(declared()) <= set(_capi.PROTOS) | {"cj_default_options"}


def test_header_compiles_as_c_and_cpp(tmp_path):
    for lang, cc in (("c", "/usr/bin/gcc"), ("c++", "/usr/bin/g++")):
        f = tmp_path / ("t." + ("c" if lang == "c" else "cpp"))
        f.write_text('#include "cj_api.h"\nint main(void) { return CJ_OK; }\n')
        subprocess.run([cc, "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-c",
                        str(f), "-o", str(tmp_path / "t.o")], check=True)


def test_cpp_host_library_exports_the_reference_api():
    out = subprocess.run(["nm", "-D", "-C", "--defined-only", HOST], capture_output=True,
                         text=True, check=True).stdout
    for sym in ("coljoin::run_join(coljoin::JoinTask const&)",
                "coljoin::primitives::radix_partition(", "coljoin::primitives::sort_pairs(",
                "coljoin::primitives::gather(", "coljoin::hashjoin::partition_relation(",
                "coljoin::hashjoin::hash_find_matches(", "coljoin::mergejoin::merge_find_matches(",
                "coljoin::materialize_gftr(", "coljoin::materialize_gfur("):
        assert sym in out, sym


def test_status_codes_mirror_reference_errors():
    from paper_2312_00720_b200 import _capi as A
    names = ["LengthMismatch", "KindError", "FanoutTooLarge", "IndexOutOfBounds", "EmptyInput",
             "NotSorted", "DuplicateBuildKeys", "FanoutMismatch", "CapacityExceeded",
             "TransformMismatch", "PhaseOrderViolation", "SpecInvalid", "UnknownShape",
             "SchemaError", "Unsupported"]
    src = open(HDR).read()
    for i, n in enumerate(names, 1):
        assert getattr(A, n).code == i
        assert re.search(rf"= {i},\s*/\* {n}", src), n


def test_no_device_means_loud_failure():
    import paper_2312_00720_b200 as cj
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(Exception):
        cj.Context(0)
