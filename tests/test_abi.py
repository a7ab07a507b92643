"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/sptrsv.h declares, and its host-side argument checks work
without a GPU (no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sptrsv.h")


@pytest.fixture(scope="module")
def S():
    from paper_1710_04985_b200 import build
    build.build()
    from paper_1710_04985_b200 import sptrsv
    return sptrsv


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sptrsv_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for required in ("sptrsv_analyze", "sptrsv_solve", "sptrsv_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol(S):
    lib = ctypes.CDLL(S.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_library_is_sm100a_only(S):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", S.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_status_strings(S):
    for code, name in S.STATUS_NAMES.items():
        assert S.sptrsv_status_string(code) == "SPTRSV_" + ("ERR_" if code else "") + name
    assert S.sptrsv_status_string(99) == "SPTRSV_UNKNOWN_STATUS"


def test_host_side_argument_checks(S):
    # rejected before any CUDA call
    assert S.sptrsv_analyze(-1, None, None, None, 0, 0, 0, None) == (1, None)
    assert S.sptrsv_analyze(4, None, None, None, 0, 0, 0, None)[0] == 1
    dummy = ctypes.c_void_p(16)
    assert S.sptrsv_analyze(4, dummy, dummy, dummy, 2, 0, 0, None)[0] == 1      # bad uplo
    assert S.sptrsv_analyze(4, dummy, dummy, dummy, 0, 5, 0, None)[0] == 1      # bad diag
    assert S.sptrsv_analyze(4, dummy, dummy, dummy, 0, 0, 7, None)[0] == 1      # bad dtype
    assert S.sptrsv_analyze(4, dummy, dummy, None, 0, 0, 0, None)[0] == 1       # NON_UNIT needs vals
    assert S.sptrsv_solve(None, None, None, 1, None) == 1
    assert S.sptrsv_solve_host(None, None, None, 1, None) == 1
    assert S.sptrsv_set_algo(None, 0) == 1
    assert S.sptrsv_get_levels(None, None, None, None) == 1
    assert S.sptrsv_get_dep_counts(None, None) == 1
    assert S.sptrsv_get_info(None)[0] == 1
    assert S.sptrsv_update_values(None, None, None, None, None) == 1
    assert S.sptrsv_destroy(None) == 0


def test_info_struct_layout_matches_header(S):
    # field order/size of sptrsv_info_t must mirror the header
    src = open(HEADER).read()
    body = re.search(r"typedef struct \{(.*?)\} sptrsv_info_t;", src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        typ, rest = decl.split(None, 1)
        for name in rest.split(","):
            fields.append((name.strip(), typ))
    assert [f for f, _ in fields] == [f for f, _ in S.sptrsv_info_t._fields_]
    size = {"int32_t": 4, "int64_t": 8, "double": 8}
    for (name, typ), (_, ctyp) in zip(fields, S.sptrsv_info_t._fields_):
        assert size[typ] == ctypes.sizeof(ctyp), name


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1710_04985_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", text).replace("oracle/", ""), f
                assert "import workloads" not in text, f


def test_build_digest_identifies_sources_and_keys_the_traffic():
    """The build digest (sha256 of the library sources and nvcc flags) is
    stable, and bench.py's roofline.traffic resolves only for a matching one
    (profiles/ncu_traffic.json is keyed by it)."""
    import sys
    from paper_1710_04985_b200 import build
    d1, d2 = build.source_digest(), build.source_digest()
    assert d1 == d2 and re.fullmatch(r"[0-9a-f]{64}", d1)
    sys.path.insert(0, ROOT)
    import bench
    assert bench.ncu_traffic("cfg2_k_block_f64", "0" * 64) is None
    assert bench.ncu_traffic("no_such_key", d1) is None
