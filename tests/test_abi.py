"""The C-ABI library loads and exports every symbol include/commdyn_cuda.h
declares (CPU: no compute calls)."""

import ctypes
import os
import re

from paper_2203_16657_b200 import _lib
from paper_2203_16657_b200.build import build_library

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(REPO, "include", "commdyn_cuda.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(cdk_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_header_symbols():
    path = build_library()
    lib = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in the header but not exported"
    # every declared symbol is bound by the Python loader with a signature
    assert set(syms) <= set(_lib.EXPORTED), set(syms) - set(_lib.EXPORTED)


def test_library_host_only_calls():
    lib = _lib.load_library(build_library())
    assert lib.cdk_abi_version() == _lib.ABI_VERSION
    assert lib.cdk_launch_count() >= 0
    assert isinstance(lib.cdk_last_error(), (bytes, type(None)))


def test_struct_layout_matches_header():
    # 2 int64 + 5 pointers + 6 int32 + 9 pointers + ... + 7 ELL pointers
    assert ctypes.sizeof(_lib.CdkGraph) == (8 * 2 + 8 * 5 + 4 * 6 + 8 * 9 + 4 * 2 + 8 + 4 * 2 + 8
                                            + 8 * 7)
    assert _lib.CdkGraph.ell_off.offset == 184
    assert ctypes.sizeof(_lib.CdkRunStatus) == 32
