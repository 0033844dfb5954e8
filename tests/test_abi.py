"""CPU: the C-ABI library loads and exports every symbol include/apb.h declares
(no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1901_04289_b200", "libapb_b200.so")


def declared():
    src = open(os.path.join(ROOT, "include", "apb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(apb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("apb_dot_batch", "apb_dot_complex_batch", "apb_matmul", "apb_matmul_complex",
                 "apb_block_int_product", "apb_plan_blocks", "apb_radius_matmul_upper",
                 "apb_dot_batch_host", "apb_matmul_host", "apb_last_error", "apb_device_status"):
        assert must in names


def test_library_exports_all_symbols():
    if not os.path.exists(LIB):
        pytest.skip("libapb_b200.so not built (run __graft_entry__.build())")
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (apb_[a-z0-9_]+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_library_loads_and_reports_version():
    if not os.path.exists(LIB):
        pytest.skip("libapb_b200.so not built")
    lib = ctypes.CDLL(LIB)
    lib.apb_version.restype = ctypes.c_int
    assert lib.apb_version() >= 1
    lib.apb_launch_count.restype = ctypes.c_uint64
    assert lib.apb_launch_count() == 0
