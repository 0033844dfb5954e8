"""ctypes binding of libapb_b200.so (the C ABI of include/apb.h).

The product path fails loudly when the CUDA extension is missing: there is no
CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

from .balls import (apb_balls, apb_dot_index, apb_dot_state, apb_dot_tuning, apb_mat,
                    apb_matmul_stats, apb_plan_info)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("APB_LIB_PATH") or os.path.join(HERE, "libapb_b200.so")  # override: tuning variants

_lib = None


class ApbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(ApbError, ValueError):
    """std::invalid_argument in the reference"""


class OverflowErrorApb(ApbError, OverflowError):
    """std::overflow_error in the reference"""


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -m paper_1901_04289_b200.build or __graft_entry__.build()); "
            "there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    I64 = C.c_int64
    I = C.c_int
    bp = C.POINTER(apb_balls)
    L.apb_dot_batch.argtypes = [bp, bp, bp, I, C.POINTER(apb_dot_index), I64, I64, I64, I,
                                C.POINTER(apb_dot_tuning), bp, P, P, I64, P]
    L.apb_dot_batch.restype = I
    L.apb_dot_complex_batch.argtypes = [bp, bp, bp, bp, C.POINTER(apb_dot_index), I64, I64, I64, I,
                                        C.POINTER(apb_dot_tuning), bp, bp, P, P]
    L.apb_dot_complex_batch.restype = I
    mp = C.POINTER(apb_mat)
    L.apb_matmul.argtypes = [mp, mp, I64, I, mp, P]
    L.apb_matmul.restype = I
    L.apb_matmul_complex.argtypes = [mp, mp, mp, mp, I64, I, mp, mp, P]
    L.apb_matmul_complex.restype = I
    L.apb_block_int_product.argtypes = [mp, mp, I64, I64, P, P, P, I64, P]
    L.apb_block_int_product.restype = I
    L.apb_block_int_product_imad.argtypes = [mp, mp, I64, I64, P, P, P, I64, P, P]
    L.apb_block_int_product_imad.restype = I
    L.apb_plan_blocks.argtypes = [mp, mp, I64, P, I64, P, P]
    L.apb_plan_blocks.restype = I
    L.apb_radius_matmul_upper.argtypes = [P, P, P, P, I64, I64, I64, P, P, P]
    L.apb_radius_matmul_upper.restype = I
    L.apb_dot_batch_host.argtypes = [bp, bp, bp, I, C.POINTER(apb_dot_index), I64, I64, I64, I, bp]
    L.apb_dot_batch_host.restype = I
    L.apb_matmul_host.argtypes = [mp, mp, I64, I, mp]
    L.apb_matmul_host.restype = I
    L.apb_matmul_host_submit.argtypes = [mp, mp, I64, I, mp]
    L.apb_matmul_host_submit.restype = I
    L.apb_matmul_host_drain.argtypes = []
    L.apb_matmul_host_drain.restype = I
    L.apb_poly_mullow.argtypes = [bp, I64, bp, I64, I64, I64, bp, P]
    L.apb_poly_mullow.restype = I
    L.apb_series_exp.argtypes = [bp, I64, I64, I64, bp, P]
    L.apb_series_exp.restype = I
    L.apb_poly_mullow_host.argtypes = [bp, I64, bp, I64, I64, I64, bp]
    L.apb_poly_mullow_host.restype = I
    L.apb_series_exp_host.argtypes = [bp, I64, I64, I64, bp]
    L.apb_series_exp_host.restype = I
    L.apb_balls_format.argtypes = [bp, I64, I64, C.c_char_p, I64]
    L.apb_balls_format.restype = I64
    L.apb_balls_parse.argtypes = [C.c_char_p, I64, bp, I64]
    L.apb_balls_parse.restype = I64
    L.apb_mat_format.argtypes = [mp, C.c_char_p, I64]
    L.apb_mat_format.restype = I64
    L.apb_mat_parse.argtypes = [C.c_char_p, I64, mp]
    L.apb_mat_parse.restype = I
    L.apb_device_status.argtypes = [P]
    L.apb_device_status.restype = I
    L.apb_matmul_stats_get.restype = C.POINTER(apb_matmul_stats)
    L.apb_matmul_stats_reset.restype = None
    L.apb_last_error.restype = C.c_char_p
    L.apb_launch_count.restype = C.c_uint64
    L.apb_version.restype = I
    L.apb_matmul_plan_info.argtypes = [mp, mp, I64, C.POINTER(apb_plan_info), P]
    L.apb_matmul_plan_info.restype = I
    L.apb_profile_enable.argtypes = [I]
    L.apb_profile_enable.restype = None
    L.apb_profile_reset.restype = None
    L.apb_profile_read.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
    L.apb_profile_read.restype = I
    L.apb_profile_dump.argtypes = [C.c_char_p, C.c_size_t]
    L.apb_profile_dump.restype = I
    L.apb_gemm_timer_read.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    L.apb_gemm_timer_read.restype = I
    L.apb_gemm_last_config.argtypes = [C.POINTER(C.c_int)] * 4
    L.apb_gemm_last_config.restype = I
    L.apb_gemm_timer_reset.argtypes = []
    L.apb_gemm_timer_reset.restype = I
    _lib = L
    return L


def check(rc: int, what: str = ""):
    if rc == 0:
        return
    msg = lib().apb_last_error().decode(errors="replace")
    if rc == 1:
        raise InvalidArgument(rc, f"{what}: {msg}")
    if rc == 2:
        raise OverflowErrorApb(rc, f"{what}: {msg}")
    raise ApbError(rc, f"{what}: {msg}")


def last_error() -> str:
    return lib().apb_last_error().decode(errors="replace")
