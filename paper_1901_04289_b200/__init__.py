"""B200-native ball dot product / block ball matmul (arXiv 1901.04289 hot path).

The product is libapb_b200.so (CUDA kernels for sm_100a behind the C ABI in
include/apb.h); this package is the host-side mirror of the reference's
operator surface (ops.py), the SoA ball arrays (balls.py) and the synthetic
config generators (gen.py).
"""
from .balls import (APB_FINITE, APB_NAN, APB_NINF, APB_PINF, APB_RAD_INF, APB_SIGN, APB_ZERO,
                    BallArray, DeviceBallArray, apb_dot_index, flat_index, limbs_for)

__all__ = ["BallArray", "DeviceBallArray", "apb_dot_index", "flat_index", "limbs_for",
           "APB_ZERO", "APB_FINITE", "APB_PINF", "APB_NINF", "APB_NAN", "APB_SIGN", "APB_RAD_INF"]

