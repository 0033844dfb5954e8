"""Ball arrays: the SoA layout of include/apb.h on the host (numpy) and on the
device (torch CUDA tensors used purely as memory), plus the ctypes structs of
the C ABI.

A ball array holds `count` balls [m +- r] (include/apball/ball.hpp:12-40 in the
reference): mantissa limbs top-aligned in `L` slots, int64 exponent, a kind
byte (zero/finite/inf/nan + sign bit) and a 30-bit Mag radius (mantissa,
exponent) (include/apball/mag.hpp:15-59).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

APB_ZERO, APB_FINITE, APB_PINF, APB_NINF, APB_NAN = 0, 1, 2, 3, 4
APB_KIND_MASK, APB_SIGN = 7, 0x80
APB_RAD_INF = 0xFFFFFFFF
APB_DOT_BALL, APB_DOT_APPROX = 0, 1
APB_MM_AUTO, APB_MM_BLOCK, APB_MM_CLASSICAL = 0, 1, 2

STATUS_NAMES = {0: "ok", 1: "invalid_argument", 2: "overflow_error", 3: "unsupported", 4: "cuda_error"}


class apb_balls(C.Structure):
    _fields_ = [
        ("mant", C.c_void_p),
        ("exp", C.c_void_p),
        ("kind", C.c_void_p),
        ("rad_man", C.c_void_p),
        ("rad_exp", C.c_void_p),
        ("count", C.c_int64),
        ("L", C.c_int32),
    ]


class apb_dot_index(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("bdiv", "x_off", "xs1", "xs2", "xstep", "y_off", "ys1", "ys2", "ystep")]


class apb_dot_state(C.Structure):
    _fields_ = [
        ("e_max", C.c_int64), ("e_min", C.c_int64), ("e_rad", C.c_int64),
        ("n_nonzero", C.c_uint64), ("p_eff", C.c_int64),
        ("extend", C.c_int32), ("padding", C.c_int32),
        ("n_s", C.c_int64), ("e_s", C.c_int64),
        ("status", C.c_int32), ("_pad", C.c_int32),
        ("err", C.c_uint64), ("srad", C.c_uint64),
    ]


class apb_dot_tuning(C.Structure):
    _fields_ = [("disable_precision_reduction", C.c_int32), ("force_threeprod", C.c_int32),
                ("threeprod_cutoff_limbs", C.c_int64)]


class apb_mat(C.Structure):
    _fields_ = [("b", apb_balls), ("rows", C.c_int64), ("cols", C.c_int64)]


class apb_matmul_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("classical_calls", "block_calls", "int_gemm_products", "last_block_count",
                 "last_height_a", "last_height_b", "last_slices_a", "last_slices_b")]


class apb_plan_info(C.Structure):
    _fields_ = [("n_blocks", C.c_int64), ("entry_prec_a", C.c_int64), ("entry_prec_b", C.c_int64),
                ("max_width_a", C.c_int64), ("max_width_b", C.c_int64), ("special", C.c_int32),
                ("radius_single", C.c_int32)]


DOT_STATE_DTYPE = np.dtype([
    ("e_max", "<i8"), ("e_min", "<i8"), ("e_rad", "<i8"), ("n_nonzero", "<u8"),
    ("p_eff", "<i8"), ("extend", "<i4"), ("padding", "<i4"), ("n_s", "<i8"), ("e_s", "<i8"),
    ("status", "<i4"), ("_pad", "<i4"), ("err", "<u8"), ("srad", "<u8")])
assert DOT_STATE_DTYPE.itemsize == C.sizeof(apb_dot_state)


def limbs_for(prec: int) -> int:
    return max(1, (int(prec) + 63) // 64)


def flat_index(n: int) -> apb_dot_index:
    """dot b reads x[b*n + i], y[b*n + i]"""
    return apb_dot_index(1, 0, n, 0, 1, 0, n, 0, 1)


@dataclass
class BallArray:
    """Host SoA ball array (numpy)."""
    mant: np.ndarray     # uint64 [count, L]
    exp: np.ndarray      # int64 [count]
    kind: np.ndarray     # uint8 [count]
    rad_man: np.ndarray  # uint32 [count]
    rad_exp: np.ndarray  # int64 [count]

    @property
    def count(self) -> int:
        return int(self.exp.shape[0])

    @property
    def L(self) -> int:
        return int(self.mant.shape[1])

    @staticmethod
    def zeros(count: int, L: int) -> "BallArray":
        return BallArray(np.zeros((count, L), np.uint64), np.zeros(count, np.int64),
                         np.zeros(count, np.uint8), np.zeros(count, np.uint32),
                         np.zeros(count, np.int64))

    def __post_init__(self):
        self.mant = np.ascontiguousarray(self.mant, dtype=np.uint64)
        if self.mant.ndim == 1:
            self.mant = self.mant.reshape(-1, 1)
        self.exp = np.ascontiguousarray(self.exp, dtype=np.int64)
        self.kind = np.ascontiguousarray(self.kind, dtype=np.uint8)
        self.rad_man = np.ascontiguousarray(self.rad_man, dtype=np.uint32)
        self.rad_exp = np.ascontiguousarray(self.rad_exp, dtype=np.int64)

    def c(self) -> apb_balls:
        return apb_balls(self.mant.ctypes.data, self.exp.ctypes.data, self.kind.ctypes.data,
                         self.rad_man.ctypes.data, self.rad_exp.ctypes.data, self.count, self.L)

    def widen(self, L: int) -> "BallArray":
        """same values in L >= self.L limb slots (top-aligned)"""
        if L == self.L:
            return self
        assert L > self.L
        m = np.zeros((self.count, L), np.uint64)
        m[:, L - self.L:] = self.mant
        return BallArray(m, self.exp.copy(), self.kind.copy(), self.rad_man.copy(), self.rad_exp.copy())

    @staticmethod
    def from_i64(vals) -> "BallArray":
        """exact balls of small integers (Ball::from_i64, include/apball/ball.hpp:22)"""
        vals = list(vals)
        a = BallArray.zeros(len(vals), 1)
        for k, v in enumerate(vals):
            if v == 0:
                continue
            m = abs(int(v))
            bl = m.bit_length()
            a.mant[k, 0] = np.uint64(m << (64 - bl))
            a.exp[k] = bl
            a.kind[k] = APB_FINITE | (APB_SIGN if v < 0 else 0)
        return a

    def take(self, idx) -> "BallArray":
        idx = np.asarray(idx, dtype=np.int64)
        return BallArray(self.mant[idx], self.exp[idx], self.kind[idx], self.rad_man[idx], self.rad_exp[idx])

    def concat(self, other: "BallArray") -> "BallArray":
        L = max(self.L, other.L)
        a, b = self.widen(L), other.widen(L)
        return BallArray(np.concatenate([a.mant, b.mant]), np.concatenate([a.exp, b.exp]),
                         np.concatenate([a.kind, b.kind]), np.concatenate([a.rad_man, b.rad_man]),
                         np.concatenate([a.rad_exp, b.rad_exp]))

    def nbytes(self) -> int:
        return int(self.mant.nbytes + self.exp.nbytes + self.kind.nbytes + self.rad_man.nbytes
                   + self.rad_exp.nbytes)

    def identical(self, other: "BallArray") -> np.ndarray:
        """per-element ball_identical (src/ball.cpp:5-8): same kind, sign, exponent,
        limbs and Mag; compares across differing L by value"""
        L = max(self.L, other.L)
        a, b = self.widen(L), other.widen(L)
        fin = (a.kind & APB_KIND_MASK) == APB_FINITE
        same = (a.kind == b.kind) & (a.rad_man == b.rad_man)
        same &= np.where(fin, (a.exp == b.exp) & np.all(a.mant == b.mant, axis=1), True)
        radfin = (a.rad_man != 0) & (a.rad_man != APB_RAD_INF)
        same &= np.where(radfin, a.rad_exp == b.rad_exp, True)
        return same

    def pinned(self) -> "BallArray":
        """copy into page-locked host memory (for end-to-end timing of H2D/D2H)"""
        import torch

        def pin(a):
            t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
            v = t.numpy().view(a.dtype).reshape(a.shape)
            v[...] = a
            return v, t  # the tensor `t` owns the pinned pages; keep it alive with the view

        parts = [pin(a) for a in (self.mant, self.exp, self.kind, self.rad_man, self.rad_exp)]
        out = BallArray.__new__(BallArray)
        out.mant, out.exp, out.kind, out.rad_man, out.rad_exp = (p[0] for p in parts)
        out._pins = [p[1] for p in parts]
        return out

    # ----------------------------------------------------------- device
    def to_device(self, device="cuda") -> "DeviceBallArray":
        import torch
        return DeviceBallArray(
            torch.from_numpy(self.mant.view(np.int64)).to(device),
            torch.from_numpy(self.exp).to(device),
            torch.from_numpy(self.kind).to(device),
            torch.from_numpy(self.rad_man.view(np.int32)).to(device),
            torch.from_numpy(self.rad_exp).to(device))


class DeviceBallArray:
    """Device SoA ball array; torch tensors are used only as device memory."""

    def __init__(self, mant, exp, kind, rad_man, rad_exp):
        self.mant, self.exp, self.kind, self.rad_man, self.rad_exp = mant, exp, kind, rad_man, rad_exp

    @property
    def count(self) -> int:
        return int(self.exp.shape[0])

    @property
    def L(self) -> int:
        return int(self.mant.shape[1])

    @staticmethod
    def empty(count: int, L: int, device="cuda") -> "DeviceBallArray":
        import torch
        # every entry is written by the kernels; no fill launches
        return DeviceBallArray(torch.empty((count, L), dtype=torch.int64, device=device),
                               torch.empty(count, dtype=torch.int64, device=device),
                               torch.empty(count, dtype=torch.uint8, device=device),
                               torch.empty(count, dtype=torch.int32, device=device),
                               torch.empty(count, dtype=torch.int64, device=device))

    def c(self) -> apb_balls:
        return apb_balls(self.mant.data_ptr(), self.exp.data_ptr(), self.kind.data_ptr(),
                         self.rad_man.data_ptr(), self.rad_exp.data_ptr(), self.count, self.L)

    def to_host(self) -> BallArray:
        return BallArray(self.mant.cpu().numpy().view(np.uint64), self.exp.cpu().numpy(),
                         self.kind.cpu().numpy(), self.rad_man.cpu().numpy().view(np.uint32),
                         self.rad_exp.cpu().numpy())

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in
                   (self.mant, self.exp, self.kind, self.rad_man, self.rad_exp))


def mat_c(arr, rows: int, cols: int) -> apb_mat:
    return apb_mat(arr.c(), rows, cols)
