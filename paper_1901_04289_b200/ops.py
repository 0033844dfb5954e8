"""Host-side mirror of the reference operator surface for the hot path.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/apball/dot.hpp:57-89, matmul.hpp:69-109):

    dot_ball(initial, subtract, x, xstep, y, ystep, n, prec)   -> ball
    dot_approx(...)                                              -> midpoint
    dot_complex_ball(x, xstep, y, ystep, n, prec)               -> complex ball
    classical_matmul_ball / block_matmul_ball / matmul_auto(A, B, prec)
    complex_matmul_ball(A, B, prec)

plus the batched device entry points the B200 build adds (dot_batch,
dot_complex_batch, matmul on device-resident matrices).  Errors raise
InvalidArgument (std::invalid_argument) and OverflowErrorApb
(std::overflow_error) like the reference.  Every call runs the CUDA library;
there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .balls import (APB_DOT_APPROX, APB_DOT_BALL, APB_MM_AUTO, APB_MM_BLOCK, APB_MM_CLASSICAL,
                    DOT_STATE_DTYPE, BallArray, DeviceBallArray, apb_dot_index, apb_dot_tuning,
                    apb_mat, flat_index, limbs_for)


def _stream_ptr(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


# ------------------------------------------------------------ batched dots

def dot_batch(x: DeviceBallArray, y: DeviceBallArray, n: int, batch: int, prec: int, *,
              initial: DeviceBallArray | None = None, subtract: bool = False, mode: str = "ball",
              index: apb_dot_index | None = None, out: DeviceBallArray | None = None,
              want_state: bool = False, acc_stride: int = 0, disable_precision_reduction=False,
              stream=None, check: bool = True):
    """Batch of independent ball dot products on device-resident SoA arrays
    (one reference dot_ball / dot_approx call per dot)."""
    import torch
    lib = _lib.lib()
    index = index or flat_index(n)
    out = out if out is not None else DeviceBallArray.empty(batch, limbs_for(prec))
    state = torch.zeros(batch * DOT_STATE_DTYPE.itemsize, dtype=torch.uint8, device="cuda") if want_state else None
    acc = torch.zeros(batch * max(acc_stride, 1), dtype=torch.int64, device="cuda") if acc_stride else None
    tun = apb_dot_tuning(int(bool(disable_precision_reduction)), 0, 128)
    xc, yc, oc = x.c(), y.c(), out.c()
    ic = initial.c() if initial is not None else None
    st = _stream_ptr(stream)
    rc = lib.apb_dot_batch(C.byref(xc), C.byref(yc), C.byref(ic) if ic is not None else None,
                           int(bool(subtract)), C.byref(index), n, batch, prec,
                           APB_DOT_APPROX if mode == "approx" else APB_DOT_BALL, C.byref(tun),
                           C.byref(oc), state.data_ptr() if state is not None else None,
                           acc.data_ptr() if acc is not None else None, acc_stride, st)
    _lib.check(rc, "apb_dot_batch")
    if check:
        _lib.check(lib.apb_device_status(st), "apb_dot_batch")
    if want_state or acc_stride:
        st_np = np.frombuffer(state.cpu().numpy().tobytes(), DOT_STATE_DTYPE) if state is not None else None
        acc_np = acc.cpu().numpy().view(np.uint64).reshape(batch, acc_stride) if acc is not None else None
        return out, st_np, acc_np
    return out


def dot_complex_batch(xre, xim, yre, yim, n: int, batch: int, prec: int, *, mode="ball",
                      index=None, stream=None, check=True, force_threeprod=False, threeprod_cutoff=128,
                      want_hits=False):
    """dot_complex_ball / dot_complex_approx over a batch (include/apball/dot.hpp:86-89).
    want_hits also returns the number of terms passing the three-multiplication
    gate (dot_threeprod_hits, dot.hpp:54; the rewrite itself is result-neutral)."""
    import torch
    lib = _lib.lib()
    index = index or flat_index(n)
    ore, oim = DeviceBallArray.empty(batch, limbs_for(prec)), DeviceBallArray.empty(batch, limbs_for(prec))
    cs = [v.c() for v in (xre, xim, yre, yim, ore, oim)]
    st = _stream_ptr(stream)
    tun = apb_dot_tuning(0, int(bool(force_threeprod)), int(threeprod_cutoff))
    hits = torch.zeros(1, dtype=torch.int64, device="cuda") if want_hits else None
    rc = lib.apb_dot_complex_batch(*[C.byref(v) for v in cs[:4]], C.byref(index), n, batch, prec,
                                   APB_DOT_APPROX if mode == "approx" else APB_DOT_BALL, C.byref(tun),
                                   C.byref(cs[4]), C.byref(cs[5]), hits.data_ptr() if want_hits else None, st)
    _lib.check(rc, "apb_dot_complex_batch")
    if check or want_hits:
        _lib.check(lib.apb_device_status(st), "apb_dot_complex_batch")
    if want_hits:
        return ore, oim, int(hits.item())
    return ore, oim


def dot_batch_host(x: BallArray, y: BallArray, n: int, batch: int, prec: int, *,
                   initial: BallArray | None = None, subtract=False, mode="ball", index=None,
                   out: BallArray | None = None) -> BallArray:
    """Same as dot_batch on HOST arrays: copies in, computes on the GPU, copies out."""
    lib = _lib.lib()
    index = index or flat_index(n)
    out = out if out is not None else BallArray.zeros(batch, limbs_for(prec))
    xc, yc, oc = x.c(), y.c(), out.c()
    ic = initial.c() if initial is not None else None
    rc = lib.apb_dot_batch_host(C.byref(xc), C.byref(yc), C.byref(ic) if ic is not None else None,
                                int(bool(subtract)), C.byref(index), n, batch, prec,
                                APB_DOT_APPROX if mode == "approx" else APB_DOT_BALL, C.byref(oc))
    _lib.check(rc, "apb_dot_batch_host")
    return out


# ------------------------------------------------------ poly consumers (§8(f))

def poly_mullow_classical(a, b, length: int, prec: int, *, stream=None, check=True):
    """poly_mullow_classical (include/apball/poly.hpp:23-24): coefficients k < length
    of a*b, each the fused ball dot over (a_i, b_{k-i}) -- one batched launch.
    Device arrays in, device array out; host BallArrays go through the host entry."""
    lib = _lib.lib()
    L = limbs_for(prec)
    na, nb = a.count, b.count
    if isinstance(a, BallArray) or isinstance(b, BallArray):
        out = BallArray.zeros(max(length, 1), L)
        ac, bc, oc = a.c(), b.c(), out.c()
        _lib.check(lib.apb_poly_mullow_host(C.byref(ac), na, C.byref(bc), nb, length, prec, C.byref(oc)),
                   "apb_poly_mullow_host")
        return out.take(range(length))
    out = DeviceBallArray.empty(max(length, 1), L)
    ac, bc, oc = a.c(), b.c(), out.c()
    st = _stream_ptr(stream)
    _lib.check(lib.apb_poly_mullow(C.byref(ac), na, C.byref(bc), nb, length, prec, C.byref(oc), st),
               "apb_poly_mullow")
    if check:
        _lib.check(lib.apb_device_status(st), "apb_poly_mullow")
    return out


def series_exp_basecase(a, length: int, prec: int, *, stream=None, check=True):
    """series_exp_basecase (include/apball/poly.hpp:27-29): b_0 = 1,
    b_k = (sum_{j=1}^{k} (j a_j) b_{k-j}) / k; raises InvalidArgument (the
    reference's std::domain_error) unless a_0 is an exact zero."""
    lib = _lib.lib()
    L = limbs_for(prec)
    if isinstance(a, BallArray):
        out = BallArray.zeros(max(length, 1), L)
        ac, oc = a.c(), out.c()
        _lib.check(lib.apb_series_exp_host(C.byref(ac), a.count, length, prec, C.byref(oc)), "apb_series_exp_host")
        return out.take(range(length))
    out = DeviceBallArray.empty(max(length, 1), L)
    ac, oc = a.c(), out.c()
    st = _stream_ptr(stream)
    _lib.check(lib.apb_series_exp(C.byref(ac), a.count, length, prec, C.byref(oc), st), "apb_series_exp")
    if check:
        _lib.check(lib.apb_device_status(st), "apb_series_exp")
    return out


# --------------------------------------------------- wire format (§8(f) row 3)

def balls_to_text(a) -> str:
    """the reference's text form, one "mid +- rad" line per ball (Ball::to_string,
    src/ball.cpp:45-47); device arrays are copied to the host first"""
    lib = _lib.lib()
    h = a.to_host() if isinstance(a, DeviceBallArray) else a
    hc = h.c()
    n = lib.apb_balls_format(C.byref(hc), 0, h.count, None, 0)
    if n < 0:
        raise _lib.InvalidArgument(1, _lib.last_error())
    buf = C.create_string_buffer(n + 1)
    lib.apb_balls_format(C.byref(hc), 0, h.count, buf, n + 1)
    return buf.value.decode()


def balls_from_text(text: str, count: int, L: int) -> BallArray:
    """inverse of balls_to_text (Ball::parse, src/ball.cpp:49-56); raises
    InvalidArgument on a malformed line or a mantissa wider than L limbs"""
    lib = _lib.lib()
    out = BallArray.zeros(count, L)
    oc = out.c()
    raw = text.encode()
    got = lib.apb_balls_parse(raw, len(raw), C.byref(oc), count)
    if got != count:
        raise _lib.InvalidArgument(1, _lib.last_error() if got < 0 else f"only {got} of {count} balls")
    return out


def matrix_to_text(m: BallMatrix) -> str:
    """write_ball_matrix (src/matmul.cpp:554-557): "rows cols" then the balls"""
    lib = _lib.lib()
    h = BallMatrix(m.balls.to_host() if m.on_device else m.balls, m.rows, m.cols)
    hc = h.c()
    n = lib.apb_mat_format(C.byref(hc), None, 0)
    buf = C.create_string_buffer(n + 1)
    lib.apb_mat_format(C.byref(hc), buf, n + 1)
    return buf.value.decode()


def matrix_from_text(text: str, L: int) -> BallMatrix:
    """read_ball_matrix (src/matmul.cpp:559-570)"""
    lib = _lib.lib()
    head = text.split("\n", 1)[0].split()
    r, c = int(head[0]), int(head[1])
    m = BallMatrix(BallArray.zeros(r * c, L), r, c)
    mc = m.c()
    raw = text.encode()
    _lib.check(lib.apb_mat_parse(raw, len(raw), C.byref(mc)), "apb_mat_parse")
    return m


# ------------------------------------------------- reference-shaped dots

def dot_ball(initial: BallArray | None, subtract: bool, x: BallArray | None, xstep: int,
             y: BallArray | None, ystep: int, n: int, prec: int, *, x_off: int = 0,
             y_off: int = 0) -> BallArray:
    """dot_ball (include/apball/dot.hpp:73-74): initial + (-1)^subtract sum x_i y_i
    with x_i = x[x_off + i*xstep] (steps may be negative)."""
    return _dot_one(initial, subtract, x, xstep, y, ystep, n, prec, x_off, y_off, "ball")


def dot_approx(initial, subtract, x, xstep, y, ystep, n, prec, *, x_off=0, y_off=0) -> BallArray:
    """dot_approx (include/apball/dot.hpp:77-78): midpoint only (zero radius)."""
    return _dot_one(initial, subtract, x, xstep, y, ystep, n, prec, x_off, y_off, "approx")


def _dot_one(initial, subtract, x, xstep, y, ystep, n, prec, x_off, y_off, mode):
    if n == 0:
        x = y = BallArray.zeros(1, 1)
    idx = apb_dot_index(1, x_off, 0, 0, xstep, y_off, 0, 0, ystep)
    return dot_batch_host(x, y, n, 1, prec, initial=initial, subtract=subtract, mode=mode, index=idx)


# ------------------------------------------------------------------ matmul

@dataclass
class BallMatrix:
    """Row-major ball matrix (include/apball/matmul.hpp:18-26), host or device."""
    balls: BallArray | DeviceBallArray
    rows: int
    cols: int

    def c(self) -> apb_mat:
        return apb_mat(self.balls.c(), self.rows, self.cols)

    @property
    def on_device(self) -> bool:
        return isinstance(self.balls, DeviceBallArray)


def _matmul(a: BallMatrix, b: BallMatrix, prec: int, algo: int, stream=None, check=True,
            out: BallMatrix | None = None) -> BallMatrix:
    """`out` (device, a.rows x b.cols, limbs_for(prec) limbs) is reused when given:
    repeated calls on the same buffers replay the library's captured CUDA graphs"""
    lib = _lib.lib()
    if a.cols != b.rows:
        raise _lib.InvalidArgument(1, "matmul: dimension mismatch")
    L = limbs_for(prec)
    if a.on_device:
        if out is not None:
            if (out.rows, out.cols) != (a.rows, b.cols) or out.balls.L != L:
                raise _lib.InvalidArgument(1, "matmul: output shape / limb count mismatch")
            c = out
        else:
            c = BallMatrix(DeviceBallArray.empty(a.rows * b.cols, L), a.rows, b.cols)
        am, bm, cm = a.c(), b.c(), c.c()
        st = _stream_ptr(stream)
        _lib.check(lib.apb_matmul(C.byref(am), C.byref(bm), prec, algo, C.byref(cm), st), "apb_matmul")
        if check:
            _lib.check(lib.apb_device_status(st), "apb_matmul")
        return c
    c = BallMatrix(BallArray.zeros(a.rows * b.cols, L), a.rows, b.cols)
    am, bm, cm = a.c(), b.c(), c.c()
    _lib.check(lib.apb_matmul_host(C.byref(am), C.byref(bm), prec, algo, C.byref(cm)), "apb_matmul_host")
    return c


def classical_matmul_ball(a: BallMatrix, b: BallMatrix, prec: int, **kw) -> BallMatrix:
    """classical_matmul_ball (include/apball/matmul.hpp:89)"""
    return _matmul(a, b, prec, APB_MM_CLASSICAL, **kw)


def block_matmul_ball(a: BallMatrix, b: BallMatrix, prec: int, **kw) -> BallMatrix:
    """block_matmul_ball (include/apball/matmul.hpp:90)"""
    return _matmul(a, b, prec, APB_MM_BLOCK, **kw)


def matmul_auto(a: BallMatrix, b: BallMatrix, prec: int, **kw) -> BallMatrix:
    """matmul_auto (include/apball/matmul.hpp:91)"""
    return _matmul(a, b, prec, APB_MM_AUTO, **kw)


def matmul_dispatch_cutoff(prec: int) -> int:
    """matmul_dispatch_cutoff (src/matmul.cpp:517-524)"""
    for lim, c in ((64, 60), (128, 56), (256, 52), (512, 48), (1024, 44)):
        if prec <= lim:
            return c
    return 40


def complex_matmul_ball(are: BallMatrix, aim: BallMatrix, bre: BallMatrix, bim: BallMatrix,
                        prec: int, stream=None, check=True):
    """complex_matmul_ball (include/apball/matmul.hpp:92-93); parts given separately"""
    lib = _lib.lib()
    if are.cols != bre.rows:
        raise _lib.InvalidArgument(1, "matmul: dimension mismatch")
    L = limbs_for(prec)
    cre = BallMatrix(DeviceBallArray.empty(are.rows * bre.cols, L), are.rows, bre.cols)
    cim = BallMatrix(DeviceBallArray.empty(are.rows * bre.cols, L), are.rows, bre.cols)
    ms = [m.c() for m in (are, aim, bre, bim, cre, cim)]
    st = _stream_ptr(stream)
    _lib.check(lib.apb_matmul_complex(*[C.byref(m) for m in ms[:4]], prec, APB_MM_AUTO,
                                      C.byref(ms[4]), C.byref(ms[5]), st), "apb_matmul_complex")
    if check:
        _lib.check(lib.apb_device_status(st), "apb_matmul_complex")
    return cre, cim


def matmul_stats() -> dict:
    s = _lib.lib().apb_matmul_stats_get().contents
    return {f: int(getattr(s, f)) for f, _ in s._fields_}


def matmul_stats_reset():
    _lib.lib().apb_matmul_stats_reset()


def launch_count() -> int:
    return int(_lib.lib().apb_launch_count())


# ------------------------------------------------------------ parity hooks

def plan_blocks(a: BallMatrix, b: BallMatrix, prec: int, stream=None):
    """plan_blocks (include/apball/matmul.hpp:73): list of (lo, hi, basecase)"""
    lib = _lib.lib()
    am, bm = a.c(), b.c()
    steps = np.zeros(3 * (a.cols + 1), np.int64)
    ns = C.c_int64(0)
    _lib.check(lib.apb_plan_blocks(C.byref(am), C.byref(bm), prec, steps.ctypes.data, a.cols + 1,
                                   C.addressof(ns), _stream_ptr(stream)), "apb_plan_blocks")
    return [tuple(int(v) for v in steps[3 * i:3 * i + 3]) for i in range(ns.value)]


def block_int_product(a: BallMatrix, b: BallMatrix, lo: int, hi: int, out_limbs: int, stream=None):
    """int_matmul(scale_block_rows(A,lo,hi), scale_block_cols(B,lo,hi)) as two's complement
    limbs (include/apball/matmul.hpp:77-84); returns (row_scale, col_scale, T)"""
    import torch
    lib = _lib.lib()
    am, bm = a.c(), b.c()
    rs = torch.zeros(a.rows, dtype=torch.int64, device="cuda")
    cs = torch.zeros(b.cols, dtype=torch.int64, device="cuda")
    out = torch.zeros(a.rows * b.cols * out_limbs, dtype=torch.int64, device="cuda")
    st = _stream_ptr(stream)
    _lib.check(lib.apb_block_int_product(C.byref(am), C.byref(bm), lo, hi, rs.data_ptr(), cs.data_ptr(),
                                         out.data_ptr(), out_limbs, st), "apb_block_int_product")
    _lib.check(lib.apb_device_status(st), "apb_block_int_product")
    return (rs.cpu().numpy(), cs.cpu().numpy(),
            out.cpu().numpy().view(np.uint64).reshape(a.rows * b.cols, out_limbs))


def block_int_product_imad(a: BallMatrix, b: BallMatrix, lo: int, hi: int, out_limbs: int, stream=None):
    """block_int_product on the CUDA cores with 32-bit limbs (the IMAD baseline the
    int8 tensor-core product is measured against); returns (row_scale, col_scale, T, gemm_ms)"""
    import torch
    lib = _lib.lib()
    am, bm = a.c(), b.c()
    rs = torch.zeros(a.rows, dtype=torch.int64, device="cuda")
    cs = torch.zeros(b.cols, dtype=torch.int64, device="cuda")
    out = torch.zeros(a.rows * b.cols * out_limbs, dtype=torch.int64, device="cuda")
    ms = C.c_float(0.0)
    st = _stream_ptr(stream)
    _lib.check(lib.apb_block_int_product_imad(C.byref(am), C.byref(bm), lo, hi, rs.data_ptr(), cs.data_ptr(),
                                              out.data_ptr(), out_limbs, C.byref(ms), st),
               "apb_block_int_product_imad")
    return (rs.cpu().numpy(), cs.cpu().numpy(),
            out.cpu().numpy().view(np.uint64).reshape(a.rows * b.cols, out_limbs), ms.value)


def radius_matmul_upper(pm, pe, qm, qe, m: int, n: int, k: int, stream=None):
    """radius_matmul_upper (include/apball/matmul.hpp:87) on Mag planes (mantissa, exponent)"""
    import torch
    lib = _lib.lib()
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
    dpm, dpe = t(np.asarray(pm, np.uint32).view(np.int32), None), t(np.asarray(pe, np.int64), None)
    dqm, dqe = t(np.asarray(qm, np.uint32).view(np.int32), None), t(np.asarray(qe, np.int64), None)
    om = torch.zeros(m * k, dtype=torch.int32, device="cuda")
    oe = torch.zeros(m * k, dtype=torch.int64, device="cuda")
    st = _stream_ptr(stream)
    _lib.check(lib.apb_radius_matmul_upper(dpm.data_ptr(), dpe.data_ptr(), dqm.data_ptr(), dqe.data_ptr(),
                                           m, n, k, om.data_ptr(), oe.data_ptr(), st), "apb_radius_matmul_upper")
    _lib.check(lib.apb_device_status(st), "apb_radius_matmul_upper")
    return om.cpu().numpy().view(np.uint32), oe.cpu().numpy()


def plan_info(a: BallMatrix, b: BallMatrix, prec: int, stream=None) -> dict:
    """planner summary (block count, entry precisions, widths, radius single-block flag)"""
    from .balls import apb_plan_info
    lib = _lib.lib()
    am, bm = a.c(), b.c()
    out = apb_plan_info()
    _lib.check(lib.apb_matmul_plan_info(C.byref(am), C.byref(bm), prec, C.byref(out), _stream_ptr(stream)),
               "apb_matmul_plan_info")
    return {f: int(getattr(out, f)) for f, _ in out._fields_}


def radius_single_block(a: BallMatrix, b: BallMatrix, prec: int = 2) -> bool:
    return bool(plan_info(a, b, prec)["radius_single"])
