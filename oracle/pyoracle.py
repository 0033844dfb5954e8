"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the two CPU checkers.

* `ref`  - oracle/_ref/libapball_ref.so: the UNMODIFIED reference library
           (/root/reference/proj/src) plus our extern "C" layout shim;
* `port` - oracle/_ref/libapb_oracle.so: our plain-C restatement (apb_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.  Both libraries are prebuilt (oracle/Makefile) and
travel to the GPU box inside the repo snapshot.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1901_04289_b200.balls import (BallArray, DOT_STATE_DTYPE, apb_dot_index, apb_mat,
                                         apb_matmul_stats)

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libapball_ref.so")
PORT_SO = os.path.join(HERE, "_ref", "libapb_oracle.so")

P = C.c_void_p
I64 = C.c_int64
I = C.c_int


def _load(path):
    if not os.path.exists(path):
        raise RuntimeError(f"oracle library missing: {path} (run `make -C oracle`)")
    return C.CDLL(path)


_ref = None
_port = None


def ref_lib():
    global _ref
    if _ref is None:
        _ref = _load(REF_SO)
        _ref.ref_last_error.restype = C.c_char_p
        for name in ("ref_dot_batch", "ref_dot_state", "ref_dot_complex_batch", "ref_matmul",
                     "ref_matmul_complex", "ref_plan_blocks", "ref_block_int_product",
                     "ref_radius_matmul_upper", "ref_dot_contains", "ref_abs_dot_upper",
                     "ref_run_verify_suite", "ref_ball_addsub", "ref_poly_mullow", "ref_series_exp"):
            getattr(_ref, name).restype = I
    return _ref


def port_lib():
    global _port
    if _port is None:
        _port = _load(PORT_SO)
        for name in ("orc_dot_batch", "orc_dot_complex_batch", "orc_matmul", "orc_matmul_complex",
                     "orc_plan_blocks", "orc_block_int_product", "orc_radius_matmul_upper",
                     "orc_poly_mullow", "orc_series_exp"):
            getattr(_port, name).restype = I
    return _port


def _p(x):
    return C.byref(x)


def _check(rc, lib=None, what=""):
    if rc != 0:
        msg = ""
        if lib is not None and hasattr(lib, "ref_last_error"):
            msg = lib.ref_last_error().decode()
        raise RuntimeError(f"{what} failed with status {rc} {msg}")


# ------------------------------------------------------------------- dots

def dot_batch(x: BallArray, y: BallArray, n: int, batch: int, prec: int, *, which="ref",
              initial: BallArray | None = None, subtract=False, mode=0, idx=None,
              disable_reduction=False, threads=1, L_out=None, want_state=False):
    from paper_1901_04289_b200.balls import flat_index, limbs_for
    idx = idx or flat_index(n)
    out = BallArray.zeros(batch, L_out or max(limbs_for(prec), 1))
    xc, yc, oc = x.c(), y.c(), out.c()
    ic = initial.c() if initial is not None else None
    st = np.zeros(batch, DOT_STATE_DTYPE) if want_state else None
    if which == "ref":
        lib = ref_lib()
        rc = lib.ref_dot_batch(_p(xc), _p(yc), _p(ic) if ic else None, I(subtract), _p(idx), I64(n),
                               I64(batch), I64(prec), I(mode), I(disable_reduction), _p(oc), I(threads))
        _check(rc, lib, "ref_dot_batch")
    else:
        lib = port_lib()
        rc = lib.orc_dot_batch(_p(xc), _p(yc), _p(ic) if ic else None, I(subtract), _p(idx), I64(n),
                               I64(batch), I64(prec), I(mode), I(disable_reduction), _p(oc),
                               P(st.ctypes.data) if st is not None else None, None, I64(0))
        _check(rc, None, "orc_dot_batch")
    return (out, st) if want_state else out


def dot_state(x, y, n, batch, prec, *, which="ref", initial=None, subtract=False, idx=None,
              disable_reduction=False, acc_stride=80):
    """plan + accumulator (s limbs, err, srad) before finalize"""
    from paper_1901_04289_b200.balls import flat_index, limbs_for
    idx = idx or flat_index(n)
    st = np.zeros(batch, DOT_STATE_DTYPE)
    acc = np.zeros((batch, acc_stride), np.uint64)
    xc, yc = x.c(), y.c()
    ic = initial.c() if initial is not None else None
    if which == "ref":
        lib = ref_lib()
        rc = lib.ref_dot_state(_p(xc), _p(yc), _p(ic) if ic else None, I(subtract), _p(idx), I64(n),
                               I64(batch), I64(prec), I(disable_reduction), P(st.ctypes.data),
                               P(acc.ctypes.data), I64(acc_stride))
        _check(rc, lib, "ref_dot_state")
    else:
        lib = port_lib()
        out = BallArray.zeros(batch, limbs_for(prec))
        oc = out.c()
        rc = lib.orc_dot_batch(_p(xc), _p(yc), _p(ic) if ic else None, I(subtract), _p(idx), I64(n),
                               I64(batch), I64(prec), I(0), I(disable_reduction), _p(oc),
                               P(st.ctypes.data), P(acc.ctypes.data), I64(acc_stride))
        _check(rc, None, "orc_dot_batch")
    return st, acc


def dot_complex_batch(xre, xim, yre, yim, n, batch, prec, *, which="ref", mode=0, idx=None,
                      threads=1, force_threeprod=False, want_hits=False):
    from paper_1901_04289_b200.balls import flat_index, limbs_for
    idx = idx or flat_index(n)
    ore, oim = BallArray.zeros(batch, limbs_for(prec)), BallArray.zeros(batch, limbs_for(prec))
    a = [v.c() for v in (xre, xim, yre, yim, ore, oim)]
    if which == "ref":
        lib = ref_lib()
        hits = C.c_uint64(0)
        rc = lib.ref_dot_complex_batch(*[_p(v) for v in a[:4]], _p(idx), I64(n), I64(batch),
                                       I64(prec), I(mode), I(force_threeprod), _p(a[4]), _p(a[5]),
                                       _p(hits), I(threads))
        _check(rc, lib, "ref_dot_complex_batch")
        if want_hits:
            return ore, oim, int(hits.value)
    else:
        lib = port_lib()
        rc = lib.orc_dot_complex_batch(*[_p(v) for v in a[:4]], _p(idx), I64(n), I64(batch),
                                       I64(prec), I(mode), _p(a[4]), _p(a[5]))
        _check(rc, None, "orc_dot_complex_batch")
    return ore, oim


def dot_contains(x, y, n, batch, out, *, initial=None, subtract=False, idx=None, threads=1):
    from paper_1901_04289_b200.balls import flat_index
    idx = idx or flat_index(n)
    ok = np.zeros(batch, np.uint8)
    xc, yc, oc = x.c(), y.c(), out.c()
    ic = initial.c() if initial is not None else None
    lib = ref_lib()
    rc = lib.ref_dot_contains(_p(xc), _p(yc), _p(ic) if ic else None, I(subtract), _p(idx), I64(n),
                              I64(batch), _p(oc), P(ok.ctypes.data), I(threads))
    _check(rc, lib, "ref_dot_contains")
    return ok.astype(bool)


def abs_dot_upper(x, y, n, batch, idx=None):
    from paper_1901_04289_b200.balls import flat_index
    idx = idx or flat_index(n)
    man = np.zeros(batch, np.uint32)
    ex = np.zeros(batch, np.int64)
    xc, yc = x.c(), y.c()
    lib = ref_lib()
    _check(lib.ref_abs_dot_upper(_p(xc), _p(yc), _p(idx), I64(n), I64(batch), P(man.ctypes.data),
                                 P(ex.ctypes.data)), lib, "ref_abs_dot_upper")
    return man, ex


# ----------------------------------------------------------------- matmul

def row_split_threads(threads, M, algo=0):
    """threads for a row-split reference product: with matmul_auto (algo 0, also inside
    complex_matmul_ball) every row block must stay above the classical dispatch cutoff
    (<= 60 rows, src/matmul.cpp:517-531), else the split product takes another path"""
    return max(1, min(threads, M // 64)) if algo == 0 else max(1, threads)


def matmul(a: BallArray, b: BallArray, M, K, N, prec, *, which="ref", algo=0, threads=1):
    from paper_1901_04289_b200.balls import limbs_for
    threads = row_split_threads(threads, M, algo)
    c = BallArray.zeros(M * N, limbs_for(prec))
    A, B, Cm = apb_mat(a.c(), M, K), apb_mat(b.c(), K, N), apb_mat(c.c(), M, N)
    if which == "ref":
        lib = ref_lib()
        st = apb_matmul_stats()
        _check(lib.ref_matmul(_p(A), _p(B), I64(prec), I(algo), _p(Cm), I(threads), _p(st)), lib,
               "ref_matmul")
        return c, int(st.last_block_count)
    lib = port_lib()
    nb = I64(0)
    _check(lib.orc_matmul(_p(A), _p(B), I64(prec), I(algo), _p(Cm), _p(nb)), None, "orc_matmul")
    return c, int(nb.value)


def matmul_complex(are, aim, bre, bim, M, K, N, prec, *, which="ref", threads=1):
    from paper_1901_04289_b200.balls import limbs_for
    threads = row_split_threads(threads, M, 0)
    cre, cim = BallArray.zeros(M * N, limbs_for(prec)), BallArray.zeros(M * N, limbs_for(prec))
    mats = [apb_mat(are.c(), M, K), apb_mat(aim.c(), M, K), apb_mat(bre.c(), K, N),
            apb_mat(bim.c(), K, N), apb_mat(cre.c(), M, N), apb_mat(cim.c(), M, N)]
    if which == "ref":
        lib = ref_lib()
        _check(lib.ref_matmul_complex(*[_p(m) for m in mats[:4]], I64(prec), _p(mats[4]),
                                      _p(mats[5]), I(threads)), lib, "ref_matmul_complex")
    else:
        lib = port_lib()
        _check(lib.orc_matmul_complex(*[_p(m) for m in mats[:4]], I64(prec), _p(mats[4]),
                                      _p(mats[5])), None, "orc_matmul_complex")
    return cre, cim


def plan_blocks(a, b, M, K, N, prec, *, which="ref"):
    A, B = apb_mat(a.c(), M, K), apb_mat(b.c(), K, N)
    steps = np.zeros(3 * (K + 1), np.int64)
    ns = I64(0)
    if which == "ref":
        lib = ref_lib()
        ep = np.zeros(2, np.int64)
        _check(lib.ref_plan_blocks(_p(A), _p(B), I64(prec), P(steps.ctypes.data), I64(K + 1),
                                   _p(ns), P(ep.ctypes.data)), lib, "ref_plan_blocks")
    else:
        lib = port_lib()
        _check(lib.orc_plan_blocks(_p(A), _p(B), I64(prec), P(steps.ctypes.data), I64(K + 1),
                                   _p(ns)), None, "orc_plan_blocks")
    return [tuple(int(v) for v in steps[3 * i:3 * i + 3]) for i in range(ns.value)]


def block_int_product(a, b, M, K, N, lo, hi, out_limbs, *, which="ref"):
    A, B = apb_mat(a.c(), M, K), apb_mat(b.c(), K, N)
    rs = np.zeros(M, np.int64)
    cs = np.zeros(N, np.int64)
    out = np.zeros((M * N, out_limbs), np.uint64)
    if which == "ref":
        lib = ref_lib()
        h = np.zeros(2, np.int64)
        _check(lib.ref_block_int_product(_p(A), _p(B), I64(lo), I64(hi), P(rs.ctypes.data),
                                         P(cs.ctypes.data), P(out.ctypes.data), I64(out_limbs),
                                         P(h.ctypes.data)), lib, "ref_block_int_product")
    else:
        lib = port_lib()
        _check(lib.orc_block_int_product(_p(A), _p(B), I64(lo), I64(hi), P(rs.ctypes.data),
                                         P(cs.ctypes.data), P(out.ctypes.data), I64(out_limbs)),
               None, "orc_block_int_product")
    return rs, cs, out


def radius_matmul_upper(pm, pe, qm, qe, m, n, k, *, which="ref"):
    om = np.zeros(m * k, np.uint32)
    oe = np.zeros(m * k, np.int64)
    args = [P(np.ascontiguousarray(pm, np.uint32).ctypes.data), P(np.ascontiguousarray(pe, np.int64).ctypes.data),
            P(np.ascontiguousarray(qm, np.uint32).ctypes.data), P(np.ascontiguousarray(qe, np.int64).ctypes.data)]
    keep = [np.ascontiguousarray(pm, np.uint32), np.ascontiguousarray(pe, np.int64),
            np.ascontiguousarray(qm, np.uint32), np.ascontiguousarray(qe, np.int64)]
    args = [P(a.ctypes.data) for a in keep]
    if which == "ref":
        lib = ref_lib()
        _check(lib.ref_radius_matmul_upper(*args, I64(m), I64(n), I64(k), P(om.ctypes.data),
                                           P(oe.ctypes.data)), lib, "ref_radius_matmul_upper")
    else:
        lib = port_lib()
        _check(lib.orc_radius_matmul_upper(*args, I64(m), I64(n), I64(k), P(om.ctypes.data),
                                           P(oe.ctypes.data)), None, "orc_radius_matmul_upper")
    return om, oe


def run_verify_suite(name: str, trials: int, seed: int) -> int:
    lib = ref_lib()
    f = C.c_uint64(0)
    _check(lib.ref_run_verify_suite(name.encode(), C.c_uint64(trials), C.c_uint64(seed), _p(f)), lib,
           "ref_run_verify_suite")
    return int(f.value)


def ball_addsub(x: BallArray, y: BallArray, prec: int, subtract=False) -> BallArray:
    """reference ball_add / ball_sub elementwise"""
    from paper_1901_04289_b200.balls import limbs_for
    out = BallArray.zeros(x.count, limbs_for(prec))
    xc, yc, oc = x.c(), y.c(), out.c()
    lib = ref_lib()
    _check(lib.ref_ball_addsub(_p(xc), _p(yc), I(subtract), I64(x.count), I64(prec), _p(oc)), lib,
           "ref_ball_addsub")
    return out


def matmul_complex_rows(are, aim, bre, bim, rows, K, N, prec, threads=1):
    """complex_matmul_ball on the first `rows` rows of A when the full product takes
    the block path: the four real products with block_matmul_ball (row-split,
    bit-identical for single-block plans) + ball_sub / ball_add"""
    sub = lambda a: a.take(np.arange(rows * K))
    ac, _ = matmul(sub(are), bre, rows, K, N, prec, which="ref", algo=1, threads=threads)
    bd, _ = matmul(sub(aim), bim, rows, K, N, prec, which="ref", algo=1, threads=threads)
    ad, _ = matmul(sub(are), bim, rows, K, N, prec, which="ref", algo=1, threads=threads)
    bc, _ = matmul(sub(aim), bre, rows, K, N, prec, which="ref", algo=1, threads=threads)
    return ball_addsub(ac, bd, prec, subtract=True), ball_addsub(ad, bc, prec)


# ------------------------------------------------------------------- poly

def poly_mullow(a: BallArray, b: BallArray, length: int, prec: int, *, which="ref") -> BallArray:
    """poly_mullow_classical (src/poly.cpp:11-26) via the reference or the C restatement"""
    from paper_1901_04289_b200.balls import limbs_for
    out = BallArray.zeros(max(length, 1), max(limbs_for(prec), 1))
    ac, bc, oc = a.c(), b.c(), out.c()
    if which == "ref":
        lib = ref_lib()
        rc = lib.ref_poly_mullow(_p(ac), I64(a.count), _p(bc), I64(b.count), I64(length), I64(prec), _p(oc))
        _check(rc, lib, "ref_poly_mullow")
    else:
        rc = port_lib().orc_poly_mullow(_p(ac), I64(a.count), _p(bc), I64(b.count), I64(length), I64(prec),
                                        _p(oc))
        _check(rc, None, "orc_poly_mullow")
    return out.take(range(length)) if length < out.count else out


def series_exp(a: BallArray, length: int, prec: int, *, which="ref") -> BallArray:
    """series_exp_basecase (src/poly.cpp:28-46); raises ValueError (the reference's
    std::domain_error) when a_0 is not an exact zero"""
    from paper_1901_04289_b200.balls import limbs_for
    out = BallArray.zeros(max(length, 1), max(limbs_for(prec), 1))
    ac, oc = a.c(), out.c()
    if which == "ref":
        lib = ref_lib()
        rc = lib.ref_series_exp(_p(ac), I64(a.count), I64(length), I64(prec), _p(oc))
    else:
        lib = port_lib()
        rc = lib.orc_series_exp(_p(ac), I64(a.count), I64(length), I64(prec), _p(oc))
    if rc == 1:
        raise ValueError("series_exp_basecase: constant term must be exactly zero")
    _check(rc, lib if which == "ref" else None, "series_exp")
    return out.take(range(length)) if length < out.count else out


# ------------------------------------------------------------- wire format

def balls_format(a: BallArray) -> str:
    """Ball::to_string per line, from the reference itself"""
    lib = ref_lib()
    lib.ref_balls_format.restype = C.c_int64
    ac = a.c()
    n = lib.ref_balls_format(_p(ac), I64(0), I64(a.count), None, I64(0))
    buf = C.create_string_buffer(n + 1)
    lib.ref_balls_format(_p(ac), I64(0), I64(a.count), buf, I64(n + 1))
    return buf.value.decode()


def balls_parse(text: str, count: int, L: int) -> BallArray | None:
    lib = ref_lib()
    lib.ref_balls_parse.restype = C.c_int64
    out = BallArray.zeros(count, L)
    oc = out.c()
    raw = text.encode()
    got = lib.ref_balls_parse(raw, I64(len(raw)), _p(oc), I64(count))
    return out if got == count else None

