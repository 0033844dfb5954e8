"""Generate the golden fixtures in tests/golden from the REFERENCE itself.

TEST INFRASTRUCTURE ONLY.  Runs in the build container (needs
oracle/_ref/libapball_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Every expected value below is produced by the reference's
own public API through ref_shim.cpp; the inputs are the seeded generators of
paper_1901_04289_b200/gen.py plus the hand-made known-answer cases of the
reference's doctest suites (tests/test_dot.cpp, tests/test_matmul.cpp in
/root/reference/proj), restated as data.

    python oracle/gen_golden.py        # rewrites tests/golden/*.npz
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import pyoracle as po  # noqa: E402
from paper_1901_04289_b200 import gen  # noqa: E402
from paper_1901_04289_b200.balls import (APB_FINITE, APB_NAN, APB_SIGN, APB_ZERO, BallArray,  # noqa: E402
                                         apb_dot_index)

OUT = os.path.join(ROOT, "tests", "golden")


def pack(prefix: str, a: BallArray) -> dict:
    return {f"{prefix}_mant": a.mant, f"{prefix}_exp": a.exp, f"{prefix}_kind": a.kind,
            f"{prefix}_rad_man": a.rad_man, f"{prefix}_rad_exp": a.rad_exp}


def idx_arr(ix: apb_dot_index) -> np.ndarray:
    return np.array([ix.bdiv, ix.x_off, ix.xs1, ix.xs2, ix.xstep, ix.y_off, ix.ys1, ix.ys2, ix.ystep],
                    np.int64)


def ball_from_i64(vals) -> BallArray:
    """Ball::from_i64 (include/apball/ball.hpp:22) for small integers"""
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


def dot_case(name, x, y, n, batch, prec, *, initial=None, subtract=False, mode=0, idx=None,
             disable_reduction=False):
    from paper_1901_04289_b200.balls import flat_index
    idx = idx or flat_index(n)
    out = po.dot_batch(x, y, n, batch, prec, which="ref", initial=initial, subtract=subtract,
                       mode=mode, idx=idx, disable_reduction=disable_reduction)
    st, acc = po.dot_state(x, y, n, batch, prec, which="ref", initial=initial, subtract=subtract,
                           idx=idx, disable_reduction=disable_reduction)
    d = {"kind": np.array("dot"), "n": np.int64(n), "batch": np.int64(batch), "prec": np.int64(prec),
         "subtract": np.int64(subtract), "mode": np.int64(mode), "idx": idx_arr(idx),
         "disable_reduction": np.int64(disable_reduction), "state": st, "acc": acc}
    d.update(pack("x", x))
    d.update(pack("y", y))
    d.update(pack("out", out))
    if initial is not None:
        d.update(pack("init", initial))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    return out


def matmul_case(name, a, b, M, K, N, prec, algo=1):
    c, nb = po.matmul(a, b, M, K, N, prec, which="ref", algo=algo)
    plan = po.plan_blocks(a, b, M, K, N, prec)
    d = {"kind": np.array("matmul"), "M": np.int64(M), "K": np.int64(K), "N": np.int64(N),
         "prec": np.int64(prec), "algo": np.int64(algo), "blocks": np.int64(nb),
         "plan": np.array(plan, np.int64).reshape(-1, 3)}
    # exact integer block products for every non-basecase block
    prods = []
    for bi, (lo, hi, base) in enumerate(plan):
        if base:
            continue
        hb = (5 * prec) // 4 + 192  # block height bound (src/matmul.cpp:137-139)
        rs, cs, T = po.block_int_product(a, b, M, K, N, lo, hi, out_limbs=(2 * hb + 16 + 63) // 64 + 1)
        d[f"int_{bi}_rows"] = rs
        d[f"int_{bi}_cols"] = cs
        d[f"int_{bi}_T"] = T
        prods.append(bi)
    d["int_blocks"] = np.array(prods, np.int64)
    d.update(pack("a", a))
    d.update(pack("b", b))
    d.update(pack("c", c))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)


def poly_cases():
    """poly_mullow_classical / series_exp_basecase fixtures from the reference:
    restated KATs (tests/test_poly.cpp:15-61) and random cases with edge values"""
    one = ball_from_i64([1, 1])
    d = {"kind": np.array("poly"), "len": 3, "prec": 64, **pack("a", one), **pack("b", one),
         **pack("out", po.poly_mullow(one, one, 3, 64))}
    np.savez_compressed(os.path.join(OUT, "poly_kat_square.npz"), **d)   # :15-25 -> 1, 2, 1
    x = ball_from_i64([0, 1, 0, 0, 0])
    d = {"kind": np.array("series"), "len": 5, "prec": 128, **pack("a", x),
         **pack("out", po.series_exp(x, 5, 128))}
    np.savez_compressed(os.path.join(OUT, "series_kat_x.npz"), **d)       # :33-48 -> 1/k!
    z = ball_from_i64([0, 0, 0, 0])
    d = {"kind": np.array("series"), "len": 4, "prec": 64, **pack("a", z),
         **pack("out", po.series_exp(z, 4, 64))}
    np.savez_compressed(os.path.join(OUT, "series_kat_zero.npz"), **d)    # :50-56 -> 1, 0, 0, 0
    rng = np.random.Generator(np.random.PCG64(20261020))
    for q, (la, lb, ln, p) in enumerate([(5, 7, 12, 64), (16, 16, 32, 128), (33, 20, 40, 256), (9, 3, 20, 700),
                                         (40, 40, 80, 128), (1, 1, 3, 30)]):
        a, _ = gen.edge_dots(rng, 1, la, specials=(q == 2))
        b, _ = gen.edge_dots(rng, 1, lb, specials=False)
        d = {"kind": np.array("poly"), "len": ln, "prec": p, **pack("a", a), **pack("b", b),
             **pack("out", po.poly_mullow(a, b, ln, p))}
        np.savez_compressed(os.path.join(OUT, f"poly_rand{q}.npz"), **d)
    for q, (la, ln, p) in enumerate([(6, 10, 64), (12, 12, 128), (20, 30, 256), (4, 16, 1000)]):
        a, _ = gen.edge_dots(rng, 1, la, specials=False)
        a.kind[0] = 0
        a.mant[0] = 0
        a.exp[0] = 0
        a.rad_man[0] = 0
        a.rad_exp[0] = 0
        d = {"kind": np.array("series"), "len": ln, "prec": p, **pack("a", a),
             **pack("out", po.series_exp(a, ln, p))}
        np.savez_compressed(os.path.join(OUT, f"series_rand{q}.npz"), **d)


def main():
    os.makedirs(OUT, exist_ok=True)
    # ---- c1 shape (65,536 x N=100 at p=128) at a small batch
    x, y = gen.config1_dots(batch=64, n=100)
    dot_case("dot_c1_b64", x, y, 100, 64, 128)
    # ---- c5b shape at small batch, each precision of the sweep
    for p in (64, 128, 256, 512, 1024, 4096):
        n = 200 if p >= 1024 else 1000
        x, y = gen.config5_dots(batch=4 if p >= 1024 else 6, n=n, p=p)
        dot_case(f"dot_c5_p{p}", x, y, n, x.count // n, p)
    # ---- mixed edge cases (random_dot_instance style): limb counts 1..4,
    #      zeros, radii, specials -> Fallback, subtract, initial, strides
    rng = np.random.Generator(np.random.PCG64(20260101))
    for n in (1, 2, 7, 33, 50):
        ex, ey = gen.edge_dots(rng, 96, n)
        init, _ = gen.edge_dots(rng, 96, 1)
        for p in (8, 53, 128, 256, 1024):
            dot_case(f"dot_edge_n{n}_p{p}", ex, ey, n, 96, p, initial=init if n % 2 else None,
                     subtract=(p % 3 == 0))
    ex, ey = gen.edge_dots(rng, 64, 20, specials=False)
    rev = apb_dot_index(1, 19, 20, 0, -1, 0, 20, 0, 1)
    dot_case("dot_edge_reverse", ex, ey, 20, 64, 128, idx=rev)
    dot_case("dot_edge_approx", ex, ey, 20, 64, 200, mode=1)
    dot_case("dot_edge_noreduce", ex, ey, 20, 64, 1000, disable_reduction=True)
    # ---- known answers restated from tests/test_dot.cpp
    ones = ball_from_i64([1] * 100)
    dot_case("dot_kat_ones100", ones, ones, 100, 1, 128)          # :24-33 padding 11, extend 8, n_s 3
    seven = ball_from_i64([1] * 7)
    dot_case("dot_kat_seven", seven, seven, 7, 1, 53)             # :125-135 -> exactly 7
    m1, p1 = ball_from_i64([-1]), ball_from_i64([1])
    dot_case("dot_kat_minus_one", m1, p1, 1, 1, 64)               # :110-123 negation path
    # precision reduction p 1000 -> 40 (:35-46): x = [0.5 +- 2^-11], y = 0.5
    xr = ball_from_i64([1])
    xr.exp[:] = 0
    xr.rad_man[:] = 1 << 29
    xr.rad_exp[:] = -10
    yr = ball_from_i64([1])
    yr.exp[:] = 0
    dot_case("dot_kat_reduction", xr, yr, 1, 1, 1000)
    # exact cancellation: x.y + (-x).y = 0 exactly
    xc, yc = gen.random_balls(rng, 8, 256, e_lo=-3, e_hi=3), gen.random_balls(rng, 8, 256, e_lo=-3, e_hi=3)
    xneg = BallArray(xc.mant.copy(), xc.exp.copy(), xc.kind ^ np.uint8(APB_SIGN), xc.rad_man.copy(),
                     xc.rad_exp.copy())
    dot_case("dot_kat_cancel", xc.concat(xneg), yc.concat(yc), 16, 1, 256)
    # NaN input -> indeterminate
    xn = ball_from_i64([1, 2, 3])
    xn.kind[1] = APB_NAN
    xn.mant[1] = 0
    dot_case("dot_kat_nan", xn, ball_from_i64([1, 1, 1]), 3, 1, 64)

    # ---- complex dots
    xr_, xi_ = gen.edge_dots(rng, 40, 9, specials=False)
    yr_, yi_ = gen.edge_dots(rng, 40, 9, specials=False)
    for p, mode in ((128, 0), (300, 0), (128, 1)):
        ore, oim = po.dot_complex_batch(xr_, xi_, yr_, yi_, 9, 40, p, which="ref", mode=mode)
        d = {"kind": np.array("cdot"), "n": np.int64(9), "batch": np.int64(40), "prec": np.int64(p),
             "mode": np.int64(mode)}
        for nm, arr in (("xre", xr_), ("xim", xi_), ("yre", yr_), ("yim", yi_), ("ore", ore), ("oim", oim)):
            d.update(pack(nm, arr))
        np.savez_compressed(os.path.join(OUT, f"cdot_p{p}_m{mode}.npz"), **d)

    # ---- matmul
    a, b = gen.config2_matrices(n=64)
    matmul_case("mm_c2_n64", a, b, 64, 64, 64, 128)
    a, b = gen.config3_matrices(n=80)
    matmul_case("mm_c3_n80", a, b, 80, 80, 80, 256)
    a, b = gen.config5_matrices(n=48, p=1024)
    matmul_case("mm_c5_n48_p1024", a, b, 48, 48, 48, 1024)
    a, b = gen.config5_matrices(n=40, p=64)
    matmul_case("mm_c5_n40_p64_auto", a, b, 40, 40, 40, 64, algo=0)   # below cutoff -> classical
    # multi-block: exponent jumps every 40 inner indices force 3 scaled blocks,
    # plus a short tail block (basecase) of 12
    n = 100
    k = np.arange(n)
    ea = np.tile((k // 35) * 600, n) + np.repeat(np.arange(n) % 5, n)
    eb = np.repeat(-(k // 35) * 600, n)
    a = gen.random_balls(rng, n * n, 128, exps=ea, rad_k=110, rad_frac=0.2, zero_frac=0.05)
    b = gen.random_balls(rng, n * n, 128, exps=eb, rad_k=110, rad_frac=0.2, zero_frac=0.05)
    matmul_case("mm_multiblock_n100", a, b, n, n, n, 128)
    # rectangular
    a = gen.random_balls(rng, 70 * 90, 192, e_lo=-5, e_hi=5, rad_k=190)
    b = gen.random_balls(rng, 90 * 65, 192, e_lo=-5, e_hi=5, rad_k=190)
    matmul_case("mm_rect_70x90x65", a, b, 70, 90, 65, 192)
    # complex
    parts = gen.config4_matrices(n=64, p=256)
    cre, cim = po.matmul_complex(*parts, 64, 64, 64, 256)
    d = {"kind": np.array("cmatmul"), "M": np.int64(64), "K": np.int64(64), "N": np.int64(64),
         "prec": np.int64(256)}
    for nm, arr in zip(("are", "aim", "bre", "bim", "cre", "cim"), (*parts, cre, cim)):
        d.update(pack(nm, arr))
    np.savez_compressed(os.path.join(OUT, "cmm_c4_n64_p256.npz"), **d)
    # radius product KAT (tests/test_matmul.cpp:178-220): random Mag planes
    m_, n_, k_ = 33, 47, 29
    pm = (np.uint32(1 << 29) + rng.integers(0, 1 << 29, size=m_ * n_).astype(np.uint32)).astype(np.uint32)
    qm = (np.uint32(1 << 29) + rng.integers(0, 1 << 29, size=n_ * k_).astype(np.uint32)).astype(np.uint32)
    pm[rng.random(m_ * n_) < 0.2] = 0
    pe = rng.integers(-300, 300, size=m_ * n_).astype(np.int64)
    qe = rng.integers(-300, 300, size=n_ * k_).astype(np.int64)
    om, oe = po.radius_matmul_upper(pm, pe, qm, qe, m_, n_, k_)
    np.savez_compressed(os.path.join(OUT, "radius_kat.npz"), kind=np.array("radius"), m=m_, n=n_, k=k_,
                        pm=pm, pe=pe, qm=qm, qe=qe, om=om, oe=oe)
    print("golden fixtures written to", OUT, len(os.listdir(OUT)), "files")


if __name__ == "__main__":
    import sys
    os.makedirs(OUT, exist_ok=True)
    if "--poly" in sys.argv:  # only the poly fixtures (the others stay byte-identical)
        poly_cases()
    else:
        main()
        poly_cases()
