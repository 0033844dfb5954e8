"""CPU: the C restatement (oracle/apb_oracle.c) reproduces the reference's
golden vectors bit for bit, and the reference build itself is consistent
with them.  No GPU involved."""
import numpy as np
import pytest

import pyoracle as po
from golden_io import balls, files, index, name
from paper_1901_04289_b200.balls import DOT_STATE_DTYPE

DOT = files("dot_")
MM = files("mm_")


@pytest.mark.parametrize("path", DOT, ids=[name(p) for p in DOT])
@pytest.mark.parametrize("which", ["port", "ref"])
def test_dot_golden(path, which):
    d = np.load(path)
    x, y, init, out = balls(d, "x"), balls(d, "y"), balls(d, "init"), balls(d, "out")
    n, batch, prec = int(d["n"]), int(d["batch"]), int(d["prec"])
    kw = dict(initial=init, subtract=bool(d["subtract"]), idx=index(d),
              disable_reduction=bool(d["disable_reduction"]))
    got = po.dot_batch(x, y, n, batch, prec, which=which, mode=int(d["mode"]), L_out=out.L, **kw)
    assert got.identical(out).all()
    if int(d["mode"]):
        return  # dot_setup is only exposed with radius scanning (include/apball/dot.hpp:57)
    st, acc = po.dot_state(x, y, n, batch, prec, which=which, **kw)
    exp_st = d["state"]
    for f in ("status", "e_max", "e_rad", "n_nonzero", "p_eff", "n_s", "e_s", "err", "srad"):
        np.testing.assert_array_equal(st[f], exp_st[f], err_msg=f)
    proceed = exp_st["status"] == 0
    np.testing.assert_array_equal(acc[proceed], d["acc"][proceed])


@pytest.mark.parametrize("path", files("cdot_"), ids=[name(p) for p in files("cdot_")])
def test_complex_dot_golden(path):
    d = np.load(path)
    args = [balls(d, k) for k in ("xre", "xim", "yre", "yim")]
    ore, oim = po.dot_complex_batch(*args, int(d["n"]), int(d["batch"]), int(d["prec"]),
                                    which="port", mode=int(d["mode"]))
    assert ore.identical(balls(d, "ore")).all()
    assert oim.identical(balls(d, "oim")).all()


@pytest.mark.parametrize("path", MM, ids=[name(p) for p in MM])
def test_matmul_golden_port(path):
    d = np.load(path)
    a, b, c = balls(d, "a"), balls(d, "b"), balls(d, "c")
    M, K, N, prec = (int(d[k]) for k in ("M", "K", "N", "prec"))
    plan = po.plan_blocks(a, b, M, K, N, prec, which="port")
    assert plan == [tuple(int(v) for v in r) for r in d["plan"]]
    for bi in d["int_blocks"]:
        lo, hi, _ = plan[int(bi)]
        T = d[f"int_{bi}_T"]
        rs, cs, got = po.block_int_product(a, b, M, K, N, lo, hi, T.shape[1], which="port")
        np.testing.assert_array_equal(rs, d[f"int_{bi}_rows"])
        np.testing.assert_array_equal(cs, d[f"int_{bi}_cols"])
        np.testing.assert_array_equal(got, T)
    got, nb = po.matmul(a, b, M, K, N, prec, which="port", algo=int(d["algo"]))
    assert got.identical(c).all()


def test_complex_matmul_golden_port():
    d = np.load(files("cmm_")[0])
    args = [balls(d, k) for k in ("are", "aim", "bre", "bim")]
    M, K, N, prec = (int(d[k]) for k in ("M", "K", "N", "prec"))
    cre, cim = po.matmul_complex(*args, M, K, N, prec, which="port")
    assert cre.identical(balls(d, "cre")).all()
    assert cim.identical(balls(d, "cim")).all()


def test_radius_kat_port():
    d = np.load(files("radius_")[0])
    om, oe = po.radius_matmul_upper(d["pm"], d["pe"], d["qm"], d["qe"], int(d["m"]), int(d["n"]),
                                    int(d["k"]), which="port")
    np.testing.assert_array_equal(om, d["om"])
    np.testing.assert_array_equal(oe[om != 0], d["oe"][om != 0])


def test_kat_plan_geometry():
    """tests/test_dot.cpp:24-33: N=100 ones at p=128 -> padding 11, extend 8, n_s 3."""
    d = np.load([p for p in DOT if p.endswith("dot_kat_ones100.npz")][0])
    st = d["state"][0]
    assert (st["padding"], st["extend"], st["n_s"], st["p_eff"]) == (11, 8, 3, 128)
    assert st["e_s"] == st["e_max"] + 8


def test_kat_reduction():
    """tests/test_dot.cpp:35-46: e_max 0, e_rad -10 -> p_eff 40."""
    d = np.load([p for p in DOT if p.endswith("dot_kat_reduction.npz")][0])
    st = d["state"][0]
    assert (st["e_max"], st["e_rad"], st["p_eff"]) == (0, -10, 40)


@pytest.mark.parametrize("suite,trials", [("dot_containment", 300), ("dot_exact_zero", 300),
                                           ("dot_accuracy", 300), ("matmul_planner", 0)])
def test_reference_verify_suites(suite, trials):
    """the reference's own verify suites pass on the build used as oracle"""
    assert po.run_verify_suite(suite, trials, 7) == 0


POLY = files("poly_")
SERIES = files("series_")


@pytest.mark.parametrize("path", POLY, ids=[name(p) for p in POLY])
@pytest.mark.parametrize("which", ["port", "ref"])
def test_poly_mullow_golden(path, which):
    """poly_mullow_classical (src/poly.cpp:11-26) fixtures, incl. the restated
    tests/test_poly.cpp:15-25 KAT (1+x)^2 = 1 + 2x + x^2"""
    d = np.load(path)
    a, b, out = balls(d, "a"), balls(d, "b"), balls(d, "out")
    got = po.poly_mullow(a, b, int(d["len"]), int(d["prec"]), which=which)
    assert got.identical(out).all()


@pytest.mark.parametrize("path", SERIES, ids=[name(p) for p in SERIES])
@pytest.mark.parametrize("which", ["port", "ref"])
def test_series_exp_golden(path, which):
    """series_exp_basecase (src/poly.cpp:28-46) fixtures, incl. the restated
    tests/test_poly.cpp:33-56 KATs (exp(x) -> 1/k!, exp(0) -> 1)"""
    d = np.load(path)
    a, out = balls(d, "a"), balls(d, "out")
    got = po.series_exp(a, int(d["len"]), int(d["prec"]), which=which)
    assert got.identical(out).all()


def test_poly_kat_values():
    """(1+x)^2 = 1 + 2x + x^2 exactly; exp(x) has an exact 1/2 at k=2 (tests/test_poly.cpp:15-48)"""
    d = np.load(files("poly_kat_square")[0])
    out = balls(d, "out")
    assert list(out.exp) == [1, 2, 1] and all(out.rad_man == 0)
    assert all(out.mant[:, -1] == np.uint64(1 << 63))
    e = balls(np.load(files("series_kat_x")[0]), "out")
    assert e.rad_man[2] == 0 and e.exp[2] == 0 and e.mant[2, -1] == np.uint64(1 << 63)  # 1/2


@pytest.mark.parametrize("which", ["port", "ref"])
def test_series_exp_rejects_nonzero_constant(which):
    """tests/test_poly.cpp:58-62: std::domain_error for a_0 != 0"""
    from paper_1901_04289_b200.balls import BallArray
    with pytest.raises(ValueError):
        po.series_exp(BallArray.from_i64([1]), 4, 64, which=which)
