"""GPU parity: the polynomial consumers of the fused dot
-- poly_mullow_classical as one batch of variable-length negative-stride dots,
series_exp_basecase as the sequential recurrence -- bit-identical to the
reference (golden fixtures and live oracle/_ref runs)."""
import numpy as np
import pytest

import pyoracle as po
from golden_io import balls, files, name
from paper_1901_04289_b200 import gen
from paper_1901_04289_b200.balls import BallArray

pytestmark = pytest.mark.gpu

POLY = files("poly_")
SERIES = files("series_")


@pytest.mark.parametrize("path", POLY, ids=[name(p) for p in POLY])
def test_poly_mullow_golden_gpu(path):
    from paper_1901_04289_b200 import ops
    d = np.load(path)
    a, b, out = balls(d, "a"), balls(d, "b"), balls(d, "out")
    got = ops.poly_mullow_classical(a.to_device(), b.to_device(), int(d["len"]), int(d["prec"]))
    assert got.to_host().take(range(int(d["len"]))).identical(out).all()


@pytest.mark.parametrize("path", SERIES, ids=[name(p) for p in SERIES])
def test_series_exp_golden_gpu(path):
    from paper_1901_04289_b200 import ops
    d = np.load(path)
    a, out = balls(d, "a"), balls(d, "out")
    got = ops.series_exp_basecase(a.to_device(), int(d["len"]), int(d["prec"]))
    assert got.to_host().take(range(int(d["len"]))).identical(out).all()


def test_poly_mullow_random_vs_reference():
    """lengths 0..~300 (empty operands, output longer/shorter than |a|+|b|-1),
    precisions 2..1000, zeros / radii / specials"""
    from paper_1901_04289_b200 import ops
    rng = np.random.Generator(np.random.PCG64(77))
    for q in range(24):
        la, lb = int(rng.integers(0, 300 if q % 4 == 0 else 40)), int(rng.integers(0, 40))
        ln = int(rng.integers(1, la + lb + 3))
        p = int(rng.choice([2, 30, 64, 100, 128, 200, 256, 512, 1000]))
        a, _ = gen.edge_dots(rng, 1, max(la, 1), specials=(q % 5 == 0))
        b, _ = gen.edge_dots(rng, 1, max(lb, 1), specials=False)
        a, b = a.take(range(la)), b.take(range(lb))
        ref = po.poly_mullow(a, b, ln, p)
        got = ops.poly_mullow_classical(a, b, ln, p)  # host entry (H2D, launch, D2H)
        assert got.identical(ref).all(), (q, la, lb, ln, p)


def test_series_exp_random_vs_reference():
    from paper_1901_04289_b200 import ops
    rng = np.random.Generator(np.random.PCG64(78))
    for q in range(10):
        la, ln = int(rng.integers(1, 30)), int(rng.integers(1, 40))
        p = int(rng.choice([2, 64, 128, 256, 700]))
        a, _ = gen.edge_dots(rng, 1, la, specials=False)
        a.kind[0], a.mant[0], a.exp[0], a.rad_man[0], a.rad_exp[0] = 0, 0, 0, 0, 0
        ref = po.series_exp(a, ln, p)
        got = ops.series_exp_basecase(a, ln, p)
        assert got.identical(ref).all(), (q, la, ln, p)


def test_series_exp_rejects_nonzero_constant_gpu():
    from paper_1901_04289_b200 import _lib, ops
    with pytest.raises(_lib.InvalidArgument):
        ops.series_exp_basecase(BallArray.from_i64([1]).to_device(), 4, 64)


def test_poly_mullow_large_vs_reference():
    """one long product at the measured size (len 1024, p=128)"""
    from paper_1901_04289_b200 import ops
    rng = np.random.Generator(np.random.PCG64(79))
    a, _ = gen.edge_dots(rng, 1, 1024, specials=False)
    b, _ = gen.edge_dots(rng, 1, 1024, specials=False)
    ref = po.poly_mullow(a, b, 1024, 128)
    got = ops.poly_mullow_classical(a.to_device(), b.to_device(), 1024, 128).to_host()
    assert got.identical(ref).all()


def test_series_exp_warp_matches_serial_and_reference():
    """the warp-cooperative series_exp (lanes over each step's dot) equals the
    one-thread version (APB_SERIES_SERIAL) and the reference at a length where
    every step's dot spans several lane rounds"""
    import os
    import subprocess
    import sys
    from paper_1901_04289_b200 import ops
    rng = np.random.Generator(np.random.PCG64(4242))
    la, ln, p = 150, 160, 256
    a, _ = gen.edge_dots(rng, 1, la, specials=False)
    a.kind[0], a.mant[0], a.exp[0], a.rad_man[0], a.rad_exp[0] = 0, 0, 0, 0, 0
    ref = po.series_exp(a, ln, p)
    got = ops.series_exp_basecase(a, ln, p)
    assert got.identical(ref).all()
    env = dict(os.environ, APB_SERIES_SERIAL="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-k", "test_series_exp and not warp",
                        os.path.abspath(__file__)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
