"""CPU: host-side logic of the package (no GPU): generators, SoA layout
helpers, argument checks of the reference-shaped API."""
import numpy as np
import pytest

from paper_1901_04289_b200 import gen
from paper_1901_04289_b200.balls import (APB_FINITE, APB_SIGN, BallArray, flat_index, limbs_for)


def test_generators_deterministic_and_shaped():
    a1, b1 = gen.config2_matrices(n=16)
    a2, b2 = gen.config2_matrices(n=16)
    assert a1.identical(a2).all() and b1.identical(b2).all()
    assert a1.L == 2 and a1.count == 256
    # 128-bit mantissas in [0.5, 1): top bit set, exponents in [-4, 4]
    assert np.all(a1.mant[:, -1] >> np.uint64(63) == 1)
    assert a1.exp.min() >= -4 and a1.exp.max() <= 4
    # radius 2^-130 |m|: Mag exponent = e - 130 (+1 when the 30-bit bound carries)
    d = a1.rad_exp - a1.exp
    assert set(np.unique(d)) <= {-130, -129}


def test_config3_structure():
    a, b = gen.config3_matrices(n=64)
    fin = (a.kind & 7) == APB_FINITE
    assert 0.03 < 1 - fin.mean() < 0.2           # ~10% exact zeros
    rows = a.exp.reshape(64, 64)
    for i in range(64):                          # row i at exponent e_i
        vals = rows[i][fin.reshape(64, 64)[i]]
        assert len(set(vals.tolist())) == 1
    has_rad = (a.rad_man != 0) & fin
    assert 0.01 < has_rad.sum() / fin.sum() < 0.12


def test_limbs_and_index():
    assert [limbs_for(p) for p in (2, 64, 65, 128, 4096)] == [1, 1, 2, 2, 64]
    ix = flat_index(100)
    assert (ix.bdiv, ix.xs1, ix.xstep) == (1, 100, 1)


def test_widen_preserves_value():
    a, _ = gen.config1_dots(batch=2, n=4)
    w = a.widen(5)
    assert w.L == 5 and np.all(w.mant[:, :3] == 0) and a.identical(w).all()


def test_identical_detects_differences():
    a, _ = gen.config2_matrices(n=8)
    b = BallArray(a.mant.copy(), a.exp.copy(), a.kind.copy(), a.rad_man.copy(), a.rad_exp.copy())
    b.kind[3] ^= np.uint8(APB_SIGN)
    b.mant[5, 0] ^= np.uint64(1)
    ok = a.identical(b)
    assert not ok[3] and not ok[5] and ok.sum() == 62


def test_dimension_mismatch_raises_before_device_work():
    ops = pytest.importorskip("paper_1901_04289_b200.ops")
    from paper_1901_04289_b200 import _lib
    import os
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    a, b = gen.config2_matrices(n=4)
    with pytest.raises(_lib.InvalidArgument):
        ops.block_matmul_ball(ops.BallMatrix(a, 4, 4), ops.BallMatrix(b, 2, 8), 128)


def test_dispatch_cutoffs():
    ops = pytest.importorskip("paper_1901_04289_b200.ops")
    # matmul_dispatch_cutoff (src/matmul.cpp:517-524)
    assert [ops.matmul_dispatch_cutoff(p) for p in (53, 64, 128, 256, 512, 1024, 4096)] == \
        [60, 60, 56, 52, 48, 44, 40]
