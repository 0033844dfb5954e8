"""Seeded random sweep of the matmul and dot paths against the reference
(oracle/_ref): shapes, precisions, exponent spreads (single- and multi-block
plans), radius and zero densities drawn per case; every output ball must be
bit-identical.  Sizes are bounded so each reference run takes seconds."""
import os

import numpy as np
import pytest

import pyoracle as po
from paper_1901_04289_b200 import gen

pytestmark = pytest.mark.gpu

CASES = list(range(40))


def _case(seed):
    rng = np.random.default_rng(0xF0225 + seed)
    p = int(rng.choice([53, 64, 100, 128, 192, 256, 320, 512, 700, 1024, 2048]))
    lim = 6e7 / max(1.0, (p / 64) ** 2)  # M K N bound for a quick reference run
    while True:
        M, K, N = (int(v) for v in rng.integers(20, 700, size=3))
        if M * K * N <= lim:
            break
    spread = int(rng.choice([0, 4, 60, 300, 900]))  # row/column exponent offsets
    ea = np.repeat(rng.integers(-spread, spread + 1, size=M), K) + rng.integers(-3, 4, size=M * K)
    eb = np.tile(rng.integers(-spread, spread + 1, size=N), K) + rng.integers(-3, 4, size=K * N)
    if rng.random() < 0.3:  # inner-index jumps: multi-block plans
        jump = (np.arange(K) // max(1, K // 3)) * int(rng.integers(100, 700))
        ea = ea + np.tile(jump, M)
        eb = eb - np.repeat(jump, N)
    rf = float(rng.choice([0.0, 0.05, 0.5, 1.0]))
    zf = float(rng.choice([0.0, 0.1]))
    a = gen.random_balls(rng, M * K, p, exps=ea, rad_k=p + 2, rad_frac=rf, zero_frac=zf)
    b = gen.random_balls(rng, K * N, p, exps=eb, rad_k=p + 2, rad_frac=rf, zero_frac=zf)
    return a, b, M, K, N, p


@pytest.mark.parametrize("seed", CASES)
def test_matmul_fuzz(seed):
    from paper_1901_04289_b200 import ops
    a, b, M, K, N, p = _case(seed)
    A, B = ops.BallMatrix(a.to_device(), M, K), ops.BallMatrix(b.to_device(), K, N)
    got = ops.matmul_auto(A, B, p).balls.to_host()
    ref, _ = po.matmul(a, b, M, K, N, p, which="ref", algo=0, threads=os.cpu_count() or 8)
    ok = got.identical(ref)
    assert ok.all(), f"case {seed} (M={M} K={K} N={N} p={p}): {(~ok).sum()} entries differ"
    # and the repeated call (graph replay / speculative step) on the same buffers
    out = ops.matmul_auto(A, B, p)
    for _ in range(2):
        again = ops.matmul_auto(A, B, p, out=out).balls.to_host()
        assert again.identical(ref).all()


@pytest.mark.parametrize("seed", CASES)
def test_dot_fuzz(seed):
    from paper_1901_04289_b200 import ops
    rng = np.random.default_rng(0xD07 + seed)
    p = int(rng.choice([32, 64, 128, 192, 256, 512, 1024, 2048]))
    n = int(rng.integers(1, 400))
    batch = int(rng.integers(1, 3000 if p <= 512 else 300))
    e_span = int(rng.choice([2, 40, 400]))
    x = gen.random_balls(rng, batch * n, p, e_lo=-e_span, e_hi=e_span, rad_k=p + 3,
                         rad_frac=float(rng.choice([0.0, 0.5, 1.0])), zero_frac=float(rng.choice([0.0, 0.2])))
    y = gen.random_balls(rng, batch * n, p, e_lo=-e_span, e_hi=e_span, rad_k=p + 3,
                         rad_frac=float(rng.choice([0.0, 0.5])), zero_frac=0.0)
    got = ops.dot_batch(x.to_device(), y.to_device(), n, batch, p).to_host()
    ref = po.dot_batch(x, y, n, batch, p, which="ref", threads=os.cpu_count() or 8)
    ok = got.identical(ref)
    assert ok.all(), f"case {seed} (n={n} batch={batch} p={p}): {(~ok).sum()} dots differ"
