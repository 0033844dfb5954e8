"""GPU parity: batched dot kernels (libapb_b200.so) vs the reference.

Bit-exact: output balls, plan, accumulator limbs, err and srad equal the
reference's dot_setup/dot_init/dot_accumulate_term/dot_finalize
(golden fixtures from the reference + live oracle/_ref runs on the box)."""
import numpy as np
import pytest

import pyoracle as po
from golden_io import balls, files, index, name
from paper_1901_04289_b200 import gen
from paper_1901_04289_b200.balls import BallArray, flat_index

pytestmark = pytest.mark.gpu

DOT = files("dot_")


def _dev(a):
    return a.to_device() if a is not None else None


@pytest.mark.parametrize("path", DOT, ids=[name(p) for p in DOT])
def test_dot_golden_gpu(path):
    from paper_1901_04289_b200 import ops
    d = np.load(path)
    x, y, init, out = balls(d, "x"), balls(d, "y"), balls(d, "init"), balls(d, "out")
    n, batch, prec = int(d["n"]), int(d["batch"]), int(d["prec"])
    got, st, acc = ops.dot_batch(_dev(x), _dev(y), n, batch, prec, initial=_dev(init),
                                 subtract=bool(d["subtract"]), index=index(d),
                                 mode="approx" if int(d["mode"]) else "ball", want_state=True,
                                 acc_stride=d["acc"].shape[1],
                                 disable_precision_reduction=bool(d["disable_reduction"]))
    got = got.to_host()
    ok = got.identical(out)
    assert ok.all(), f"{(~ok).sum()} of {batch} dots differ, first {np.nonzero(~ok)[0][:8]}"
    if int(d["mode"]):
        return  # the reference exposes dot_setup only with radius scanning (dot.hpp:57)
    exp_st = d["state"]
    for f in ("status", "e_max", "e_rad", "n_nonzero", "p_eff", "n_s", "e_s", "err", "srad"):
        np.testing.assert_array_equal(st[f], exp_st[f], err_msg=f)
    proceed = exp_st["status"] == 0
    np.testing.assert_array_equal(acc[proceed], d["acc"][proceed])


@pytest.mark.parametrize("path", files("cdot_"), ids=[name(p) for p in files("cdot_")])
def test_complex_dot_golden_gpu(path):
    from paper_1901_04289_b200 import ops
    d = np.load(path)
    args = [balls(d, k).to_device() for k in ("xre", "xim", "yre", "yim")]
    ore, oim = ops.dot_complex_batch(*args, int(d["n"]), int(d["batch"]), int(d["prec"]),
                                     mode="approx" if int(d["mode"]) else "ball")
    assert ore.to_host().identical(balls(d, "ore")).all()
    assert oim.to_host().identical(balls(d, "oim")).all()


def test_c1_full_batch_vs_reference():
    """config 1 at full size: all 65,536 dots bit-identical to the reference
    (reference timed multithreaded on the host), sampled containment."""
    from paper_1901_04289_b200 import ops
    import os
    x, y = gen.config1_dots()
    got = ops.dot_batch(x.to_device(), y.to_device(), 100, 65536, 128).to_host()
    ref = po.dot_batch(x, y, 100, 65536, 128, which="ref", threads=os.cpu_count() or 8)
    ok = got.identical(ref)
    assert ok.all(), f"{(~ok).sum()} dots differ"
    sample = np.arange(0, 65536, 257)
    xs = x.take((sample[:, None] * 100 + np.arange(100)).ravel())
    ys = y.take((sample[:, None] * 100 + np.arange(100)).ravel())
    assert po.dot_contains(xs, ys, 100, len(sample), got.take(sample)).all()


@pytest.mark.parametrize("p", [64, 128, 256, 512, 1024, 4096])
def test_c5_dots_vs_reference(p):
    from paper_1901_04289_b200 import ops
    n = 1000 if p <= 1024 else 300
    batch = 64 if p <= 512 else 16
    x, y = gen.config5_dots(batch=batch, n=n, p=p)
    got = ops.dot_batch(x.to_device(), y.to_device(), n, batch, p).to_host()
    ref = po.dot_batch(x, y, n, batch, p, which="ref", threads=8)
    assert got.identical(ref).all()


def test_edge_random_vs_reference():
    from paper_1901_04289_b200 import ops
    rng = np.random.Generator(np.random.PCG64(99))
    for n in (1, 5, 31, 32, 33, 64, 129, 300):
        for p in (2, 30, 64, 100, 128, 129, 256, 500, 700, 2000):
            x, y = gen.edge_dots(rng, 40, n)
            init, _ = gen.edge_dots(rng, 40, 1)
            sub = bool(rng.integers(0, 2))
            kw = dict(initial=init if n % 3 == 0 else None, subtract=sub)
            got = ops.dot_batch(x.to_device(), y.to_device(), n, 40, p,
                                initial=_dev(kw["initial"]), subtract=sub).to_host()
            ref = po.dot_batch(x, y, n, 40, p, which="ref", **kw)
            ok = got.identical(ref)
            assert ok.all(), (n, p, np.nonzero(~ok)[0][:5])


def test_term_counts_just_past_a_multiple_of_32():
    """dots of 32 k + (1..4) terms (config 1 has 100 = 96 + 4: the last register slot of the register
    kernel is mostly padding): batches that are no multiple of 8, edge values (zeros, specials ->
    Fallback, radii), window sizes 2 and 3, subtract, state / accumulator outputs"""
    from paper_1901_04289_b200 import ops
    rng = np.random.Generator(np.random.PCG64(4242))
    for n in (33, 34, 36, 65, 67, 68, 97, 98, 100):
        for p, batch in ((64, 70), (128, 203), (129, 64), (53, 97)):
            x, y = gen.edge_dots(rng, batch, n, max_limbs=2, spread=40 if p > 64 else 6)
            sub = bool(rng.integers(0, 2))
            got = ops.dot_batch(x.to_device(), y.to_device(), n, batch, p, subtract=sub).to_host()
            ref = po.dot_batch(x, y, n, batch, p, which="ref", subtract=sub)
            ok = got.identical(ref)
            assert ok.all(), (n, p, batch, np.nonzero(~ok)[0][:5])
    # config-1 distributions at full length, accumulator limbs and plan checked against the reference
    x, y = gen.config1_dots(batch=1000)
    got, st, acc = ops.dot_batch(x.to_device(), y.to_device(), 100, 1000, 128, want_state=True, acc_stride=3)
    ref = po.dot_batch(x, y, 100, 1000, 128, which="ref")
    rst, racc = po.dot_state(x, y, 100, 1000, 128, which="ref", acc_stride=3)
    assert got.to_host().identical(ref).all()
    for f in ("status", "e_max", "e_rad", "n_nonzero", "p_eff", "n_s", "e_s", "err"):
        np.testing.assert_array_equal(st[f], rst[f], err_msg=f)
    proceed = rst["status"] == 0
    np.testing.assert_array_equal(np.asarray(acc).reshape(1000, 3)[proceed], racc[proceed])


def test_host_entry_matches_device_entry():
    from paper_1901_04289_b200 import ops
    x, y = gen.config1_dots(batch=512)
    a = ops.dot_batch(x.to_device(), y.to_device(), 100, 512, 128).to_host()
    b = ops.dot_batch_host(x, y, 100, 512, 128)
    assert a.identical(b).all()


def test_reference_shaped_dot_ball():
    """dot_ball with negative strides and an initial value, as poly/basecase call it"""
    from paper_1901_04289_b200 import ops
    rng = np.random.Generator(np.random.PCG64(5))
    x, y = gen.edge_dots(rng, 1, 25, specials=False)
    init, _ = gen.edge_dots(rng, 1, 1, specials=False)
    got = ops.dot_ball(init, True, x, -1, y, 1, 25, 150, x_off=24)
    from paper_1901_04289_b200.balls import apb_dot_index
    ref = po.dot_batch(x, y, 25, 1, 150, which="ref", initial=init, subtract=True,
                       idx=apb_dot_index(1, 24, 0, 0, -1, 0, 0, 0, 1))
    assert got.identical(ref).all()


@pytest.mark.parametrize("hook", ["APB_DOT_KEEP", "APB_DOT_STAGE", "APB_DOT_GENERIC", "APB_DOT_TPD", "APB_DOT_BULK",
                                  "APB_DOT_NOREG", "APB_REG_TPD", "APB_REG_PF"])
def test_dot_kernel_variants(hook):
    """the register-resident (KEEP) and cp.async-staged (STAGE) dot kernels,
    selected by their tuning hooks in a subprocess, on the golden and edge cases"""
    import os
    import subprocess
    import sys
    val = {"APB_DOT_TPD": "32", "APB_REG_TPD": "16"}.get(hook, "1")  # TPD 32: one warp per dot
    env = dict(os.environ, **{hook: val})
    if hook in ("APB_DOT_KEEP", "APB_DOT_STAGE", "APB_DOT_TPD", "APB_DOT_BULK"):
        env["APB_DOT_NOREG"] = "1"  # these select among the round-1 kernels
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-k",
                        "test_dot_golden_gpu or test_edge_random or test_host_entry or test_c1_full",
                        os.path.abspath(__file__)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]


@pytest.mark.parametrize("force,bits,p", [(True, 192, 1024), (True, 128, 2048), (True, 64, 256),
                                          (False, 192, 1024), (True, 192, 64)])
def test_complex_threeprod_hits_vs_reference(force, bits, p):
    """dot_threeprod_hits (include/apball/dot.hpp:54) counted like the reference's
    gate (src/dot.cpp:427-458), on the inputs of its verify suite (exact values,
    <= 3 limbs, exponents in [-80, 80], src/bench.cpp:587-625); the outputs equal
    the reference's (rewritten) results -- the rewrite is unobservable"""
    from paper_1901_04289_b200 import ops
    rng = np.random.Generator(np.random.PCG64(100 + bits + p))
    n, batch = 12, 64
    parts = [gen.random_balls(rng, n * batch, bits, e_lo=-80, e_hi=80) for _ in range(4)]
    ore, oim, hits = ops.dot_complex_batch(*[q.to_device() for q in parts], n, batch, p,
                                           force_threeprod=force, want_hits=True)
    rre, rim, rhits = po.dot_complex_batch(*parts, n, batch, p, force_threeprod=force, want_hits=True)
    assert ore.to_host().identical(rre).all() and oim.to_host().identical(rim).all()
    assert hits == rhits
    if force and p >= 1024:
        assert hits > 0
