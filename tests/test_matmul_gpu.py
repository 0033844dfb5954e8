"""GPU parity: block ball matmul (scale/pack -> tcgen05 int8 slice GEMM ->
recombine -> radius) vs the reference.  Exact integer block products, block
plans, midpoints and radii are compared bit for bit."""
import os

import numpy as np
import pytest

import pyoracle as po
from golden_io import balls, files, name
from paper_1901_04289_b200 import gen

pytestmark = pytest.mark.gpu

MM = files("mm_")


def _mat(a, r, c):
    from paper_1901_04289_b200 import ops
    return ops.BallMatrix(a.to_device(), r, c)


@pytest.mark.parametrize("path", MM, ids=[name(p) for p in MM])
def test_matmul_golden_gpu(path):
    from paper_1901_04289_b200 import ops
    d = np.load(path)
    a, b, c = balls(d, "a"), balls(d, "b"), balls(d, "c")
    M, K, N, prec, algo = (int(d[k]) for k in ("M", "K", "N", "prec", "algo"))
    A, B = _mat(a, M, K), _mat(b, K, N)
    assert ops.plan_blocks(A, B, prec) == [tuple(int(v) for v in r) for r in d["plan"]]
    for bi in d["int_blocks"]:
        lo, hi, _ = (int(v) for v in d["plan"][int(bi)])
        T = d[f"int_{bi}_T"]
        rs, cs, got = ops.block_int_product(A, B, lo, hi, T.shape[1])
        np.testing.assert_array_equal(rs, d[f"int_{bi}_rows"])
        np.testing.assert_array_equal(cs, d[f"int_{bi}_cols"])
        bad = np.nonzero((got != T).any(axis=1))[0]
        assert len(bad) == 0, f"{len(bad)} entries of the exact product differ, first {bad[:5]}"
    f = {0: ops.matmul_auto, 1: ops.block_matmul_ball, 2: ops.classical_matmul_ball}[algo]
    got = f(A, B, prec).balls.to_host()
    ok = got.identical(c)
    assert ok.all(), f"{(~ok).sum()} of {M*N} entries differ, first {np.nonzero(~ok)[0][:5]}"


def test_complex_matmul_golden_gpu():
    from paper_1901_04289_b200 import ops
    d = np.load(files("cmm_")[0])
    M, K, N, prec = (int(d[k]) for k in ("M", "K", "N", "prec"))
    are, aim, bre, bim = (balls(d, k) for k in ("are", "aim", "bre", "bim"))
    cre, cim = ops.complex_matmul_ball(_mat(are, M, K), _mat(aim, M, K), _mat(bre, K, N), _mat(bim, K, N), prec)
    assert cre.balls.to_host().identical(balls(d, "cre")).all()
    assert cim.balls.to_host().identical(balls(d, "cim")).all()


def test_radius_kat_gpu():
    from paper_1901_04289_b200 import ops
    d = np.load(files("radius_")[0])
    om, oe = ops.radius_matmul_upper(d["pm"], d["pe"], d["qm"], d["qe"], int(d["m"]), int(d["n"]), int(d["k"]))
    np.testing.assert_array_equal(om, d["om"])
    np.testing.assert_array_equal(oe[om != 0], d["oe"][om != 0])


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_full_config_vs_reference(cfg):
    """configs 2 and 3 at full size, every entry bit-identical to block_matmul_ball
    (the reference runs row-split across the host cores; bit-identical for single-block plans)"""
    from paper_1901_04289_b200 import ops
    if cfg == "c2":
        a, b = gen.config2_matrices()
        n, p = 256, 128
    else:
        a, b = gen.config3_matrices()
        n, p = 512, 256
    got = ops.block_matmul_ball(_mat(a, n, n), _mat(b, n, n), p).balls.to_host()
    ref, nb = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
    ok = got.identical(ref)
    assert ok.all(), f"{(~ok).sum()} entries differ"


@pytest.mark.parametrize("hook", ["APB_FORCE_UNIT_GEMM=1", "APB_PACK_V1=1", "APB_RAD_V1=1", "APB_RAD_V2=1", "APB_RAD_ORDER=1",
                                  "APB_RAD_ORDER=0", "APB_RAD_ORDER=2", "APB_RAD_ORDER=3", "APB_BAND_BN=128", "APB_BAND_V2=1",
                                  "APB_NO_SPEC_PACK=1", "APB_NO_GRAPHS=1",
                                  "APB_RECOMBINE64=1", "APB_NO_RAD_FUSE=1", "APB_NO_PDL=1",
                                  "APB_NO_SPEC_STEP=1", "APB_NO_PRIO=1", "APB_RAD_SPLIT=1", "APB_RAD_BESIDE=1",
                                  "APB_BAND_KBNORM=1", "APB_NO_SCAN_PLANES=1", "APB_RAD_MAIN=1",
                                  "APB_RAD_NO_SMALL=1", "APB_NO_RAW_EPI=1", "APB_RAD_QUAD=1", "APB_RAD_QUAD=1,APB_RAD_QUAD_BESIDE=1",
                                  "APB_BAND_BN=128,APB_NO_RAW_EPI=1", "APB_BAND_KSPLIT=2", "APB_BAND_BN=128,APB_BAND_KSPLIT=2",
                                  "APB_BAND_BN=256,APB_BAND_KSPLIT=1", "APB_RAW32=1", "APB_RAW32=1,APB_BAND_KSPLIT=2", "APB_RAD_BOTH=1", "APB_RC_PDL=1", "APB_NO_RAD_ALONG=1", "APB_NO_EARLY_PACK=1", "APB_PACK_A1=1"])
def test_kernel_variants_golden(hook):
    """alternative kernels / schedules selected by the library's tuning hooks
    (unit GEMM used when a diagonal could overflow int32, byte-serial pack,
    list-based sparse radius, radius stream placement, 128-wide band tiles),
    on the golden cases and configs 2 and 3 in a subprocess"""
    import subprocess
    import sys
    env = dict(os.environ, **dict(kv.split("=") for kv in hook.split(",")))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-k",
                        "test_matmul_golden_gpu or test_full_config_vs_reference or test_repeated_calls or test_graph_replay", os.path.abspath(__file__)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_repeated_calls_replay_graphs(cfg):
    """the same operands and output buffer three times: the first call runs
    eagerly and captures the launch sequence, later calls replay the CUDA
    graphs; every result bit-identical to the reference, counters consistent"""
    from paper_1901_04289_b200 import ops
    if cfg == "c2":
        a, b = gen.config2_matrices()
        n, p = 256, 128
    else:
        a, b = gen.config3_matrices()
        n, p = 512, 256
    A, B = _mat(a, n, n), _mat(b, n, n)
    ref, _ = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
    out = ops.block_matmul_ball(A, B, p)
    launches = []
    for rep in range(3):
        ops.matmul_stats_reset() if hasattr(ops, "matmul_stats_reset") else None
        l0 = ops.launch_count()
        got = ops.block_matmul_ball(A, B, p, out=out)
        launches.append(ops.launch_count() - l0)
        assert got.balls.to_host().identical(ref).all(), f"rep {rep}"
    assert launches[1] == launches[2] and launches[1] > 0, launches


def test_graph_replay_tracks_new_inputs():
    """same buffers, new contents: the replayed graphs read the current data"""
    from paper_1901_04289_b200 import ops
    n, p = 256, 128
    a1, b1 = gen.config2_matrices(seed_salt=0)
    a2, b2 = gen.config2_matrices(seed_salt=7)
    A, B = _mat(a1, n, n), _mat(b1, n, n)
    out = ops.block_matmul_ball(A, B, p)
    ops.block_matmul_ball(A, B, p, out=out)
    # overwrite the device operands in place with the second pair
    for dst, src in ((A, a2), (B, b2)):
        d = src.to_device()
        for f in ("mant", "exp", "kind", "rad_man", "rad_exp"):
            getattr(dst.balls, f).copy_(getattr(d, f))
    got = ops.block_matmul_ball(A, B, p, out=out).balls.to_host()
    ref, _ = po.matmul(a2, b2, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
    assert got.identical(ref).all()


def test_repeated_calls_centred_radius_planes():
    """config-4-like radii (2^-515 |m|: beyond the range of the scan's uncentred planes): the first
    call redoes the radius with centred planes, later calls run the centred planes inside the
    speculative branch; a product whose planes are in range follows; all bit-identical"""
    from paper_1901_04289_b200 import ops
    n, p = 192, 512
    rng = gen.rng_for(4, 77)
    far = [gen.random_balls(rng, n * n, p, e_lo=-16, e_hi=16, rad_k=515) for _ in range(2)]
    near = [gen.random_balls(rng, n * n, p, e_lo=-16, e_hi=16, rad_k=300) for _ in range(2)]
    refs = {}
    for key, (a, b) in (("far", far), ("near", near)):
        refs[key], _ = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
    for k, key in enumerate(["far", "far", "far", "near", "near", "far"]):
        a, b = far if key == "far" else near
        got = ops.block_matmul_ball(_mat(a, n, n), _mat(b, n, n), p).balls.to_host()
        assert got.identical(refs[key]).all(), f"call {k} ({key})"
    # the same buffers again and again: 69 slices take the 72-slice pack template, the speculative
    # pack and the captured graphs (with the centred planes inside the radius branch)
    A, B = _mat(far[0], n, n), _mat(far[1], n, n)
    out = ops.block_matmul_ball(A, B, p)
    assert ops.matmul_stats()["last_slices_a"] > 64
    for k in range(4):
        got = ops.block_matmul_ball(A, B, p, out=out).balls.to_host()
        assert got.identical(refs["far"]).all(), f"replay {k}"


def test_graph_replay_slice_count_changes():
    """same buffers, but the exponent spread (and with it the slice counts) grows and shrinks between
    calls: the fused step's graph packs only the slices it speculates on, so a product that needs
    more must be re-packed by the host; all bit-identical"""
    from paper_1901_04289_b200 import ops
    n, p = 256, 128
    rng = gen.rng_for(2, 321)
    narrow = [gen.random_balls(rng, n * n, p, e_lo=-2, e_hi=2, rad_k=130) for _ in range(2)]
    wide = [gen.random_balls(rng, n * n, p, e_lo=-30, e_hi=30, rad_k=130) for _ in range(2)]
    refs, slices = {}, {}
    for key, (a, b) in (("narrow", narrow), ("wide", wide)):
        refs[key], _ = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
    A, B = _mat(narrow[0], n, n), _mat(narrow[1], n, n)
    out = ops.block_matmul_ball(A, B, p)
    for k, key in enumerate(["narrow"] * 4 + ["wide"] * 4 + ["narrow"] * 3 + ["wide", "narrow"]):
        a, b = narrow if key == "narrow" else wide
        for dst, src in ((A, a), (B, b)):
            d = src.to_device()
            for f in ("mant", "exp", "kind", "rad_man", "rad_exp"):
                getattr(dst.balls, f).copy_(getattr(d, f))
        got = ops.block_matmul_ball(A, B, p, out=out).balls.to_host()
        assert got.identical(refs[key]).all(), f"call {k} ({key})"
        slices[key] = ops.matmul_stats()["last_slices_a"]
    assert slices["wide"] > slices["narrow"], slices


def test_graph_replay_radius_variant_changes():
    """same buffers and slice counts, but the radius density flips between calls: the fused
    step's graph holds only the radius kernels of the last operands (sparse or dense), so a
    replay whose operands need the other kind must redo the radius products"""
    from paper_1901_04289_b200 import ops
    n, p = 256, 128
    rng = gen.rng_for(2, 123)
    dense = [gen.random_balls(rng, n * n, p, e_lo=-4, e_hi=4, rad_k=130) for _ in range(2)]
    sparse = [gen.random_balls(rng, n * n, p, e_lo=-4, e_hi=4, rad_k=130, rad_frac=0.04) for _ in range(2)]
    refs = {}
    for key, (a, b) in (("dense", dense), ("sparse", sparse)):
        refs[key], _ = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
    A, B = _mat(dense[0], n, n), _mat(dense[1], n, n)
    out = ops.block_matmul_ball(A, B, p)
    seq = ["dense"] * 4 + ["sparse"] * 4 + ["dense"] * 2 + ["sparse", "dense"]
    for k, key in enumerate(seq):
        a, b = dense if key == "dense" else sparse
        for dst, src in ((A, a), (B, b)):
            d = src.to_device()
            for f in ("mant", "exp", "kind", "rad_man", "rad_exp"):
                getattr(dst.balls, f).copy_(getattr(d, f))
        got = ops.block_matmul_ball(A, B, p, out=out).balls.to_host()
        assert got.identical(refs[key]).all(), f"call {k} ({key})"


@pytest.mark.parametrize("path", MM, ids=[name(p) for p in MM])
def test_imad_baseline_golden(path):
    """the CUDA-core IMAD-limb baseline of the exact block product equals the
    reference's int_matmul on every golden block (heights up to 19 x 32 bits)"""
    from paper_1901_04289_b200 import ops
    d = np.load(path)
    a, b = balls(d, "a"), balls(d, "b")
    M, K, N = (int(d[k]) for k in ("M", "K", "N"))
    A, B = _mat(a, M, K), _mat(b, K, N)
    checked = 0
    for bi in d["int_blocks"]:
        lo, hi, _ = (int(v) for v in d["plan"][int(bi)])
        T = d[f"int_{bi}_T"]
        try:
            rs, cs, got, ms = ops.block_int_product_imad(A, B, lo, hi, T.shape[1])
        except RuntimeError as e:
            assert "19 limbs" in str(e)
            continue
        np.testing.assert_array_equal(rs, d[f"int_{bi}_rows"])
        np.testing.assert_array_equal(cs, d[f"int_{bi}_cols"])
        bad = np.nonzero((got != T).any(axis=1))[0]
        assert len(bad) == 0, f"{len(bad)} entries differ, first {bad[:5]}"
        checked += 1
    assert checked or not len(d["int_blocks"]) or int(d["prec"]) > 512


def test_imad_baseline_matches_tensor_core_c3():
    """config 3 at full size: IMAD-limb and int8 tensor-core exact products agree bit for bit"""
    from paper_1901_04289_b200 import ops
    a, b = gen.config3_matrices()
    A, B = _mat(a, 512, 512), _mat(b, 512, 512)
    rs, cs, t8 = ops.block_int_product(A, B, 0, 512, 10)
    rs2, cs2, ti, ms = ops.block_int_product_imad(A, B, 0, 512, 10)
    np.testing.assert_array_equal(rs, rs2)
    np.testing.assert_array_equal(cs, cs2)
    np.testing.assert_array_equal(t8, ti)
    assert ms > 0


def test_multiblock_wide_vs_reference():
    """multi-block plan on a matrix wide enough for the 256-column band tiles
    (16-bit band digits through the general recombine, blocks after the first
    adding into C): bit-identical to block_matmul_ball, exact block products
    identical between the tensor-core and IMAD-limb paths"""
    from paper_1901_04289_b200 import ops
    rng = np.random.default_rng(0xB200 + 300)
    n = 300
    k = np.arange(n)
    ea = np.tile((k // 110) * 600, n) + np.repeat(np.arange(n) % 5, n)
    eb = np.repeat(-(k // 110) * 600, n)
    a = gen.random_balls(rng, n * n, 128, exps=ea, rad_k=110, rad_frac=0.2, zero_frac=0.05)
    b = gen.random_balls(rng, n * n, 128, exps=eb, rad_k=110, rad_frac=0.2, zero_frac=0.05)
    A, B = _mat(a, n, n), _mat(b, n, n)
    plan = ops.plan_blocks(A, B, 128)
    assert sum(1 for r in plan if not r[2]) >= 2, plan
    got = ops.block_matmul_ball(A, B, 128).balls.to_host()
    ref, nb = po.matmul(a, b, n, n, n, 128, which="ref", algo=1, threads=os.cpu_count() or 8)
    ok = got.identical(ref)
    assert ok.all(), f"{(~ok).sum()} entries differ"
    lo, hi, _ = next(r for r in plan if not r[2])
    _, _, t8 = ops.block_int_product(A, B, lo, hi, 8)
    _, _, ti, _ = ops.block_int_product_imad(A, B, lo, hi, 8)
    np.testing.assert_array_equal(t8, ti)


@pytest.mark.parametrize("n,p", [(2048, 512), (1024, 1024)])
def test_band_normalised_high_precision(n, p):
    """BASELINE config 5 shapes where a diagonal could overflow int32 over the full K
    (pairs * K >= 2^17): the band GEMM with in-place accumulator normalisations equals
    the one-diagonal-at-a-time unit GEMM on every entry, and sampled rows equal the
    reference"""
    import subprocess
    import sys
    from paper_1901_04289_b200 import ops
    a, b = gen.config5_matrices(n=n, p=p)
    A, B = _mat(a, n, n), _mat(b, n, n)
    got = ops.block_matmul_ball(A, B, p).balls.to_host()
    rows = 2
    ref, _ = po.matmul(a.take(np.arange(rows * n)), b, rows, n, n, p, which="ref", algo=1,
                       threads=os.cpu_count() or 8)
    assert got.take(np.arange(rows * n)).identical(ref).all()
    # unit path in a subprocess on the same inputs: full-matrix equality
    code = ("import sys, numpy as np; sys.path[:0] = %r; from paper_1901_04289_b200 import gen, ops;"
            "a, b = gen.config5_matrices(n=%d, p=%d);"
            "A = ops.BallMatrix(a.to_device(), %d, %d); B = ops.BallMatrix(b.to_device(), %d, %d);"
            "c = ops.block_matmul_ball(A, B, %d).balls.to_host(); np.save(sys.argv[1], c.mant)"
            % (sys.path[:3], n, p, n, n, n, n, p))
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "unit.npy")
        env = dict(os.environ, APB_NO_BAND_NORM="1")
        r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        np.testing.assert_array_equal(np.load(f), got.mant)


def test_host_pipeline_matches_sync():
    """apb_matmul_host_submit/drain over three different products (pinned host
    buffers, alternating device buffer sets): every result equals the reference"""
    import ctypes as C
    from paper_1901_04289_b200 import ops
    from paper_1901_04289_b200.balls import BallArray, apb_mat, limbs_for
    lib = ops._lib.lib()
    n, p = 256, 128
    jobs = []
    for salt in range(3):
        a, b = gen.config2_matrices(seed_salt=salt)
        ha, hb = a.pinned(), b.pinned()
        hc = BallArray.zeros(n * n, limbs_for(p)).pinned()
        jobs.append((a, b, ha, hb, hc, apb_mat(ha.c(), n, n), apb_mat(hb.c(), n, n), apb_mat(hc.c(), n, n)))
    for _ in range(2):  # also reuse both buffer sets
        for j in jobs:
            ops._lib.check(lib.apb_matmul_host_submit(C.byref(j[5]), C.byref(j[6]), p, 1, C.byref(j[7])), "submit")
        ops._lib.check(lib.apb_matmul_host_drain(), "drain")
        for a, b, ha, hb, hc, *_ in jobs:
            ref, _ = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
            assert hc.identical(ref).all()


@pytest.mark.parametrize("shift", [700, -700, 0])
def test_radius_planes_far_exponents(shift):
    """single-block products whose operand exponents sit far from 1 (|e| ~ 700):
    the scan's uncentred radius planes are flagged unsafe on the device and the
    centred planes (src/matmul.cpp:386-403) take over; repeated calls (graph
    replays) stay bit-identical to the reference"""
    from paper_1901_04289_b200 import ops
    rng = np.random.default_rng(0xB200 + 700 + shift)
    n, p = 256, 128
    ea = shift + rng.integers(-4, 5, size=n * n)
    eb = -shift // 2 + rng.integers(-4, 5, size=n * n)
    a = gen.random_balls(rng, n * n, p, exps=ea, rad_k=130, rad_frac=0.3)
    b = gen.random_balls(rng, n * n, p, exps=eb, rad_k=130, rad_frac=0.3)
    A, B = _mat(a, n, n), _mat(b, n, n)
    ref, _ = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
    out = ops.block_matmul_ball(A, B, p)
    for rep in range(3):
        got = ops.block_matmul_ball(A, B, p, out=out).balls.to_host()
        ok = got.identical(ref)
        assert ok.all(), f"rep {rep}: {(~ok).sum()} entries differ"


def test_complex_c4_shape_vs_reference():
    """config 4 distributions (independent 512-bit parts, exponents in [-16, 16], radii
    2^-515|m|) at N=256: every entry of both parts bit-identical to complex_matmul_ball
    (reference run multithreaded on the host)"""
    from paper_1901_04289_b200 import ops
    n, p = 256, 512
    parts = gen.config4_matrices(n=n, p=p)
    M4 = [_mat(x, n, n) for x in parts]
    cre, cim = ops.complex_matmul_ball(*M4, p)
    rre, rim = po.matmul_complex(*parts, n, n, n, p, which="ref", threads=os.cpu_count() or 8)
    assert cre.balls.to_host().identical(rre).all()
    assert cim.balls.to_host().identical(rim).all()


def test_host_pipeline_growth_and_errors():
    """pipelined entry with operands that grow between submissions (the buffer
    sets reallocate while the worker thread holds earlier products), a
    dimension mismatch mid-stream (drain returns APB_ERR_INVALID with the
    library's message), and a clean stream afterwards"""
    import ctypes as C
    from paper_1901_04289_b200 import ops
    from paper_1901_04289_b200.balls import BallArray, apb_mat, limbs_for
    lib = ops._lib.lib()
    jobs = []
    for n, p, salt in [(64, 128, 0), (256, 128, 1), (128, 256, 2), (512, 256, 3)]:
        a, b = (gen.config2_matrices(n=n, p=p, seed_salt=salt) if p == 128
                else gen.config3_matrices(n=n, p=p, seed_salt=salt))
        ha, hb = a.pinned(), b.pinned()
        hc = BallArray.zeros(n * n, limbs_for(p)).pinned()
        jobs.append((n, p, a, b, ha, hb, hc, apb_mat(ha.c(), n, n), apb_mat(hb.c(), n, n), apb_mat(hc.c(), n, n)))
    for n, p, a, b, ha, hb, hc, am, bm, cm in jobs:
        ops._lib.check(lib.apb_matmul_host_submit(C.byref(am), C.byref(bm), p, 1, C.byref(cm)), "submit")
    ops._lib.check(lib.apb_matmul_host_drain(), "drain")
    for n, p, a, b, ha, hb, hc, *_ in jobs:
        ref, _ = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
        assert hc.identical(ref).all(), (n, p)
    # A (64 x 64) times B (128 x 128): invalid dimensions, reported by drain
    bad_c = BallArray.zeros(64 * 128, limbs_for(128)).pinned()
    bm_bad = jobs[2][8]
    cm_bad = apb_mat(bad_c.c(), 64, 128)
    assert lib.apb_matmul_host_submit(C.byref(jobs[0][7]), C.byref(bm_bad), 128, 1, C.byref(cm_bad)) == 0
    rc = lib.apb_matmul_host_drain()
    assert rc == 1, rc
    assert b"dimension" in lib.apb_last_error()
    # the pipeline recovers
    n, p, a, b, ha, hb, hc, am, bm, cm = jobs[1]
    ops._lib.check(lib.apb_matmul_host_submit(C.byref(am), C.byref(bm), p, 1, C.byref(cm)), "submit")
    ops._lib.check(lib.apb_matmul_host_drain(), "drain")
    ref, _ = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
    assert hc.identical(ref).all()


def test_host_pipeline_interleaved_with_other_entries():
    """other entry points called between submit and drain (same thread and a
    second thread) wait for the pipelined products (library API lock): every
    result is right, the stats see the pipelined products, and an error of a
    pipelined product is still reported by drain after an intervening call"""
    import ctypes as C
    import threading
    from paper_1901_04289_b200 import ops
    from paper_1901_04289_b200.balls import BallArray, apb_mat, limbs_for
    lib = ops._lib.lib()
    n, p = 256, 128
    a, b = gen.config2_matrices(n=n, p=p, seed_salt=7)
    ha, hb = a.pinned(), b.pinned()
    outs = [BallArray.zeros(n * n, limbs_for(p)).pinned() for _ in range(3)]
    am, bm = apb_mat(ha.c(), n, n), apb_mat(hb.c(), n, n)
    cms = [apb_mat(o.c(), n, n) for o in outs]
    ref, _ = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
    x, y = gen.config1_dots(batch=512)
    dref = po.dot_batch(x, y, 100, 512, 128, which="ref")
    errs = []

    def other_thread():
        try:
            for _ in range(3):
                got = ops.dot_batch(x.to_device(), y.to_device(), 100, 512, 128).to_host()
                assert got.identical(dref).all()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = threading.Thread(target=other_thread)
    th.start()
    for cm in cms:
        ops._lib.check(lib.apb_matmul_host_submit(C.byref(am), C.byref(bm), p, 1, C.byref(cm)), "submit")
    # same thread, before drain: a synchronous product and a dot batch
    dA, dB = _mat(a, n, n), _mat(b, n, n)
    assert ops.block_matmul_ball(dA, dB, p).balls.to_host().identical(ref).all()
    assert ops.dot_batch(x.to_device(), y.to_device(), 100, 512, 128).to_host().identical(dref).all()
    th.join()
    assert not errs, errs
    ops._lib.check(lib.apb_matmul_host_drain(), "drain")
    for o in outs:
        assert o.identical(ref).all()
    # a failing pipelined product, then another entry point, then drain: still reported
    bad_c = BallArray.zeros(n * 2 * n, limbs_for(p)).pinned()
    assert lib.apb_matmul_host_submit(C.byref(am), C.byref(bm), p, 1, C.byref(apb_mat(bad_c.c(), n, 2 * n))) == 0
    assert ops.dot_batch(x.to_device(), y.to_device(), 100, 512, 128).to_host().identical(dref).all()
    assert lib.apb_matmul_host_drain() == 1
