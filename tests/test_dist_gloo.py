"""CPU, world_size 2 over gloo: the row-block sharded matmul driver
(paper_1901_04289_b200/dist.py) -- scatter A row blocks, broadcast B, plan
agreement, gather C -- returns exactly the single-call product.  The local
compute here is the oracle port (tests only); on the GPU box it is the CUDA
block matmul (tests/test_dist_gpu.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mag_f_upper(mant_top, exp):
    b = (mant_top >> np.uint64(34)) + np.uint64(1)
    return np.where(b == np.uint64(1 << 30), exp + 1, exp)


def _plan_info_port(a, b, r, k, n, p):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    from paper_1901_04289_b200.dist import PlanInfo
    steps = po.plan_blocks(a, b, r, k, n, p, which="port")
    # radius windows (f, f-30) of |A|, R_A rows and R_B, |B|+R_B columns with one bit of slack
    def width(f, valid, axis):
        top = np.where(valid, f, -(1 << 62)).max(axis=axis)
        bot = np.where(valid, f - 30, 1 << 62).min(axis=axis)
        return np.where(top > -(1 << 62), top - bot, 0).max() + 1
    fin_a = (a.kind & 7) == 1
    fa = _mag_f_upper(a.mant[:, -1], a.exp).reshape(r, k)
    ra = a.rad_exp.reshape(r, k)
    fb = _mag_f_upper(b.mant[:, -1], b.exp).reshape(k, n)
    rb = b.rad_exp.reshape(k, n)
    w = max(width(fa, fin_a.reshape(r, k), 1), width(ra, (a.rad_man != 0).reshape(r, k), 1),
            width(rb, (b.rad_man != 0).reshape(k, n), 0),
            width(np.maximum(fb, rb) + 1, ((b.kind & 7) == 1).reshape(k, n) | (b.rad_man != 0).reshape(k, n), 0))
    return PlanInfo(blocks=len(steps), radius_single=w <= 900)


def _compute_port(a, b, r, k, n, p):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    c, _ = po.matmul(a, b, r, k, n, p, which="port", algo=1)
    return c


def _worker(rank, world, port, case, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1901_04289_b200 import dist as pdist
        a, b, M, K, N, p = _case(case)
        c = pdist.sharded_matmul(a if rank == 0 else None, b if rank == 0 else None, M, K, N, p,
                                 device="cpu", compute=_compute_port, plan_info=_plan_info_port)
        if rank == 0:
            q.put((c.mant, c.exp, c.kind, c.rad_man, c.rad_exp))
    finally:
        dist.destroy_process_group()


def _case(case):
    from paper_1901_04289_b200 import gen
    if case == "c3_small":
        a, b = gen.config3_matrices(n=40)
        return a, b, 40, 40, 40, 256
    if case == "c2_rect":
        rng = np.random.Generator(np.random.PCG64(11))
        a = gen.random_balls(rng, 37 * 33, 128, e_lo=-4, e_hi=4, rad_k=130)
        b = gen.random_balls(rng, 33 * 35, 128, e_lo=-4, e_hi=4, rad_k=130)
        return a, b, 37, 33, 35, 128
    if case == "multiblock":  # only row 0 forces a split: the local plans disagree -> fallback
        rng = np.random.Generator(np.random.PCG64(12))
        n = 64
        ea = np.zeros((n, n), np.int64)
        ea[0, 32:] = 5000
        a = gen.random_balls(rng, n * n, 128, exps=ea.ravel(), rad_k=120, rad_frac=0.3)
        b = gen.random_balls(rng, n * n, 128, e_lo=-3, e_hi=3, rad_k=120, rad_frac=0.3)
        return a, b, n, n, n, 128
    raise ValueError(case)


@pytest.mark.parametrize("case", ["c3_small", "c2_rect", "multiblock"])
def test_sharded_matmul_gloo(case):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    from paper_1901_04289_b200.balls import BallArray
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    a, b, M, K, N, prec = _case(case)
    ref, _ = po.matmul(a, b, M, K, N, prec, which="port", algo=1)
    assert BallArray(*got).identical(ref).all()


def test_row_ranges_cover():
    from paper_1901_04289_b200.dist import row_range
    for M in (1, 7, 512, 1000):
        for W in (1, 2, 3, 8):
            cov = []
            for r in range(W):
                lo, hi, per = row_range(M, W, r)
                assert hi - lo <= per
                cov += list(range(lo, hi))
            assert cov == list(range(M))
