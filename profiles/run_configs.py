"""Timing + sampled-row parity for BASELINE configs 4 and 5 (GPU).
Row samples of the product are checked bit for bit against the reference
(oracle/_ref) run on the same rows of A (bit-identical for single-block plans)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import pyoracle as po  # noqa: E402
from paper_1901_04289_b200 import gen, ops  # noqa: E402


def timed(f, reps=2):
    f()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        r = f()
        e.record()
        torch.cuda.synchronize()
        t.append(s.elapsed_time(e))
    return r, min(t)


def rows_of(a, n, rows):
    return a.take(np.arange(rows * n))


def main():
    which = sys.argv[1:] or ["c4", "c5"]
    out = {}
    T = os.cpu_count() or 8
    if "c4" in which:
        n, p = 1024, 512
        are, aim, bre, bim = gen.config4_matrices()
        M = [ops.BallMatrix(x.to_device(), n, n) for x in (are, aim, bre, bim)]
        (cre, cim), ms = timed(lambda: ops.complex_matmul_ball(*M, p))
        rows = 8
        rre, rim = po.matmul_complex_rows(are, aim, bre, bim, rows, n, n, p, threads=T)
        ok = cre.balls.to_host().take(np.arange(rows * n)).identical(rre).all() and \
            cim.balls.to_host().take(np.arange(rows * n)).identical(rim).all()
        out["c4"] = {"ms": ms, "complex_terms_per_s": n ** 3 / (ms * 1e-3), "rows_checked": rows, "bit_identical": bool(ok),
                     "stats": ops.matmul_stats()}
        print(json.dumps({"c4": out["c4"]}), flush=True)
    if "c5" in which:
        for p in (64, 128, 256, 512, 1024, 4096):
            n = 2048
            a, b = gen.config5_matrices(n=n, p=p)
            A, B = ops.BallMatrix(a.to_device(), n, n), ops.BallMatrix(b.to_device(), n, n)
            ops.matmul_stats_reset()
            lib = ops._lib.lib()
            lib.apb_profile_reset()
            lib.apb_profile_enable(1)
            c, ms = timed(lambda: ops.block_matmul_ball(A, B, p), reps=1)
            lib.apb_profile_enable(0)
            import ctypes as C
            kms = {}
            for k in ("slice_gemm", "pack", "recombine", "rad_gemm"):
                t, cnt = C.c_double(0), C.c_uint64(0)
                lib.apb_profile_read(k.encode(), C.byref(t), C.byref(cnt))
                kms[k] = t.value / max(cnt.value, 1)
            st = ops.matmul_stats()
            res = {"ms": ms, "terms_per_s": n ** 3 / (ms * 1e-3), "kernel_ms": kms, "stats": st}
            if p <= 1024:
                rows = 4
                ref, _ = po.matmul(rows_of(a, n, rows), b, rows, n, n, p, which="ref", algo=1, threads=T)
                res["rows_checked"] = rows
                res["bit_identical"] = bool(c.balls.to_host().take(np.arange(rows * n)).identical(ref).all())
            out[f"c5_p{p}"] = res
            print(json.dumps({f"c5_p{p}": res}), flush=True)
            del A, B, c
            torch.cuda.empty_cache()
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "configs.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
