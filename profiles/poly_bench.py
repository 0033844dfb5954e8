"""Measurement of the poly consumer row: poly_mullow_classical
on the GPU (device-resident operands, one batched launch of variable-length
dots, CUDA events) against the reference's single-threaded CPU implementation
(oracle/_ref) on the same seeded inputs.  Terms = sum_k n_k multiply-adds.
Usage: python profiles/poly_bench.py [len] [prec]"""
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


def main():
    ln = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    rng = np.random.Generator(np.random.PCG64(1024))
    a, _ = gen.edge_dots(rng, 1, ln, specials=False)
    b, _ = gen.edge_dots(rng, 1, ln, specials=False)
    terms = ln * (ln + 1) // 2
    da, db = a.to_device(), b.to_device()
    for _ in range(3):
        ops.poly_mullow_classical(da, db, ln, p)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        got = ops.poly_mullow_classical(da, db, ln, p, check=False)
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1) / reps
    t0 = time.perf_counter()
    ref = po.poly_mullow(a, b, ln, p)
    cpu_s = time.perf_counter() - t0
    same = bool(got.to_host().take(range(ln)).identical(ref).all())
    print(json.dumps({"op": "poly_mullow_classical", "len": ln, "prec": p, "terms": terms,
                      "gpu_ms": gpu_ms, "gpu_terms_per_s": terms / (gpu_ms * 1e-3),
                      "cpu_ref_s": cpu_s, "cpu_ref_terms_per_s": terms / cpu_s, "cpu_threads": 1,
                      "bit_identical": same}))


if __name__ == "__main__":
    main()
