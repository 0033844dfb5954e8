"""int8-slice (tcgen05) vs IMAD-limb (CUDA cores) exact block product, per
precision (BASELINE config 5 distributions: p-bit mantissas, exponents in
[-32, 32], radii 2^-(p+2)|m|), at N = 512 and 1024 (the IMAD kernel is too slow
for N = 2048 sweeps).  Both produce the same exact integer (checked).  Reports
the product-kernel time of each and the ratio.  Usage: python profiles/imad_crossover.py"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1901_04289_b200 import gen, ops  # noqa: E402

lib = ops._lib.lib()
rows = []
for n in (512, 1024):
    for p in (64, 128, 256, 512):
        a, b = gen.config5_matrices(n=n, p=p)
        A, B = ops.BallMatrix(a.to_device(), n, n), ops.BallMatrix(b.to_device(), n, n)
        limbs = (2 * (p + 64) + 64) // 64 + 2
        # tensor-core product: median of 5 launches, time from the library's event regions
        lib.apb_profile_reset()
        lib.apb_profile_enable(1)
        for _ in range(5):
            rs, cs, t8 = ops.block_int_product(A, B, 0, n, limbs)
        lib.apb_profile_enable(0)
        t, cnt = C.c_double(0), C.c_uint64(0)
        lib.apb_profile_read(b"slice_gemm", C.byref(t), C.byref(cnt))
        ms8 = t.value / max(cnt.value, 1)
        best = None
        for _ in range(3):
            _, _, ti, ms = ops.block_int_product_imad(A, B, 0, n, limbs)
            best = ms if best is None else min(best, ms)
        ok = bool(np.array_equal(t8, ti))
        st = ops.matmul_stats()
        r = {"n": n, "p": p, "height_bits": st.get("last_height_a"), "slices": st.get("last_slices_a"),
             "int8_gemm_ms": round(ms8, 4), "imad_gemm_ms": round(best, 4), "imad_over_int8": round(best / ms8, 2),
             "int8_terms_per_s": n ** 3 / (ms8 * 1e-3), "imad_terms_per_s": n ** 3 / (best * 1e-3), "identical": ok}
        print(json.dumps(r), flush=True)
        rows.append(r)
        del A, B
        torch.cuda.empty_cache()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(rows, open(os.path.join(ROOT, "gpurun_out", "imad_crossover.json"), "w"), indent=1)
