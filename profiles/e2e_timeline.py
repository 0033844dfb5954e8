"""Stage timeline of one end-to-end apb_matmul_host call (pinned host buffers,
H2D + kernels + D2H), from the library's event regions.
Usage: python profiles/e2e_timeline.py [c3|c2] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1901_04289_b200 import balls as bl, gen, ops  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    a, b = gen.config3_matrices() if which == "c3" else gen.config2_matrices()
    n, p = (512, 256) if which == "c3" else (256, 128)
    import ctypes as C
    lib = ops._lib.lib()
    ha, hb = a.pinned(), b.pinned()
    hc = bl.BallArray.zeros(n * n, bl.limbs_for(p)).pinned()
    am, bm, cm = bl.apb_mat(ha.c(), n, n), bl.apb_mat(hb.c(), n, n), bl.apb_mat(hc.c(), n, n)
    for r in range(reps + 2):
        lib.apb_profile_reset()
        lib.apb_profile_enable(1 if r >= 2 else 0)
        t0 = time.perf_counter()
        ops._lib.check(lib.apb_matmul_host(C.byref(am), C.byref(bm), p, 1, C.byref(cm)), "e2e")
        t1 = time.perf_counter()
        lib.apb_profile_enable(0)
        if r < 2:
            continue
        k = lib.apb_profile_dump(None, 0)
        buf = bytes(k + 1)
        lib.apb_profile_dump(buf, k + 1)
        print(f"rep {r - 2}: host wall {(t1 - t0) * 1e6:.0f} us")
        for line in buf.decode().strip("\x00").strip().splitlines():
            name, b_, e_ = line.split("\t")
            print(f"   {name:12s} {float(b_) * 1e3:8.1f} .. {float(e_) * 1e3:8.1f} us  ({(float(e_) - float(b_)) * 1e3:7.1f})")


if __name__ == "__main__":
    main()
