"""Small driver for ncu captures: runs config 1 (dots) and config 3 (matmul)
a few times on cuda:0.  Usage: python profiles/prof_run.py [c1|c3|c2|all] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1901_04289_b200 import gen, ops  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    if which in ("c1", "all"):
        x, y = gen.config1_dots()
        dx, dy = x.to_device(), y.to_device()
        for _ in range(reps):
            ops.dot_batch(dx, dy, 100, 65536, 128)
    if which in ("c3", "all"):
        a, b = gen.config3_matrices()
        A, B = ops.BallMatrix(a.to_device(), 512, 512), ops.BallMatrix(b.to_device(), 512, 512)
        for _ in range(reps):
            ops.block_matmul_ball(A, B, 256)
    if which in ("c2", "all"):
        a, b = gen.config2_matrices()
        A, B = ops.BallMatrix(a.to_device(), 256, 256), ops.BallMatrix(b.to_device(), 256, 256)
        for _ in range(reps):
            ops.block_matmul_ball(A, B, 128)
    if which in ("c5d", "all"):  # wide-precision dots (warp per dot)
        for p in (1024, 4096):
            x, y = gen.config5_dots(batch=2048, p=p)
            dx, dy = x.to_device(), y.to_device()
            for _ in range(reps):
                ops.dot_batch(dx, dy, 1000, 2048, p)
    if which in ("c5m", "all"):  # slice GEMM (unit path) at p = 512, N = 1024
        a, b = gen.config5_matrices(n=1024, p=512)
        A, B = ops.BallMatrix(a.to_device(), 1024, 1024), ops.BallMatrix(b.to_device(), 1024, 1024)
        for _ in range(reps):
            ops.block_matmul_ball(A, B, 512)
    if which in ("imad", "all"):  # IMAD-limb baseline product at N = 512, p = 128
        a, b = gen.config5_matrices(n=512, p=128)
        A, B = ops.BallMatrix(a.to_device(), 512, 512), ops.BallMatrix(b.to_device(), 512, 512)
        for _ in range(reps):
            ops.block_int_product_imad(A, B, 0, 512, 6)
    if which in ("c5m64", "all"):  # dense radius products + band GEMM at N = 2048, p = 64
        a, b = gen.config5_matrices(n=2048, p=64)
        A, B = ops.BallMatrix(a.to_device(), 2048, 2048), ops.BallMatrix(b.to_device(), 2048, 2048)
        for _ in range(reps):
            ops.block_matmul_ball(A, B, 64)
    if which in ("c5ds", "all"):  # dot_small_kernel: 8192 dots of N = 1000 at p = 256
        x, y = gen.config5_dots(p=256)
        dx, dy = x.to_device(), y.to_device()
        for _ in range(reps):
            ops.dot_batch(dx, dy, 1000, 8192, 256)
    torch.cuda.synchronize()
    print("prof_run ok", which, reps)


if __name__ == "__main__":
    main()
