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
    torch.cuda.synchronize()
    print("prof_run ok", which, reps)


if __name__ == "__main__":
    main()
