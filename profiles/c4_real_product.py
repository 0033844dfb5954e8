import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1901_04289_b200 import gen, ops
parts = gen.config4_matrices(n=1024)
A, B = ops.BallMatrix(parts[0].to_device(), 1024, 1024), ops.BallMatrix(parts[2].to_device(), 1024, 1024)
out = ops.block_matmul_ball(A, B, 512)
for _ in range(3):
    ops.block_matmul_ball(A, B, 512, out=out)
torch.cuda.synchronize()
print("ok")
