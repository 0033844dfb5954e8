"""e2e (host buffers) timing of config 3 alone: the pipelined and the synchronous host entry,
several repetitions.  Usage: python profiles/e2e_only.py [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402,F401

import bench  # noqa: E402
from paper_1901_04289_b200 import gen, ops  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
a, b = gen.config3_matrices()
for r in range(reps):
    e = bench.e2e_matmul(ops, a, b, 512, 256, 40)
    print(f"rep {r}: pipelined {e['ms_per_step']:.4f} ms/step, sync {e['sync_call']['ms_per_step']:.4f} ms/step", flush=True)
