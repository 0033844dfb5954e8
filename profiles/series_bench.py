"""series_exp_basecase on the GPU (one warp; the recurrence is sequential, each
step's dot is spread over the lanes) vs the one-thread device version
(APB_SERIES_SERIAL=1, run as a subprocess) and the reference CPU implementation.
Usage: python profiles/series_bench.py [len] [prec]"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import pyoracle as po  # noqa: E402
from paper_1901_04289_b200 import gen, ops  # noqa: E402

ln = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = int(sys.argv[2]) if len(sys.argv) > 2 else 128
rng = np.random.Generator(np.random.PCG64(512))
a, _ = gen.edge_dots(rng, 1, ln, specials=False)
a.kind[0], a.mant[0], a.exp[0], a.rad_man[0], a.rad_exp[0] = 0, 0, 0, 0, 0
ops.series_exp_basecase(a, ln, p)
torch.cuda.synchronize()
t0 = time.perf_counter()
got = ops.series_exp_basecase(a, ln, p)
torch.cuda.synchronize()
gpu_s = time.perf_counter() - t0
t0 = time.perf_counter()
ref = po.series_exp(a, ln, p)
cpu_s = time.perf_counter() - t0
res = {"op": "series_exp_basecase", "len": ln, "prec": p, "terms": ln * (ln - 1) // 2, "gpu_warp_s": gpu_s,
       "cpu_ref_s": cpu_s, "bit_identical": bool(got.identical(ref).all()),
       "mode": os.environ.get("APB_SERIES_SERIAL") and "serial" or "warp"}
print(json.dumps(res), flush=True)
if not os.environ.get("APB_SERIES_SERIAL"):
    subprocess.run([sys.executable, __file__, str(ln), str(p)], env=dict(os.environ, APB_SERIES_SERIAL="1"))
