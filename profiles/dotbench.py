"""Dot kernel timing on config 1 (65,536 x N=100, p=128) and the config-5 dot
sweep (8192 x N=1000), CUDA events over 10 launches, L2 not flushed (inputs
419 MB > L2 at c1).  Usage: python profiles/dotbench.py [c1|c5|all]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1901_04289_b200 import gen, ops  # noqa: E402
from paper_1901_04289_b200.balls import DeviceBallArray  # noqa: E402


def run(x, y, n, batch, p, L, reps=10):
    dx, dy = x.to_device(), y.to_device()
    out = DeviceBallArray.empty(batch, L)
    for _ in range(3):
        ops.dot_batch(dx, dy, n, batch, p, out=out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps):
        ops.dot_batch(dx, dy, n, batch, p, out=out, check=False)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    L_in = x.L
    gbs = batch * n * 2 * (8 * L_in + 21) / ms / 1e6
    return {"ms": ms, "terms_per_s": batch * n / ms * 1e3, "GB/s": gbs}


which = sys.argv[1] if len(sys.argv) > 1 else "all"
tag = os.environ.get("APB_DOT_TPD", "auto")
if which in ("c1", "all"):
    x, y = gen.config1_dots()
    print(json.dumps({"c1": run(x, y, 100, 65536, 128, 2), "tpd": tag}), flush=True)
if which in ("c5", "all"):
    for p in (64, 128, 256, 512, 1024, 4096):
        x, y = gen.config5_dots(p=p)
        r = run(x, y, 1000, 8192, p, max(1, p // 64), reps=3 if p >= 1024 else 10)
        print(json.dumps({"c5_dot_p%d" % p: r, "tpd": tag}), flush=True)
