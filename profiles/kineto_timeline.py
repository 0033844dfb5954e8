"""Device timeline of block_matmul_ball steps from CUPTI (torch.profiler):
every kernel / memcpy of the last profiled step with its start offset, duration
and stream, including kernels replayed from the library's CUDA graphs.
Usage: python profiles/kineto_timeline.py [c3|c2|c4] [steps]"""
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1901_04289_b200 import gen, ops  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if which == "c3":
    a, b = gen.config3_matrices()
    n, p = 512, 256
elif which == "c2":
    a, b = gen.config2_matrices()
    n, p = 256, 128
else:
    parts = gen.config4_matrices(n=1024)
    n, p = 1024, 512
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
if which == "c4":  # complex product: four real block products + ball_sub / ball_add
    Ms = [ops.BallMatrix(x.to_device(), n, n) for x in parts]

    def step():
        ops.complex_matmul_ball(*Ms, p)
else:
    A, B = ops.BallMatrix(a.to_device(), n, n), ops.BallMatrix(b.to_device(), n, n)
    out = ops.block_matmul_ball(A, B, p)

    def step():
        ops.block_matmul_ball(A, B, p, out=out)
for _ in range(3):
    step()
torch.cuda.synchronize()
marks = []
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for s in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        step()
        torch.cuda.synchronize()
path = os.path.join(tempfile.gettempdir(), "apb_trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
# split into steps at the flush kernels (fill/zero kernels of torch)
steps_ev, cur = [], []
for e in gpu:
    if "elementwise" in e["name"] or "fill" in e["name"].lower():
        if cur:
            steps_ev.append(cur)
        cur = []
        continue
    cur.append(e)
if cur:
    steps_ev.append(cur)
last = steps_ev[-1]
t0 = last[0]["ts"]
end = max(e["ts"] + e["dur"] for e in last)
print(f"{which}: step span {end - t0:.1f} us, {len(last)} device ops")
for e in last:
    nm = e["name"]
    nm = nm.replace("(anonymous namespace)::", "").replace("void ", "").replace("apb::", "").split("(")[0][:60]
    print(f"  +{e['ts'] - t0:8.1f}  {e['dur']:7.1f} us  stream {e['args'].get('stream', '?'):>3}  {nm}")
