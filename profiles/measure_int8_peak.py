"""Measure the dense INT8 tensor peak of this B200 (the roofline denominator for
the slice GEMM; MEASURED_PEAKS.json only holds bf16 and HBM): cuBLASLt
s8 x s8 -> s32 via torch._int_mm at 8192^3, best of 10 with CUDA events, plus
a 4-second back-to-back (sustained) figure.  Writes profiles/int8_peak.json."""
import json
import os
import time

import torch

n = 8192
a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    torch._int_mm(a, b)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
ops = 2.0 * n ** 3
burst = ops / (best * 1e-3) / 1e12
t0 = time.time()
cnt = 0
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
s.record()
while time.time() - t0 < 4.0:
    for _ in range(10):
        torch._int_mm(a, b)
    cnt += 10
    torch.cuda.synchronize()
e.record()
torch.cuda.synchronize()
sustained = ops * cnt / (s.elapsed_time(e) * 1e-3) / 1e12
out = {"int8_tops": burst, "int8_tops_sustained": sustained,
       "how": "torch._int_mm (cuBLASLt s8s8s32) 8192^3: best of 10 (burst) and 4 s back to back (sustained)",
       "gpu": torch.cuda.get_device_name()}
print(json.dumps(out))
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "int8_peak.json"), "w"), indent=1)
