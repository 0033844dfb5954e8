"""Per-stage device timeline of one block_matmul_ball step (both streams),
from the library's event regions (apb_profile_dump).  Also reports the host
time of the call.  Usage: python profiles/timeline.py [c3|c2] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1901_04289_b200 import gen, ops  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    prof = os.environ.get("TIMELINE_NOPROF") is None  # host-trace-only mode keeps launches lean
    if which == "c3":
        a, b = gen.config3_matrices()
        n, p = 512, 256
    else:
        a, b = gen.config2_matrices()
        n, p = 256, 128
    A, B = ops.BallMatrix(a.to_device(), n, n), ops.BallMatrix(b.to_device(), n, n)
    lib = ops._lib.lib()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ops.block_matmul_ball(A, B, p)
    torch.cuda.synchronize()
    for r in range(reps):
        flush.fill_(1)
        torch.cuda.synchronize()
        lib.apb_profile_reset()
        lib.apb_profile_enable(1 if prof else 0)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        t0 = time.perf_counter()
        ops.block_matmul_ball(A, B, p, check=False)
        t1 = time.perf_counter()
        e1.record(st)
        torch.cuda.synchronize()
        lib.apb_profile_enable(0)
        n_ = lib.apb_profile_dump(None, 0)
        buf = bytes(n_ + 1)
        lib.apb_profile_dump(buf, n_ + 1)
        print(f"rep {r}: step {e0.elapsed_time(e1) * 1e3:.1f} us, host call {(t1 - t0) * 1e6:.1f} us")
        for line in buf.decode().strip("\x00").strip().splitlines():
            name, b_, e_ = line.split("\t")
            print(f"   {name:12s} {float(b_) * 1e3:8.1f} .. {float(e_) * 1e3:8.1f} us  ({(float(e_) - float(b_)) * 1e3:7.1f})")


if __name__ == "__main__":
    main()
