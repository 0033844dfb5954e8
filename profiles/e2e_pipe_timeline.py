"""CUPTI timeline (torch.profiler) of the pipelined host entry
(apb_matmul_host_submit/drain) on config 3: every memcpy and kernel of a few
consecutive steps with start offset, duration and stream, to see how the
copy-in, compute and copy-out of neighbouring steps overlap.
Usage: python profiles/e2e_pipe_timeline.py [steps]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1901_04289_b200 import gen, ops  # noqa: E402
from paper_1901_04289_b200.balls import BallArray, apb_mat, limbs_for  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    a, b = gen.config3_matrices()
    n, p = 512, 256
    lib = ops._lib.lib()
    ha, hb = a.pinned(), b.pinned()
    hc = BallArray.zeros(n * n, limbs_for(p)).pinned()
    am, bm, cm = apb_mat(ha.c(), n, n), apb_mat(hb.c(), n, n), apb_mat(hc.c(), n, n)
    for _ in range(4):
        ops._lib.check(lib.apb_matmul_host_submit(C.byref(am), C.byref(bm), p, 1, C.byref(cm)), "warmup")
    ops._lib.check(lib.apb_matmul_host_drain(), "warmup")
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            ops._lib.check(lib.apb_matmul_host_submit(C.byref(am), C.byref(bm), p, 1, C.byref(cm)), "e2e")
        ops._lib.check(lib.apb_matmul_host_drain(), "drain")
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    span = ev[-1].time_range.end - t0
    print(f"{steps} pipelined steps: device span {span:.1f} us = {span / steps:.1f} us/step")
    # merge consecutive memcpys per stream into one segment for readability
    segs = []
    for e in ev:
        name = e.name
        kind = "H2D" if "HtoD" in name else ("D2H" if "DtoH" in name else ("memset" if "Memset" in name else "kernel"))
        s, d = e.time_range.start - t0, e.time_range.end - t0
        st = getattr(e, "device_resource_id", None)
        if segs and segs[-1][0] == kind and segs[-1][3] == st and kind != "kernel" and s - segs[-1][2] < 5:
            segs[-1][2] = d
            segs[-1][4] += 1
        else:
            segs.append([kind, s, d, st, 1, name[:40]])
    for k, s, d, st, cnt, name in segs:
        if k == "kernel":
            print(f"  {s:9.1f} {d - s:8.1f} us  stream {st}  {name}")
        else:
            print(f"  {s:9.1f} {d - s:8.1f} us  stream {st}  {k} x{cnt}")


if __name__ == "__main__":
    main()
