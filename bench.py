#!/usr/bin/env python
"""bench.py - B200 ball matmul / ball dot throughput (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c1|c4|c5]
                    [--impl ours|reference]

Headline workload (N=1): config 3 of BASELINE.json -- the badly scaled real
ball matmul N=512, p=256, on which the north-star's "% of int8 tensor peak"
target is stated.  One step = one block_matmul_ball (plan, scale/pack, tcgen05
slice GEMM, recombine, radius) on device-resident inputs; the L2 is flushed
(256 MiB write) before every step, outside the timed events.  The same JSON
line carries configs 1, 2 and 4 under "also".

--gpus N (launched by torchrun): weak scaling, one process per GPU; every rank
multiplies its own row block A_r (512 x 512, seed salted by rank) by the
shared B (same seed on every rank, so there is no data-path collective);
value = all ranks' terms / max-over-ranks time.

--impl reference: the reference CPU implementation (oracle/_ref, the unmodified
apball library built from its sources) on the same config with all host threads,
each step a bounded row sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

INT8_PEAK_FILE = os.path.join(ROOT, "profiles", "int8_peak.json")
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every ~2 ms through NVML
    while the timed region runs (the nvidia-smi clocks line of B200_PROFILING.md,
    at a rate that still sees a millisecond-scale timed region)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            dev_index = self.index
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    dev_index = int(vis.split(",")[self.index])
                except ValueError:
                    pass
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.N = None
        return self

    def _run(self):
        N = self.N
        names = {N.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 N.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwPowerCap: "sw_power_cap"}
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if getattr(self, "N", None):
            self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "NVML, 2 ms"}


# --------------------------------------------------------------- helpers

def int8_peak():
    """the larger of the measured int8 ceilings: cuBLASLt s8 GEMM and the raw
    tcgen05 issue-rate microbenchmark (the conservative denominator)"""
    try:
        d = json.load(open(INT8_PEAK_FILE))
        cands = [(d["int8_tops"], d.get("how", "measured"))]
        if "tcgen05_ss_tops" in d:
            cands.append((d["tcgen05_ss_tops"], d.get("tcgen05_how", "tcgen05 microbenchmark")))
        return max(cands)
    except Exception:  # noqa: BLE001
        return 4500.0, "datasheet dense INT8 4.5 POPS (no measurement found)"


def hbm_peak():
    try:
        return json.load(open(PEAKS_FILE))["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback B200_PROFILING.md 6.65 TB/s"


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu capture, if any"""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(kernel)
    except Exception:  # noqa: BLE001
        return None


class L2Flush:
    def __init__(self, torch, nbytes=256 << 20):
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")

    def __call__(self):
        self.buf.fill_(1)


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------ workloads

L2_NOTE = ("GPU arm: L2 flushed before every step (256 MiB write, outside the timed events); "
           "reference arm: host-resident inputs on the CPU")


def gemm_kernel_name(lib):
    """the band GEMM instantiation of the last product (apb_gemm_last_config)"""
    import ctypes as C
    v = [C.c_int(0) for _ in range(4)]
    lib.apb_gemm_last_config(*[C.byref(x) for x in v])
    tn, bw, raw, ks = [x.value for x in v]
    name = f"band3_gemm_kernel<{tn},{bw}>"
    if raw:
        name += " raw-accumulator epilogue"
    if ks > 1:
        name += f", K split {ks}"
    return name


def matmul_config(cfg, n, p, world):
    """the `config` object of both arms (identical, so the driver can pair them)"""
    return {"workload": f"BASELINE config {cfg[1:]}: real ball matmul N={n}, p={p}",
            "M": n, "N": n, "K": n, "prec": p, "l2": L2_NOTE,
            "parallelism": f"row-block weak scaling x{world}"}


def dots_config(batch, n, p, world):
    return {"workload": f"BASELINE config 1: {batch:,} real ball dots, N={n}, p={p}",
            "batch": batch, "n": n, "prec": p, "l2": L2_NOTE,
            "parallelism": f"batch weak scaling x{world}"}


def matmul_workload(cfg, rank, p_override=None):
    from paper_1901_04289_b200 import gen
    if cfg == "c2":
        n, p = 256, 128
        a, _ = gen.config2_matrices(n=n, seed_salt=rank)
        _, b = gen.config2_matrices(n=n, seed_salt=0)
    elif cfg == "c3":
        n, p = 512, 256
        a, _ = gen.config3_matrices(n=n, seed_salt=rank)
        _, b = gen.config3_matrices(n=n, seed_salt=0)
    elif cfg == "c5":
        p = p_override or 128
        n = 2048
        a, _ = gen.config5_matrices(n=n, p=p, seed_salt=rank)
        _, b = gen.config5_matrices(n=n, p=p, seed_salt=0)
    else:
        raise ValueError(cfg)
    return a, b, n, p


def run_matmul(torch, cfg, steps, warmup, world, rank, want_e2e=True, want_cpu=True, p_override=None):
    from paper_1901_04289_b200 import ops
    lib = ops._lib.lib()
    a, b, n, p = matmul_workload(cfg, rank, p_override)
    A = ops.BallMatrix(a.to_device(), n, n)
    B = ops.BallMatrix(b.to_device(), n, n)
    flush = L2Flush(torch)
    st = torch.cuda.current_stream()
    import ctypes as C
    out = ops.block_matmul_ball(A, B, p)  # persistent output: steps replay the library's CUDA graphs
    for _ in range(warmup):
        ops.block_matmul_ball(A, B, p, out=out)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = ops.launch_count()
    lib.apb_gemm_timer_reset()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for k in range(steps):
            flush()
            ev[k][0].record(st)
            ops.block_matmul_ball(A, B, p, check=False, out=out)
            ev[k][1].record(st)
        torch.cuda.synchronize()
    launches = ops.launch_count() - launches0
    # dominant kernel: the tcgen05 band GEMM, timed on the device inside the timed
    # region by its own span timer (first CTA start to last CTA end, %globaltimer)
    gns, gl = C.c_uint64(0), C.c_uint64(0)
    lib.apb_gemm_timer_read(C.byref(gns), C.byref(gl))
    if world > 1:
        torch.distributed.barrier()
    step_ms = [s.elapsed_time(e) for s, e in ev]
    ms = sum(step_ms) / steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    status = lib.apb_device_status(st.cuda_stream)
    if status:
        raise RuntimeError(f"device status {status}: {lib.apb_last_error().decode()}")
    stats = ops.matmul_stats()
    terms = float(n) ** 3
    value = world * terms / (ms * 1e-3)
    per_launch_ms = gns.value / max(gl.value, 1) / 1e6
    ha, hb = stats["last_height_a"], stats["last_height_b"]
    credited_ops = 2.0 * n * n * n * ((ha + 7) // 8) * ((hb + 7) // 8)
    achieved = credited_ops / (per_launch_ms * 1e-3) / 1e12
    peak, peak_src = int8_peak()
    # per-stage breakdown from a separate short pass with per-kernel event regions
    # (eager launches: the event registry is not captured into graphs)
    lib.apb_profile_reset()
    lib.apb_profile_enable(1)
    nprof = min(steps, 5)
    for _ in range(nprof):
        flush()
        ops.block_matmul_ball(A, B, p, check=False, out=out)
    torch.cuda.synchronize()
    lib.apb_profile_enable(0)
    other = {}
    for kname in ("scan", "pack", "slice_gemm", "recombine", "rad_gemm", "radius", "combine"):
        t, c = C.c_double(0), C.c_uint64(0)
        lib.apb_profile_read(kname.encode(), C.byref(t), C.byref(c))
        if c.value:
            other[kname] = round(t.value / nprof, 5)
    lib.apb_profile_reset()
    res = {
        "metric": "ball matmul terms/s (N^3 multiply-adds of p-bit balls per second)",
        "value": value, "unit": "terms/s", "ms_per_step": ms,
        "config": matmul_config(cfg, n, p, world),
        "plan": {"blocks": stats["last_block_count"], "height_a": ha, "height_b": hb,
                 "slices_a": stats["last_slices_a"], "slices_b": stats["last_slices_b"]},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS (int8)",
                     "frac": achieved / peak, "traffic": ncu_traffic("band3_gemm"),
                     "kernel": gemm_kernel_name(lib), "kernel_ms": per_launch_ms,
                     "kernel_launches_timed": gl.value,
                     "timing": "device span timer (%globaltimer) over the timed steps",
                     "work": f"2*M*N*K*ceil(h_A/8)*ceil(h_B/8) = {credited_ops:.4g} int8 ops per launch",
                     "peak_source": peak_src},
        "stage_ms_profiled_pass": other,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if want_e2e and rank == 0:
        res["e2e"] = e2e_matmul(ops, a, b, n, p, steps)
    if want_cpu and rank == 0 and world == 1:
        res["cpu_baseline"] = cpu_matmul(a, b, n, p)
    return res


def run_complex(torch, steps, warmup):
    """BASELINE config 4: complex ball matmul N=1024, p=512 (4 real block products,
    ball_sub / ball_add), device-resident operands, L2 flushed before every step"""
    import ctypes as C
    from paper_1901_04289_b200 import gen, ops
    lib = ops._lib.lib()
    n, p = 1024, 512
    parts = gen.config4_matrices(n=n, p=p)
    M = [ops.BallMatrix(x.to_device(), n, n) for x in parts]
    flush = L2Flush(torch)
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        ops.complex_matmul_ball(*M, p)
    torch.cuda.synchronize()
    lib.apb_gemm_timer_reset()
    ms_all = []
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(steps):
            flush()
            s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(st)
            ops.complex_matmul_ball(*M, p, check=False)
            e0.record(st)
            torch.cuda.synchronize()
            ms_all.append(s0.elapsed_time(e0))
    gns, gl = C.c_uint64(0), C.c_uint64(0)
    lib.apb_gemm_timer_read(C.byref(gns), C.byref(gl))
    ms = sum(ms_all) / steps
    stats = ops.matmul_stats()
    ha, hb = stats["last_height_a"], stats["last_height_b"]
    credited = 2.0 * n ** 3 * ((ha + 7) // 8) * ((hb + 7) // 8)
    per_launch_ms = gns.value / max(gl.value, 1) / 1e6
    achieved = credited / (per_launch_ms * 1e-3) / 1e12
    peak, _ = int8_peak()
    # reference on a row sample (row-split is bit-identical for single-block plans)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    T = cpu_threads()
    rows = max(2, T)
    t0 = time.perf_counter()
    po.matmul_complex_rows(*parts, rows, n, n, p, threads=T)
    dt = time.perf_counter() - t0
    return {"metric": "complex ball matmul terms/s (N^3 complex multiply-adds per second)",
            "value": n ** 3 / (ms * 1e-3), "unit": "terms/s", "ms_per_step": ms,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS (int8)",
                         "frac": achieved / peak, "kernel": gemm_kernel_name(lib),
                         "kernel_ms": per_launch_ms, "kernel_launches_timed": gl.value,
                         "work": f"4 real products x 2*N^3*ceil(h/8)^2 = 4 x {credited:.4g} int8 ops"},
            "clocks": clk.summary(),
            "cpu_baseline": {"value": rows * n * n / dt, "unit": "terms/s", "cores": T, "kind": "reference",
                             "sample": f"complex_matmul_ball on {rows} of {n} rows of A (row-split over {T} threads)"}}


def e2e_matmul(ops, a, b, n, p, steps):
    """host->device copy of A, B from pinned memory, compute, device->host read of C,
    every step, through the C ABI's host entry (apb_matmul_host)"""
    import ctypes as C
    from paper_1901_04289_b200.balls import BallArray, apb_mat, limbs_for
    lib = ops._lib.lib()
    ha, hb = a.pinned(), b.pinned()
    hc = BallArray.zeros(n * n, limbs_for(p)).pinned()
    am, bm, cm = apb_mat(ha.c(), n, n), apb_mat(hb.c(), n, n), apb_mat(hc.c(), n, n)
    # warm-up: every device buffer set needs three products before its whole step replays from the
    # library's captured graphs (eager + capture, then the graphs); the pipelined entry has two sets
    for _ in range(4):
        ops._lib.check(lib.apb_matmul_host(C.byref(am), C.byref(bm), p, 1, C.byref(cm)), "e2e warmup")
    t0 = time.perf_counter()
    for _ in range(steps):
        ops._lib.check(lib.apb_matmul_host(C.byref(am), C.byref(bm), p, 1, C.byref(cm)), "e2e")
    dt_sync = (time.perf_counter() - t0) / steps
    # pipelined entry: product i+1's H2D overlaps product i's compute and D2H
    for _ in range(8):
        ops._lib.check(lib.apb_matmul_host_submit(C.byref(am), C.byref(bm), p, 1, C.byref(cm)), "e2e warmup")
    ops._lib.check(lib.apb_matmul_host_drain(), "e2e warmup")
    t0 = time.perf_counter()
    for _ in range(steps):
        ops._lib.check(lib.apb_matmul_host_submit(C.byref(am), C.byref(bm), p, 1, C.byref(cm)), "e2e")
    ops._lib.check(lib.apb_matmul_host_drain(), "e2e drain")
    dt = (time.perf_counter() - t0) / steps
    return {"value": n ** 3 / dt, "unit": "terms/s", "ms_per_step": dt * 1e3,
            "h2d_bytes_per_step": a.nbytes() + b.nbytes(), "d2h_bytes_per_step": hc.nbytes(),
            "path": "apb_matmul_host_submit/drain (pinned host buffers; every step H2D of A and B, kernels, "
                    "D2H of C; consecutive steps overlap on copy-in / compute / copy-out streams)",
            "sync_call": {"value": n ** 3 / dt_sync, "ms_per_step": dt_sync * 1e3,
                          "path": "apb_matmul_host (one synchronous call per step)"}}


def cpu_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def cpu_matmul(a, b, n, p, rows=None, threads=None):
    """reference block_matmul_ball (oracle/_ref) on a row sample of A, all host threads"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    T = threads or cpu_threads()
    rows = rows or min(n, max(8, (16 if n >= 512 else 64) * T))
    sub = a.take(range(rows * n))
    t0 = time.perf_counter()
    po.matmul(sub, b, rows, n, n, p, which="ref", algo=1, threads=T)
    dt = time.perf_counter() - t0
    return {"value": rows * n * n / dt, "unit": "terms/s", "cores": T, "kind": "reference",
            "sample": f"block_matmul_ball on {rows} of {n} rows of A x full B (row-split over {T} threads)",
            "seconds": dt}


def run_dots(torch, steps, warmup, world, rank, want_e2e=True, want_cpu=True):
    from paper_1901_04289_b200 import gen, ops
    lib = ops._lib.lib()
    batch, n, p = 65536, 100, 128
    x, y = gen.config1_dots(batch=batch, n=n, p=p, seed_salt=rank)
    dx, dy = x.to_device(), y.to_device()
    from paper_1901_04289_b200.balls import DeviceBallArray, limbs_for
    out = DeviceBallArray.empty(batch, limbs_for(p))
    flush = L2Flush(torch)
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        ops.dot_batch(dx, dy, n, batch, p, out=out)
    torch.cuda.synchronize()
    lib.apb_profile_reset()
    lib.apb_profile_enable(1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    launches0 = ops.launch_count()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for k in range(steps):
            flush()
            ev[k][0].record(st)
            ops.dot_batch(dx, dy, n, batch, p, out=out, check=False)
            ev[k][1].record(st)
        torch.cuda.synchronize()
    launches = ops.launch_count() - launches0
    lib.apb_profile_enable(0)
    ms = sum(s.elapsed_time(e) for s, e in ev) / steps
    import ctypes as C
    t, c = C.c_double(0), C.c_uint64(0)
    lib.apb_profile_read(b"dot", C.byref(t), C.byref(c))
    lib.apb_profile_reset()
    kms = t.value / max(c.value, 1)
    terms = batch * n
    alg_bytes = terms * 2 * (8 * limbs_for(p) + 16)  # 2 balls x (8L+16) B per term
    peak, src = hbm_peak()
    res = {"metric": "ball dot terms/s", "value": world * terms / (ms * 1e-3), "unit": "terms/s",
           "ms_per_step": ms,
           "config": dots_config(batch, n, p, world),
           "roofline": {"bound": "hbm", "achieved": alg_bytes / (kms * 1e-3) / 1e9, "peak": peak,
                        "unit": "GB/s", "frac": alg_bytes / (kms * 1e-3) / 1e9 / peak,
                        "traffic": ncu_traffic("dot_reg_kernel"), "kernel": "dot_reg_kernel<32,4,1,0>",
                        "kernel_ms": kms, "work": f"{alg_bytes} algorithmic bytes per launch",
                        "timing": "CUDA events around the library's dot launch sequence (dot_reg_kernel "
                                  "+ the special-value pass) inside the timed steps",
                        "peak_source": src},
           "gpu_launches": launches, "clocks": clk.summary()}
    if want_e2e and rank == 0:
        xh, yh = x.pinned(), y.pinned()
        for _ in range(2):
            ops.dot_batch_host(xh, yh, n, batch, p)
        t0 = time.perf_counter()
        for _ in range(steps):
            ops.dot_batch_host(xh, yh, n, batch, p)
        dt = (time.perf_counter() - t0) / steps
        res["e2e"] = {"value": terms / dt, "unit": "terms/s", "ms_per_step": dt * 1e3,
                      "h2d_bytes_per_step": x.nbytes() + y.nbytes(),
                      "d2h_bytes_per_step": batch * (8 * limbs_for(p) + 21),
                      "path": "apb_dot_batch_host (pinned host buffers)"}
    if want_cpu and rank == 0 and world == 1:
        res["cpu_baseline"] = cpu_dots(x, y, n, batch, p)
    return res


def cpu_dots(x, y, n, batch, p, sample=None, threads=None):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    T = threads or cpu_threads()
    sample = sample or min(batch, 2048 * T)
    xs, ys = x.take(range(sample * n)), y.take(range(sample * n))
    t0 = time.perf_counter()
    po.dot_batch(xs, ys, n, sample, p, which="ref", threads=T)
    dt = time.perf_counter() - t0
    return {"value": sample * n / dt, "unit": "terms/s", "cores": T, "kind": "reference",
            "sample": f"dot_ball on {sample} of {batch} dots (batch split over {T} threads)",
            "seconds": dt}


# ------------------------------------------------------------- reference arm

def reference_arm(args, world, rank):
    if rank != 0:
        return 0
    from paper_1901_04289_b200 import gen
    T = cpu_threads()
    if args.config == "c1":
        batch, n, p = 65536, 100, 128
        x, y = gen.config1_dots(batch=batch, n=n, p=p)
        meas = [cpu_dots(x, y, n, batch, p, threads=T) for _ in range(args.warmup + args.steps)][args.warmup:]
        metric, cfg = "ball dot terms/s", dots_config(batch, n, p, world)
    else:
        a, b, n, p = matmul_workload(args.config, 0, args.prec)
        rows = min(n, max(8, 8 * T)) if n >= 1024 else None
        meas = [cpu_matmul(a, b, n, p, rows=rows, threads=T) for _ in range(args.warmup + args.steps)][args.warmup:]
        metric = "ball matmul terms/s (N^3 multiply-adds of p-bit balls per second)"
        cfg = matmul_config(args.config, n, p, world)
    v = statistics.median(m["value"] for m in meas)
    line = {"impl": "reference", "metric": metric, "value": v, "unit": "terms/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(m["seconds"] for m in meas) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64 limbs",
            "data": "synthetic (seeded generators, paper_1901_04289_b200/gen.py)", "config": cfg,
            "cpu_baseline": {"value": v, "unit": "terms/s", "cores": T, "kind": "reference",
                             "sample": meas[0]["sample"]},
            "e2e": {"value": v, "unit": "terms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c5"])
    ap.add_argument("--prec", type=int, default=None, help="precision for c5")
    ap.add_argument("--no-also", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        return reference_arm(args, world, rank)
    import torch
    dev = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    if world > 1:
        # NCCL over NVLink on a real multi-GPU box; BENCH_DIST_BACKEND=gloo only for
        # functional checks of the multi-rank path when fewer GPUs than ranks exist
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            torch.distributed.init_process_group(backend)
    from paper_1901_04289_b200 import build
    if not os.path.exists(build.LIB):
        raise SystemExit("libapb_b200.so missing: run __graft_entry__.build() first")
    if args.config == "c1":
        res = run_dots(torch, args.steps, args.warmup, world, rank)
    else:
        res = run_matmul(torch, args.config, args.steps, args.warmup, world, rank, p_override=args.prec)
    also = {}
    if not args.no_also and world == 1:
        for cfg in ("c2", "c1", "c4") if args.config == "c3" else ():
            try:
                if cfg == "c1":
                    r = run_dots(torch, 5, 3, 1, 0, want_e2e=False, want_cpu=True)
                elif cfg == "c4":
                    r = run_complex(torch, 3, 3)
                else:
                    r = run_matmul(torch, cfg, 5, 3, 1, 0, want_e2e=False, want_cpu=True)
                also[cfg] = {k: r[k] for k in ("metric", "value", "unit", "ms_per_step", "roofline",
                                               "cpu_baseline") if k in r}
            except Exception as e:  # noqa: BLE001
                also[cfg] = {"error": str(e)}
    if rank == 0:
        line = {"metric": res["metric"], "value": res["value"], "unit": res["unit"], "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "int8 slices / int32 accumulate (exact integer), u64 limbs",
                "data": "synthetic (seeded generators, paper_1901_04289_b200/gen.py)",
                "config": res["config"], "roofline": res["roofline"], "e2e": res.get("e2e"),
                "cpu_baseline": res.get("cpu_baseline"), "gpu_launches": res["gpu_launches"],
                "clocks": res["clocks"]}
        for extra in ("plan", "kernel_ms_per_step", "stage_ms_profiled_pass"):
            if extra in res:
                line[extra] = res[extra]
        if also:
            line["also"] = also
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
