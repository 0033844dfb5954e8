"""Summarise an ncu report (--set full) per kernel: duration, DRAM bytes,
throughputs, occupancy, registers and the top warp-stall reasons.
Usage: python profiles/ncu_summary.py report.ncu-rep [> summary.txt]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active", "imma_pct"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}
    ki = col["Kernel Name"]
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "")
        parts = []
        for k, short in KEYS:
            if k in col and r[col[k]] not in ("", "n/a"):
                parts.append(f"{short}={r[col[k]]}{units[col[k]] if units[col[k]] not in ('', 'n/a') else ''}")
        stalls = []
        for k, i in col.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(v for v, _ in stalls) or 1.0
        top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in stalls[:4])
        print(f"{name}\n    " + "  ".join(parts) + f"\n    stalls: {top}")


if __name__ == "__main__":
    main(sys.argv[1])
