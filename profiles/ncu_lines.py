"""Per-source-line instruction counts and stall samples from an ncu report
(--page source --print-source cuda,sass), top N lines.
Usage: python profiles/ncu_lines.py REPORT.ncu-rep [N] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
f = fname = None
rows = []
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0] != "":
        try:
            ie = int(r[hdr.index("Instructions Executed")])
            ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        rows.append((ie, ss, f"{fname}:{r[0]}", r[1].strip()[:100]))
ti = sum(x[0] for x in rows)
ts = sum(x[1] for x in rows)
print(f"total warp instructions {ti}  stall samples {ts}")
for ie, ss, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{ie:>11} {100*ie/max(ti,1):5.1f}%  stall {100*ss/max(ts,1):5.1f}%  {loc:24s} {src}")
