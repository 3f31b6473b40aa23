"""Summarize an ncu report's SASS source page: instructions executed and stall samples by opcode,
and the hottest instructions.  usage: python tools/ncu_sass_summary.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
si, ii, ai = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
by_op = defaultdict(lambda: [0, 0])
lines = []
tot_i = tot_s = 0
for r in rows[2:]:
    if len(r) <= max(si, ii, ai):
        continue
    src = r[si].strip()
    try:
        n = int(r[ii] or 0)
        s = int(r[ai] or 0)
    except ValueError:
        continue
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    by_op[op][0] += n
    by_op[op][1] += s
    tot_i += n
    tot_s += s
    lines.append((s, n, r[0], src))
print(f"total warp-instructions {tot_i}  stall samples {tot_s}")
for op, (n, s) in sorted(by_op.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{op:12s} inst {n:12d} ({100*n/max(tot_i,1):5.1f}%)  stalls {100*s/max(tot_s,1):5.1f}%")
print("--- hottest instructions by stall samples ---")
for s, n, addr, src in sorted(lines, reverse=True)[:top]:
    print(f"{100*s/max(tot_s,1):5.1f}% {n:10d} {src[:90]}")
