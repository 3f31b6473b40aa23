"""Per-instruction SASS walk of one kernel in an ncu report: executed warp-instructions
normalized by a unit count (e.g. warp-tiles), stall share, and the instruction text.
usage: python tools/sass_walk.py report.ncu-rep kernel_regex unit_count [min_norm]"""
import csv
import io
import subprocess
import sys

rep, kern, unit = sys.argv[1], sys.argv[2], float(sys.argv[3])
min_norm = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
si, ii, ai = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
tot_i = tot_s = 0
data = []
for r in rows[2:]:
    if len(r) <= max(si, ii, ai):
        continue
    try:
        n, s = int(r[ii] or 0), int(r[ai] or 0)
    except ValueError:
        continue
    tot_i += n
    tot_s += s
    data.append((r[0][-5:], n, s, r[si].strip()))
print(f"total {tot_i} warp-inst = {tot_i / unit:.1f} per unit; stall samples {tot_s}")
for a, n, s, src in data:
    if n / unit >= min_norm:
        print(f"{a} {n / unit:7.2f} {100 * s / max(tot_s, 1):5.1f}% {src[:110]}")
