"""One line per kernel from an ncu report: duration, DRAM bytes, issue, tensor, top stall reasons.
usage: python tools/ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]


def col(r, name):
    return r[h.index(name)] if name in h else "?"


for r in rows[2:]:
    stalls = []
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warp_latency_issue_stalled_") or \
           (name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued")):
            try:
                stalls.append((float(r[i].replace(",", "")), name.split("stalled_")[1]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    tot = sum(v for v, _ in stalls) or 1.0
    print(f"{col(r, 'Kernel Name')[:48]:48s} {col(r, 'gpu__time_duration.sum'):>9s} us  "
          f"dram R/W {col(r, 'dram__bytes_read.sum')}/{col(r, 'dram__bytes_write.sum')} MB  "
          f"issue {col(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active')}%  "
          f"tensor {col(r, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active')}%  "
          f"regs {col(r, 'launch__registers_per_thread')}")
    print("    stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in stalls[:6]))
