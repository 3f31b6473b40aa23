"""Compact text summary of one ncu --set full report (for profiles/).
usage: python tools/ncu_report.py report.ncu-rep [alg_bytes] > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
print(f"# ncu --set full summary of {rep.split('/')[-1]}")
for r in rows[2:]:
    m = dict(zip(h, r))
    um = dict(zip(h, u))
    print(f"kernel: {m.get('Kernel Name')}  grid {m.get('launch__grid_size')} x block {m.get('launch__block_size')}"
          f"  regs {m.get('launch__registers_per_thread')}  dyn smem {m.get('launch__shared_mem_per_block_dynamic')}")
    def g(k):
        return m.get(k, "n/a"), um.get(k, "")
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
            "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active"]
    for k in keys:
        v, unit = g(k)
        print(f"  {k:70s} {v:>18s} {unit}")
    try:
        dur = float(m["gpu__time_duration.sum"]) * (1e-9 if um["gpu__time_duration.sum"] == "ns" else 1e-6)
        traffic = float(m["dram__bytes_read.sum"]) * (1e6 if um["dram__bytes_read.sum"] == "Mbyte" else 1) + \
            float(m["dram__bytes_write.sum"]) * (1e6 if um["dram__bytes_write.sum"] == "Mbyte" else 1)
        print(f"  dram traffic per launch: {traffic:.4g} B")
        if alg:
            print(f"  algorithmic bytes per launch: {alg:.4g} B  (traffic/alg = {traffic / alg:.2f})")
    except Exception:
        pass
    stalls = [(float(m[k]), k) for k in h if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")
              and m.get(k, "").replace(".", "").isdigit()]
    tot = sum(x for x, _ in stalls) or 1
    print("  warp stall samples:")
    for x, k in sorted(stalls, reverse=True)[:6]:
        print(f"    {100 * x / tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
