"""Summarise an ncu --set full report: per-kernel duration, DRAM bytes, occupancy, top stall reasons,
smem wavefronts/bank conflicts and L1 wavefronts (prints a compact table)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]


def g(r, name):
    try:
        return float(r[hdr.index(name)].replace(",", ""))
    except Exception:
        return float("nan")


for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0][:40]
    dur = g(r, "gpu__time_duration.sum")
    rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
    occ = g(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
    regs = g(r, "launch__registers_per_thread")
    shw = g(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    shc = g(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
    gw = g(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
    ipc = g(r, "sm__inst_executed.avg.per_cycle_active")
    fp64 = g(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
    stalls = []
    for h in hdr:
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            v = g(r, h)
            if v == v and v > 0.2:
                stalls.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    stalls.sort(reverse=True)
    print(f"{name:40s} {dur/1e3:9.1f}us dram r/w {rd:.3g}/{wr:.3g} occ {occ:.0f}% regs {regs:.0f} ipc {ipc:.2f} "
          f"fp64 {fp64:.0f}% smem wf {shw:.3g} conf {shc:.3g}")
    print("      stalls:", ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))
