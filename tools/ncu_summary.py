"""Summarise an ncu --set full report (raw page) into the profiles/ text format:
key throughput / pipe / DRAM metrics and the top warp-stall reasons.

usage: ncu_summary.py REPORT.ncu-rep TITLE > summary.txt
"""
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
print(f"# {title}")
print("# ncu --set full --clock-control none --import-source on (metric value, unit)")
for w in want:
    if w in hdr:
        k = hdr.index(w)
        print(f"{w} {vals[k]} {units[k]}".rstrip())
st = [(h, vals[i]) for i, h in enumerate(hdr)
      if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
tot = sum(float(v or 0) for _, v in st) or 1.0
for h, v in sorted(st, key=lambda x: -float(x[1] or 0))[:8]:
    print(f"{h} {100 * float(v) / tot:.1f}%")
