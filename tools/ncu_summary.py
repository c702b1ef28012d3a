"""Key metrics + stall breakdown + hottest SASS blocks of one ncu report:
python tools/ncu_summary.py REPORT.ncu-rep [launch index]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2 + idx]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
for i, n in enumerate(h):
    if n in want or "pipe_tensor" in n and "pct" in n:
        print(f"{n:70s} {v[i]}")
st = [(n, v[i]) for i, n in enumerate(h)
      if n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio")]
st = sorted(((float(x), n.split("stalled_")[1].split("_per")[0]) for n, x in st if x), reverse=True)
print("stalls per issue:", ", ".join(f"{n} {x:.2f}" for x, n in st[:9]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = rows[2:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex, ismp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iex] or 0) for r in data) or 1
totsmp = sum(float(r[ismp] or 0) for r in data) or 1
print(f"total SASS instructions executed {tot:.4g}")
top = sorted(data, key=lambda r: -float(r[ismp] or 0))[:25]
for r in top:
    print(f"  {float(r[ismp] or 0) / totsmp * 100:5.1f}% smp  ex={float(r[iex] or 0):9.3g}  {r[isrc][:90]}")
