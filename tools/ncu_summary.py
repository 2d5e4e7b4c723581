"""Key metrics of an ncu report (details page) + warp-state breakdown.
    python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Eligible Warps", "No Eligible", "Warp Cycles Per Issued", "Executed Instructions", "Registers Per Thread",
        "Block Limit", "Achieved Active Warps", "Theoretical Occupancy", "Dynamic Shared", "Grid Size", "Block Size",
        "L1/TEX Hit", "L2 Hit", "Mem Busy", "Max Bandwidth", "Compute (SM)", "Shared Memory", "Bank")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    name = d.get("Metric Name", "")
    if any(k in name for k in KEEP):
        print(f"{d.get('Section Name','')[:28]:28s} {name[:48]:48s} {d.get('Metric Unit','')[:10]:10s} {d.get('Metric Value','')}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units, vals = rr[0], rr[1], rr[2]
stalls = []
for name, u, v in zip(h, units, vals):
    if name.startswith("smsp__average_warp_latency_issue_stalled_") and name.endswith(".ratio"):
        try:
            stalls.append((float(v), name.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", "")))
        except ValueError:
            pass
    if name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active"):
        print(f"{'raw':28s} {name:60s} {u:10s} {v}")
print("\nwarp stall cycles per issued instruction (top):")
for v, n in sorted(stalls, reverse=True)[:12]:
    print(f"  {n:40s} {v:.2f}")
