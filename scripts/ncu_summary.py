"""Key metrics of each kernel in an ncu report (details page)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
want = {"Duration", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Compute (SM) Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Block Limit Registers",
        "FP64 Pipe Utilization", "Dynamic Shared Memory Per Block"}
cur = None
for r in rows[1:]:
    if r[mi] in want:
        tag = (r[ii], r[ki][:70])
        if tag != cur:
            print("==", *tag)
            cur = tag
        print(f"    {r[mi]}: {r[vi]} {r[ui]}")
