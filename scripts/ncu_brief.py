"""Key counters of an `ncu --page details --csv` export (one or more kernels)."""
import csv
import sys

KEYS = ("Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Registers Per Thread",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Theoretical Occupancy",
        "Warp Cycles Per Issued Instruction", "Issued Warp Per Scheduler", "Compute (SM) Throughput",
        "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate")
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr = rows[0]
    ki, ii = hdr.index("Kernel Name"), hdr.index("ID")
    cur = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d["ID"] != cur:
            cur = d["ID"]
            print(f"[{cur}] {d['Kernel Name'][:110]}")
        if d["Metric Name"] in KEYS:
            print(f"    {d['Metric Name'][:40]:40s} {d['Metric Value']} {d['Metric Unit']}")
