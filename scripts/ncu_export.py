#!/usr/bin/env python
"""Box-side: shrink an ncu report to a small CSV of the counters we read,
then delete the .ncu-rep (gpurun only copies back <= 64 MiB of gpurun_out/).

    python scripts/ncu_export.py gpurun_out/x.ncu-rep gpurun_out/x_raw.csv

Keeps the identification columns and every metric whose name starts with one
of PREFIXES (times, DRAM / L2 / L1 bytes and hit rates, pipe utilisation,
issue / occupancy, launch configuration, warp stall breakdown)."""
import csv
import io
import os
import subprocess
import sys

PREFIXES = ("ID", "Kernel Name", "Block Size", "Grid Size", "gpu__time_duration", "dram__bytes", "dram__throughput",
            "gpu__dram_throughput", "gpu__compute_memory_throughput", "sm__throughput", "sm__pipe_",
            "sm__inst_executed_pipe_", "smsp__issue_active", "sm__warps_active", "launch__", "lts__t_bytes",
            "lts__t_sector_hit_rate", "l1tex__t_bytes", "l1tex__t_sector_hit_rate", "smsp__average_warp",
            "smsp__pcsamp_warps_issue_stalled", "sm__maximum_warps", "smsp__warps_eligible",
            "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "dram__sectors")


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if not rows:
        print("empty report", file=sys.stderr)
        return 1
    hdr = rows[0]
    keep = [i for i, h in enumerate(hdr) if h.startswith(PREFIXES)]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        for r in rows:
            w.writerow([r[i] if i < len(r) else "" for i in keep])
    os.remove(rep)
    print(f"{out}: {len(rows) - 2} kernels x {len(keep)} columns")
    return 0


if __name__ == "__main__":
    sys.exit(main())
