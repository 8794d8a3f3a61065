"""Where a kernel's instructions go: per CUDA source line, the warp-level
instructions executed and stall samples of one launch in an ncu report
(-lineinfo build, --import-source on).

    python scripts/ncu_insts.py report.ncu-rep [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hi]
print(rows[0][:2] if rows else "")
ie = next((i for i, h in enumerate(hdr) if h.startswith("Instructions Executed")), None)
ss = next((i for i, h in enumerate(hdr) if h.startswith("Warp Stall Sampling (All")), None)
isrc, iln = hdr.index("Source"), hdr.index("#") if "#" in hdr else 0


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


data = [(num(r[ie]) if ie is not None else 0, num(r[ss]) if ss is not None else 0, r[iln], r[isrc].strip()[:100])
        for r in rows[hi + 1:] if len(r) > isrc]
tot_i = sum(d[0] for d in data) or 1
tot_s = sum(d[1] for d in data) or 1
print(f"instructions {tot_i:.4g}  stall samples {tot_s:.4g}")
for d in sorted(data, key=lambda d: -d[0])[:top]:
    print(f"{100 * d[0] / tot_i:5.1f}% inst {100 * d[1] / tot_s:5.1f}% stall  L{d[2]:>5} {d[3]}")
