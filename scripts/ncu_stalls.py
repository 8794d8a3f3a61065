"""Top stall sites of one kernel launch in an ncu report (SASS source page)."""
import csv
import io
import subprocess
import sys

rep, skip = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
seen, d2 = set(), []
for r in rows[2:]:
    if not r or not r[0].startswith("0x") or r[0] in seen:
        continue
    seen.add(r[0])
    d2.append(r)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
val = lambda r: int(r[i_s]) if r[i_s].strip().isdigit() else 0
tot = sum(val(r) for r in d2)
print(rows[0][1][:80], "samples", tot)
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
for k, r in enumerate(d2[:-1]):
    if val(r) > thr * tot or any(x in r[1] for x in ("UTCHMMA", "TRYWAIT", "UTMALDG")):
        print(str(val(r)).rjust(6), r[0][-5:], r[1][:90])
