"""One-line summary of a bench JSON line (gpurun_out/bench_cfgN.json)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as ex:
        print(f, "unreadable", ex)
        continue
    r = d["roofline"]
    print(f"{f}: {d['value']:.0f} {d['unit']} ms/step {d['ms_per_step']:.3f} e2e {d['e2e']['value']:.0f} "
          f"dense x{d.get('speedup_vs_dense')} roof {r['kernel']} {r['achieved']} frac {r['frac']} share {r['share_of_step']:.3f}")
    kr = d.get("kernel_roofline", {})
    for k, v in sorted(d["kernel_ms_per_step"].items(), key=lambda x: -x[1]):
        print(f"    {k:22s} {v:8.3f} ms  {kr.get(k, '')}")
