"""Summarise ST_PROF_TRACE=1 stderr lines (bf16 encoder) per (kernel class, layer)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle
import workloads as W

cfgn, log = int(sys.argv[1]), sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
bf = sys.argv[4] if len(sys.argv) > 4 else "1"
cfg = W.get_config(cfgn)
net = cfg.build_net()
shp = oracle.shapes(net)
recs = [dict(kv.split("=") for kv in l.split()[1:]) for l in open(log) if l.startswith(f"[st-prof] bf={bf}")]
agg = collections.defaultdict(list)
info = {}
for d in recs:
    k = (int(d["cls"]), int(d["layer"]))
    agg[k].append(float(d["ms"]))
    info[k] = (d.get("M"), d.get("Min"), d.get("GBps"))
n = int(os.environ.get("TRACE_STEPS", "0")) or max(len(v) for v in agg.values())
tot = sum(sum(v) for v in agg.values()) / n
print(f"cfg{cfgn}: {n} passes, {tot:.3f} ms per pass")
for (c, li), v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:top]:
    L = net.layers[li] if li >= 0 else {"kind": -1}
    print(f"cls={c:2d} L{li:3d} kind={L['kind']} out={shp[li] if li >= 0 else None} k={L.get('k_h', '')} "
          f"g={L.get('groups', '')} ms={sum(v) / n:.3f} ({100 * sum(v) / n / tot:.1f}%) M,Min,GB/s={info[(c, li)]}")
