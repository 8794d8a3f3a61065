#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (tracked).

  python scripts/ncu_summary.py --round r01 --launches gpurun_out/launches_r01.csv \
      --full conv_sparse=gpurun_out/conv_sparse_r01.ncu-rep [...]

Writes profiles/<round>_launches.md (per-kernel share of the step from the
`--metrics gpu__time_duration.sum --clock-control none` launch list: cold-
cache and serialised, so compare SHARES), profiles/<round>_ncu_<class>.txt
(key counters of one `--set full` capture) and merges dram bytes per launch
into profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "lts__t_bytes.sum", "l1tex__t_bytes.sum"]


def short(name):
    m = re.search(r"(k_\w+)", name)
    return m.group(1) if m else name[:40]


def launches(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    per = collections.OrderedDict()
    tot = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        v = v / 1e3 if unit in ("usecond", "us") else v / 1e6 if unit in ("nsecond", "ns") else v
        k = short(r["Kernel Name"])
        d = per.setdefault(k, [0, 0.0])
        d[0] += 1
        d[1] += v
        tot += v
    return per, tot, len(rows)


def full(path):
    """Key counters per kernel from an .ncu-rep, or from the raw CSV that
    scripts/ncu_export.py wrote box-side (*.csv)."""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                d[k] = (vals[hdr.index(k)], units[hdr.index(k)])
        res.append(d)
    return res


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--config", type=int, default=2, help="bench config the captures were taken on")
    a = ap.parse_args()
    os.makedirs("profiles", exist_ok=True)
    if a.launches:
        per, tot, n = launches(a.launches)
        with open(f"profiles/{a.round}_launches.md", "w") as f:
            f.write(f"# {a.round} launch list ({a.launches}; ncu --metrics gpu__time_duration.sum "
                    f"--clock-control none; cold-cache, serialised -> compare shares)\n\n")
            f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
            for k, (c, ms) in sorted(per.items(), key=lambda kv: -kv[1][1]):
                f.write(f"| {k} | {c} | {ms:.3f} | {ms / tot:.1%} |\n")
            f.write(f"\nTotal {tot:.3f} ms over {n} launches.\n")
    summ_p = "profiles/ncu_summary.json"
    summ = json.load(open(summ_p)) if os.path.exists(summ_p) else {"kernels": {}}
    for spec in a.full:
        cls, path = spec.split("=", 1)
        pat = None
        if "@" in path:   # cls=path@regex: keep kernels whose name matches regex
            path, pat = path.split("@", 1)
        res = full(path)
        if pat:
            res = [d for d in res if re.search(pat, d["kernel"])]
        with open(f"profiles/{a.round}_ncu_{cls}.txt", "w") as f:
            f.write(f"# {a.round} ncu --set full --clock-control none ({os.path.basename(path)})\n")
            for d in res:
                f.write(f"\n{d['kernel']}\n")
                for k in KEYS:
                    if k in d:
                        f.write(f"  {k:70s} {d[k][0]} {d[k][1]}\n")
        rd = sum(to_bytes(*d["dram__bytes_read.sum"]) for d in res) / len(res)
        wr = sum(to_bytes(*d["dram__bytes_write.sum"]) for d in res) / len(res)
        ten = [float(d[k][0]) for d in res for k in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",)
               if k in d and d[k][0] not in ("", "n/a")]
        summ["kernels"][cls] = {"round": a.round, "config": a.config, "kernel": res[0]["kernel"],
                                "launches_averaged": len(res),
                                "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                                "tensor_pipe_active_pct_mean": (sum(ten) / len(ten)) if ten else None,
                                "source": os.path.basename(path)}
    json.dump(summ, open(summ_p, "w"), indent=1)


if __name__ == "__main__":
    main()
