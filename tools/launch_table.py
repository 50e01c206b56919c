"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv`) per kernel: launches, mean ms and DRAM MB per launch; with
`--traffic CFG` also write the sampling phase's per-step DRAM bytes (k_sample + k_big, the last
launch of each) into profiles/ncu_traffic.json for bench.py's roofline.traffic.

    python tools/launch_table.py launches.csv [--traffic C5 --source profiles/r01/launches.csv]"""
import argparse
import csv
import json
import os
import re
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(path):
    per = OrderedDict()  # launch id -> {name, metrics}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        d = per.setdefault(r["ID"], {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return per


def short(name):
    m = re.match(r"(?:void )?(?:girg::)?([A-Za-z_0-9]+(?:<[^>]*>)?)", name)
    return m.group(1) if m else name[:40]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--traffic", default=None)
    ap.add_argument("--source", default=None)
    a = ap.parse_args()
    per = load(a.csv)
    agg = OrderedDict()
    last = {}
    for lid, d in per.items():
        k = short(d["name"])
        g = agg.setdefault(k, [0, 0.0, 0.0, 0.0])
        g[0] += 1
        g[1] += d.get("gpu__time_duration.sum", 0.0)
        g[2] += d.get("dram__bytes_read.sum", 0.0)
        g[3] += d.get("dram__bytes_write.sum", 0.0)
        last[k] = d
    print("| kernel | launches | ms / launch | DRAM read MB | DRAM write MB |")
    print("|---|---|---|---|---|")
    for k, (c, t, r, w) in agg.items():
        unit = 1e-6 if t > 1e3 else 1e-3  # gpu__time_duration in ns (or us)
        print(f"| {k} | {c} | {t / c * unit:.3f} | {r / c / 1e6:.0f} | {w / c / 1e6:.1f} |")
    if a.traffic:
        ks = [k for k in last if k.startswith("k_sample")]
        kb = [k for k in last if k.startswith("k_big")]
        s = last[ks[-1]] if ks else {}
        b = last[kb[-1]] if kb else {}
        tr = lambda d: int(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0))  # noqa: E731
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        t = json.load(open(p)) if os.path.exists(p) else {}
        t["_note"] = ("per-step DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum, summed over k_sample and "
                      "k_big) from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none` of `python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e`; written by "
                      "tools/launch_table.py; consumed by bench.py as roofline.traffic")
        t[a.traffic] = {"sample_phase_dram_bytes": tr(s) + tr(b), "k_sample_dram_bytes": tr(s),
                        "k_big_dram_bytes": tr(b), "source": a.source or a.csv}
        with open(p, "w") as f:
            json.dump(t, f, indent=1)
        print("wrote", p, t[a.traffic])


if __name__ == "__main__":
    main()
