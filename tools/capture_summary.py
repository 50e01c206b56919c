"""Summarise `ncu --page raw --csv` exports of the sampling kernels (one launch each) into
profiles/ncu_issue.json (bench.py's roofline.issue): the issue-slot evidence of the phase.
    python tools/capture_summary.py CFG k_sample_raw.csv k_big_raw.csv m_edges"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "ms_ncu": "gpu__time_duration.sum",
    "warp_inst": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_read_gb": "dram__bytes_read.sum",
    "registers": "launch__registers_per_thread",
    "threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
}


def one(path):
    with open(path) as f:
        rows = [r for r in csv.reader(line for line in f if line.startswith('"'))]
    hdr, units, vals = rows[0], rows[1], rows[-1]
    out = {}
    for k, m in KEYS.items():
        if m not in hdr:
            continue
        i = hdr.index(m)
        v = float(vals[i].replace(",", ""))
        u = units[i]
        if m == "gpu__time_duration.sum":
            v = v / 1e6 if u == "ns" else (v / 1e3 if u == "us" else v)
        if m == "dram__bytes_read.sum":
            v = v / 1e3 if u == "Mbyte" else (v / 1e6 if u == "Kbyte" else v)
        out[k] = v
    return out


def main():
    cfg, fs, fb, m = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
    s, b = one(fs), one(fb)
    wi = s["warp_inst"] + b["warp_inst"]
    p = os.path.join(ROOT, "profiles", "ncu_issue.json")
    t = json.load(open(p)) if os.path.exists(p) else {}
    t["_note"] = ("issue-slot evidence of the sampling kernels (ncu --set full --clock-control none, one launch each, "
                  "python tools/prof_one.py CFG merged 1 nostats); raw pages in profiles/r02/final/; consumed by bench.py as "
                  "roofline.issue; written by tools/capture_summary.py")
    t[cfg] = {"k_sample": s, "k_big": b, "sampling_phase": {
        "warp_inst": wi, "warp_inst_per_edge": wi / m,
        "issue_active_pct_weighted": (s["issue_active_pct"] * s["ms_ncu"] + b["issue_active_pct"] * b["ms_ncu"]) /
        (s["ms_ncu"] + b["ms_ncu"])}}
    with open(p, "w") as f:
        json.dump(t, f, indent=1)
    print(json.dumps(t[cfg], indent=1))


if __name__ == "__main__":
    main()
