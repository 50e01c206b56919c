"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export (gzip ok) into source
regions (line ranges per file): share of warp instructions and of stall samples.
    python tools/ncu_regions.py src.csv.gz"""
import csv
import gzip
import sys

REGIONS = [  # (file, lo, hi, name): sample.cuh / girg_device.cuh as of the final round-2 code (with R27)
    ("sample.cuh", 290, 387, "warp helpers, emit/flush"),
    ("sample.cuh", 388, 404, "load_rec"),
    ("sample.cuh", 405, 459, "divmod/chunk_log2/exact/make_task"),
    ("sample.cuh", 460, 621, "setup_common (region, ranges, children)"),
    ("sample.cuh", 622, 861, "setup_job (classify, prefixes, offsets)"),
    ("sample.cuh", 862, 985, "setup_job_ref (R27 refined jobs)"),
    ("sample.cuh", 986, 1113, "setup_job1 (d = 1)"),
    ("sample.cuh", 1114, 1227, "locate"),
    ("sample.cuh", 1228, 1271, "counters/push_items"),
    ("sample.cuh", 1272, 1434, "tile/item source"),
    ("sample.cuh", 1435, 1738, "engine loop"),
    ("sample.cuh", 1739, 1786, "engine_cand (T = 0)"),
    ("girg_device.cuh", 1, 39, "philox/u53"),
    ("girg_device.cuh", 40, 113, "morton"),
    ("girg_device.cuh", 114, 196, "det_log/exp (R26, exact paths)"),
    ("girg_device.cuh", 197, 220, "dist/prob"),
    ("girg_device.cuh", 221, 400, "fast paths"),
]


def region(fn, ln):
    for f, lo, hi, name in REGIONS:
        if fn == f and lo <= ln <= hi:
            return name
    return fn


def main(path):
    op = gzip.open if path.endswith(".gz") else open
    agg, cur = {}, None
    with op(path, "rt") as f:
        hdr = None
        for r in csv.reader(f):
            if len(r) == 2 and r[0] == "File Path":
                cur = r[1].split("/")[-1]
                continue
            if r and r[0] == "Line No":
                hdr = r
                continue
            if hdr is None or not r or not r[0]:
                continue
            try:
                ln, smp, inst = int(r[0]), int(r[4]), int(r[7])
            except (ValueError, IndexError):
                continue
            k = region(cur, ln)
            a = agg.setdefault(k, [0, 0])
            a[0] += smp
            a[1] += inst
    ts = sum(a[0] for a in agg.values()) or 1
    ti = sum(a[1] for a in agg.values()) or 1
    print(f"warp instructions {ti:.3e}, stall samples {ts}")
    for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% samples  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
