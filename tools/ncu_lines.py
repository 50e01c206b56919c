"""Summarise an `ncu --page source --csv --print-source cuda,sass` export per CUDA source line:
top lines by warp-stall samples, with instructions executed and average active threads.
    python tools/ncu_lines.py src.csv [top]"""
import csv
import sys

rows, cur_file = [], None
with open(sys.argv[1]) as f:
    rd = csv.reader(f)
    hdr = None
    for r in rd:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0]:
            continue
        d = dict(zip(hdr[:4], r[:4]))
        try:
            samples = int(r[4]); inst = int(r[7]); thr = float(r[10])
        except (ValueError, IndexError):
            continue
        rows.append((samples, inst, thr, cur_file, r[0], r[1][:90]))
tot_s = sum(x[0] for x in rows) or 1
tot_i = sum(x[1] for x in rows) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(f"total stall samples {tot_s}, warp instructions {tot_i:.3e}")
for s, i, t, fn, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst thr {t:4.1f} {fn}:{ln} {src}")
