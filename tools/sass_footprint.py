"""Hot-code footprint of a kernel from an `ncu --page source --csv --print-source cuda,sass` export:
SASS instructions sorted by execution count, the bytes (16 per instruction) that cover 50/90/99 % of
the executed warp instructions, and the no-instruction stall samples by source region.
    python tools/sass_footprint.py src.csv.gz"""
import csv
import gzip
import sys
from collections import defaultdict


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


f = gzip.open(sys.argv[1], "rt") if sys.argv[1].endswith(".gz") else open(sys.argv[1])
rd = csv.reader(f)
cur, curline, hdr = None, None, None
sass = {}  # address -> (executed, source line, stall samples, no-instr samples)
for r in rd:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] != "":
        curline = f"{cur}:{r[0]}"
        continue
    addr = r[2]
    if addr in sass:
        continue
    sass[addr] = (num(r[7]), curline, num(r[4]))
tot = sum(v[0] for v in sass.values())
xs = sorted((v[0] for v in sass.values()), reverse=True)
print(f"SASS instructions {len(sass)} ({16 * len(sass) / 1024:.0f} KB), executed warp instructions {tot:.3e}")
acc, marks = 0, [0.5, 0.9, 0.99, 0.999]
for i, x in enumerate(xs):
    acc += x
    while marks and acc >= marks[0] * tot:
        print(f"  {marks[0] * 100:.1f}% of executed instructions covered by {i + 1} instructions = {16 * (i + 1) / 1024:.1f} KB")
        marks.pop(0)
print("executed-once-or-more instructions:", sum(1 for x in xs if x > 0), f"= {16 * sum(1 for x in xs if x > 0) / 1024:.0f} KB")

if len(sys.argv) > 2:  # per source line: SASS instructions in the hot set (covering 99 %) and executions
    thr = None
    acc = 0
    for x in xs:
        acc += x
        if acc >= 0.99 * tot:
            thr = x
            break
    per = defaultdict(lambda: [0, 0])
    for ex, line, _ in sass.values():
        if ex >= thr:
            per[line][0] += 1
            per[line][1] += ex
    rows = sorted(per.items(), key=lambda kv: -kv[1][0])
    print(f"hot set (executions >= {thr}): {sum(v[0] for v in per.values())} SASS instructions")
    for line, (n, ex) in rows[: int(sys.argv[2])]:
        print(f"{n:5d} instr {ex / tot * 100:5.1f}% exec  {line}")
