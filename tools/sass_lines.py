"""Static SASS size per source line of one kernel, from `nvdisasm -g` output (line-info comments):
    python tools/sass_lines.py all.sass <mangled kernel name> [top]"""
import re
import sys
from collections import Counter

path, name = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
per, cur, inside, n = Counter(), None, False, 0
for line in open(path):
    if line.startswith(".text."):
        inside = line.strip() == f".text.{name}:"
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s", line):
        per[cur] += 1
        n += 1
print(f"{name}: {n} instructions ({16 * n / 1024:.0f} KB)")
for k, v in per.most_common(top):
    print(f"{v:6d}  {k}")
