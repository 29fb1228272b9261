"""Aggregate an ncu SASS source-page CSV (per-instruction stall samples) to CUDA source lines,
using the line table nvdisasm -g prints for the kernel's cubin.

    cuobjdump -xelf all libems_b200.so; nvdisasm -g -c fwd2_tc.sm_100a.cubin > k.dis
    ncu -i X.ncu-rep --page source --csv --print-source sass > k.csv
    python tools/ncu_lines_sass.py k.dis k.csv <kernel-substring> [N]"""
import csv
import re
import sys
from collections import defaultdict

dis, csvf, kname = sys.argv[1], sys.argv[2], sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.strip().startswith(".section") and kname in l and ".text." in l)
cur = None
m = {}
for l in lines[start + 1:]:
    if l.strip().startswith(".section"):
        break
    mm = re.search(r'//## File "(.*?)", line (\d+)', l)
    if mm:
        cur = (mm.group(1).split("/")[-1], int(mm.group(2)))
        continue
    mm = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if mm and cur:
        m[int(mm.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
base = int(rows[2][ix["Address"]], 16)
agg = defaultdict(lambda: defaultdict(int))
cols = ["Warp Stall Sampling (All Samples)", "stall_long_sb", "stall_mio", "stall_wait", "stall_math",
        "stall_short_sb", "stall_barrier", "stall_branch_resolving", "stall_not_selected", "stall_selected"]
for r in rows[2:]:
    try:
        off = int(r[ix["Address"]], 16) - base
    except ValueError:
        continue
    key = m.get(off, ("?", 0))
    for c in cols:
        try:
            agg[key][c] += int(r[ix[c]] or 0)
        except (ValueError, KeyError):
            pass
tot = sum(v[cols[0]] for v in agg.values())
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][cols[0]])[:N]:
    extra = " ".join(f"{c[6:]}={v[c]}" for c in cols[1:] if v[c] > 0.05 * v[cols[0]])
    print(f"{v[cols[0]]:7d} {100 * v[cols[0]] / tot:5.1f}% {k[0]}:{k[1]:<5} {extra}")
