"""Top SASS instructions by sampled stalls from an ncu source-page CSV
    ncu -i X.ncu-rep --page source --csv --print-source sass > x.csv; python tools/ncu_sass_top.py x.csv [N] [stall]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
cols = ["stall_long_sb", "stall_mio", "stall_wait", "stall_math", "stall_short_sb", "stall_barrier",
        "stall_branch_resolving", "stall_not_selected", "stall_selected"]
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ix[key]] or 0), r))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total", key, tot)
for n, r in sorted(data, key=lambda x: -x[0])[:N]:
    extra = " ".join(f"{c[6:]}={r[ix[c]]}" for c in cols if r[ix[c]] not in ("0", ""))
    print(f"{n:7d} {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:70]:70s} {extra}")
