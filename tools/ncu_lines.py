"""Per-source-line warp-stall samples of one kernel in an ncu report (cuda,sass correlation).

    python tools/ncu_lines.py REPORT.ncu-rep [TOP] [--reasons]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, agg, hdr, per = None, {}, None, {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 5 and r[0] == "Line No":
            hdr = r
            continue
        if len(r) > 5 and r[0].isdigit():
            try:
                s = int(r[4])
            except ValueError:
                continue
            key = (cur, int(r[0]), r[1].strip()[:90])
            agg[key] = agg.get(key, 0) + s
            if hdr:
                d = per.setdefault(key, {})
                for i, n in enumerate(hdr):
                    if n.startswith("stall_") and "Not Issued" not in n:
                        try:
                            d[n] = d.get(n, 0) + int(r[i])
                        except ValueError:
                            pass
    tot = sum(agg.values())
    print("total samples", tot)
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        rs = sorted(per.get(k, {}).items(), key=lambda x: -x[1])[:3]
        print(f"{v:7d} {100 * v / tot:5.1f}%  {k[0]}:{k[1]}  {k[2]}   " + " ".join(f"{n[6:]}={c}" for n, c in rs))


if __name__ == "__main__":
    main()
