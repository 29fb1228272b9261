"""Extract the judged metrics from ncu reports into a committed text summary.

    python profiles/ncu_summary.py OUT.md REPORT.ncu-rep [REPORT2.ncu-rep ...]
    python profiles/ncu_summary.py --launches OUT.md launches.csv

Reports are produced on the GPU box; only the text
summaries are committed (the .ncu-rep files are large)."""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
]


def report_rows(path: str):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        yield {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def summarize(paths):
    lines = []
    for p in paths:
        for r in report_rows(p):
            name = r.get("Kernel Name", ("?", ""))[0]
            lines.append(f"### {p.split('/')[-1]} :: {name[:90]}")
            lines.append("| metric | value | unit |")
            lines.append("|---|---|---|")
            for m in METRICS:
                if m in r:
                    v, u = r[m]
                    lines.append(f"| {m} | {v} | {u} |")
            lines.append("")
    return "\n".join(lines)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"].split("(")[0][-70:]
                unit = d["Metric Unit"]
                v = float(d["Metric Value"].replace(",", ""))
                scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                         "msecond": 1e3, "s": 1e6, "second": 1e6}.get(unit, 1.0)
                v = v * scale
                agg.setdefault(k, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in agg.items():
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot:.1%} |")
    return "\n".join(lines)


if __name__ == "__main__":
    out_arg = sys.argv[2] if sys.argv[1] == "--launches" else sys.argv[1]
    if not out_arg.endswith(".md"):
        sys.exit(f"output must be a .md summary, got {out_arg!r} (would clobber a report)")
    if sys.argv[1] == "--launches":
        text = launches(sys.argv[3])
        out = sys.argv[2]
    else:
        out = sys.argv[1]
        text = summarize(sys.argv[2:])
    with open(out, "a") as f:
        f.write(text + "\n")
    print(text)
