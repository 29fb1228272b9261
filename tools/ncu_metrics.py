"""Print the key pipe/stall metrics of an ncu report (first kernel)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines())); d = dict(zip(rows[0], rows[2]))
for k in ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_issued.avg.pct_of_peak_sustained_active",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread"]:
    print(f"{k:70s} {d.get(k)}")
st = sorted(((float(v.replace(',', '')), k) for k, v in d.items()
             if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")), reverse=True)
for v, k in st[:10]:
    print(f"{int(v):10d} {k}")
