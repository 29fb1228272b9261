"""Score-pass time drift: 40 back-to-back config-3 passes (the power cap engaging), then 10
passes separated by 200 ms idle gaps (each starts unthrottled).  python tools/drift.py"""
import torch, time, sys, os
sys.path.insert(0, os.getcwd())
from paper_2412_08521_b200 import ems
from paper_2412_08521_b200.inputs import CONFIGS, make_batch_torch
w = CONFIGS["cfg3"]; dev = torch.device("cuda")
q, kr, kw, v = make_batch_torch(w, seed=1, device=dev)
B, Hq, L, d = q.shape
plan = ems.Plan(B, Hq, w.heads_kv, L, d, q.dtype, ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma), dev, "tcgen05", want_out=True)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(40)]
torch.cuda.synchronize()
for i, (a, m, b) in enumerate(ev):
    a.record(); plan.score(q, kr, v); b.record()
torch.cuda.synchronize()
print("back-to-back:", [round(a.elapsed_time(b), 2) for a, m, b in ev])
# with idle gaps between steps
ts = []
for i in range(10):
    time.sleep(0.2)
    a, m, b = ev[i]; a.record(); plan.score(q, kr, v); b.record(); torch.cuda.synchronize(); ts.append(round(a.elapsed_time(b), 2))
print("with 200ms idle gaps:", ts)
