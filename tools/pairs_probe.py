"""P1 / P2 kernel times at equal attention FLOPs and growing work-item counts (G = 4, 8 KV heads:
B x L = 1 x 32768, 4 x 16384, 16 x 8192, 64 x 4096): separates per-item overhead from the
per-key-tile loop (the measurement behind the persistent P1).  python tools/pairs_probe.py"""
import torch, json, sys
sys.path.insert(0, '/root/repo')
from paper_2412_08521_b200 import ems
from torch.profiler import ProfilerActivity, profile
dev = torch.device('cuda')
for (B, L) in [(1, 32768), (4, 16384), (16, 8192), (64, 4096)]:
    Hq, Hkv, d = 32, 8, 128
    g = torch.Generator(device=dev).manual_seed(1)
    q = torch.randn(B, Hq, L, d, device=dev, generator=g).bfloat16()
    k = torch.randn(B, Hkv, L, d, device=dev, generator=g).bfloat16()
    v = torch.randn(B, Hkv, L, d, device=dev, generator=g).bfloat16()
    plan = ems.Plan(B, Hq, Hkv, L, d, q.dtype, ems.EmsConfig(256, 32, 0.6, 4.0), dev, "tcgen05", want_out=True)
    for _ in range(3): plan.score(q, k, v)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5): plan.score(q, k, v)
        torch.cuda.synchronize()
    kern = {}
    for e in prof.key_averages():
        if e.device_time_total > 0 and ("fwd2" in e.key or "colsum_tc" in e.key):
            kern["P1" if "fwd2" in e.key else "P2"] = round(e.device_time_total / e.count / 1e3, 3)
    nT = L // 128
    pairs = B * Hkv * (4 * nT // 2)
    print(json.dumps({"B": B, "L": L, "pairs": pairs, **kern}), flush=True)
    del q, k, v, plan
    torch.cuda.empty_cache()
