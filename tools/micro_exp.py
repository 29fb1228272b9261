"""Packed exp2 throughput (MUFU f16x2 / bf16x2) next to fp32 ex2, per SM per clock."""
import ctypes as C
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = C.CDLL(os.path.join(ROOT, "tests", "_build", "libems_selftest.so"))
L.ems_micro.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]


def run(kind, threads, iters, blocks=148):
    cyc = torch.zeros(blocks, dtype=torch.int64, device="cuda")
    sink = torch.zeros(1024, device="cuda")
    assert L.ems_micro(kind, threads, blocks, iters, cyc.data_ptr(), sink.data_ptr()) == 0
    return cyc.double().median().item()


res = {}
for threads in (256, 512):
    w = threads // 32
    res[f"ex2_f32_{w}w"] = w * 32 * 4096 * 8 / run(2, threads, 4096)
    res[f"ex2_f16x2_{w}w_elem"] = 2 * w * 32 * 4096 * 8 / run(6, threads, 4096)
    res[f"ex2_bf16x2_{w}w_elem"] = 2 * w * 32 * 4096 * 8 / run(7, threads, 4096)
print(json.dumps(res, indent=1))
