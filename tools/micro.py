"""Microbenchmarks of the per-SM pipes the score kernels lean on (one CTA per SM):
TMEM load bandwidth, MUFU.EX2, FFMA, FFMA2 and the polynomial exp2 throughput."""
import ctypes as C
import json
import os
import sys

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
for threads in (128, 256, 512):
    w = threads // 32
    it = 4096
    c = run(0, threads, it)
    res[f"tmem_ld_x32_wait_each_{w}w_B_per_clk"] = w * it * 32 * 32 * 4 / c
    c = run(1, threads, it)
    res[f"tmem_ld_4x32_then_wait_{w}w_B_per_clk"] = w * it * 32 * 32 * 4 / c
    c = run(2, threads, it)
    res[f"mufu_ex2_{w}w_per_clk"] = w * 32 * it * 8 / c
    c = run(3, threads, it)
    res[f"ffma_{w}w_per_clk"] = w * 32 * it * 8 / c
    c = run(4, threads, it)
    res[f"ffma2_{w}w_elem_per_clk"] = w * 32 * it * 8 / c
    c = run(5, threads, 1024)
    res[f"poly_exp2_{w}w_elem_per_clk"] = w * 32 * 1024 * 8 / c
print(json.dumps(res, indent=1))

shapes = {10: "32x32b.x32 x2", 11: "16x64b.x32 x2", 12: "16x128b.x16 x2", 13: "16x256b.x8 x2", 14: "32x32b.x64"}
res2 = {}
for threads in (128, 256, 512):
    w = threads // 32
    for kind, name in shapes.items():
        c = run(kind, threads, 4096)
        res2[f"{name} {w}w B/clk"] = w * 4096 * 32 * 32 * 4 / c
print(json.dumps(res2, indent=1))

L.ems_mma_micro.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p]
res3 = {}
for kind, (name, n) in {0: ("SS 128x128", 128), 1: ("TS 128x128", 128), 2: ("SS 128x256", 256),
                        3: ("SS 128x128 B MN-major", 128)}.items():
    cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
    it = 4096
    assert L.ems_mma_micro(kind, 148, it, cyc.data_ptr()) == 0
    c = cyc.double().median().item()
    res3[name + " MAC/clk/SM"] = 128 * n * 16 * it / c
print(json.dumps(res3, indent=1))

L.ems_mma2_micro.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p]
res4 = {}
for kind, (name, n) in {0: ("2SM SS 256x128", 128), 1: ("2SM TS 256x128", 128), 2: ("2SM SS 256x256", 256)}.items():
    cyc = torch.zeros(74, dtype=torch.int64, device="cuda")
    it = 4096
    rc = L.ems_mma2_micro(kind, 74, it, cyc.data_ptr())
    if rc:
        res4[name] = f"rc={rc}"
        continue
    c = cyc.double().median().item()
    res4[name + " MAC/clk/SM"] = 256 * n * 16 * it / c / 2
print(json.dumps(res4, indent=1))

res5 = {}
for kind, (name, n) in {4: ("SS 128x128 pre-desc", 128), 5: ("TS 128x128 pre-desc", 128), 6: ("SS 128x256 pre-desc", 256),
                        7: ("SS 128x128 2 accumulators alternating", 128), 8: ("TS 128x128 2 accumulators alternating", 128),
                        9: ("SS 128x128 4 accumulators rotating", 128)}.items():
    cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
    it = 4096
    assert L.ems_mma_micro(kind, 148, it, cyc.data_ptr()) == 0
    c = cyc.double().median().item()
    res5[name + " MAC/clk/SM"] = 128 * n * 16 * it / c
print(json.dumps(res5, indent=1))

L.ems_epi_micro.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
res6 = {}
for poly in (0, 2, 3, 4):
    for dbl in (0, 1):
        cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
        sink = torch.zeros(1024, device="cuda")
        it = 2048
        assert L.ems_epi_micro(poly, dbl, 148, it, cyc.data_ptr(), sink.data_ptr()) == 0
        res6[f"P2 epilogue poly={poly} double={dbl} elem/clk/SM"] = 512 * 64 * it / cyc.double().median().item()
print(json.dumps(res6, indent=1))
