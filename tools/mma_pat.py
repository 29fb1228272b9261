"""tcgen05.mma issue-pattern microbenchmark: MAC/clk/SM for 8-MMA patterns (see tc_selftest.cu)."""
import ctypes as C
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = C.CDLL(os.path.join(ROOT, "tests", "_build", "libems_selftest.so"))
L.ems_mma_pat.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]


def run(ts, n, d, a=(256,) * 8, same_b=0, it=4096):
    pat = (C.c_int * 19)(ts, n, *d, *a, same_b)
    cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
    assert L.ems_mma_pat(pat, 148, it, cyc.data_ptr()) == 0
    return 128 * n * 16 * it / cyc.double().median().item()


P = {
    "SS n128 d=0": (0, 128, [0] * 8),
    "SS n128 d=0,128 alt": (0, 128, [0, 128] * 4),
    "SS n128 d=0,256 alt": (0, 128, [0, 256] * 4),
    "SS n128 d=128,384 alt": (0, 128, [128, 384] * 4),
    "SS n128 d=0,128,256,384": (0, 128, [0, 128, 256, 384] * 2),
    "SS n128 d=0,256,128,384": (0, 128, [0, 256, 128, 384] * 2),
    "SS n128 d=0x4,128x4": (0, 128, [0] * 4 + [128] * 4),
    "SS n64 d=0": (0, 64, [0] * 8),
    "SS n64 d=0,64 alt": (0, 64, [0, 64] * 4),
    "SS n256 d=0": (0, 256, [0] * 8),
    "SS n256 d=0,256 alt": (0, 256, [0, 256] * 4),
    "SS n128 d=0,128 alt sameB": (0, 128, [0, 128] * 4, (256,) * 8, 1),
}
for name, args in P.items():
    print(f"{name:32s} {run(*args):8.0f}")
TS = {
    "TS n128 d=0 a=256": (1, 128, [0] * 8, [256 + 8 * k for k in range(8)]),
    "TS n128 d=0,128 alt a=256": (1, 128, [0, 128] * 4, [256 + 8 * k for k in range(8)]),
    "TS n128 d=256,384 alt a=0/128": (1, 128, [256, 384] * 4, [8 * (k // 2) + 128 * (k % 2) for k in range(8)]),
    "TS n128 d=0,256 alt a=128/384": (1, 128, [0, 256] * 4, [128 + 8 * (k // 2) + 256 * (k % 2) for k in range(8)]),
    "TS n128 d=256 a=0": (1, 128, [256] * 8, [8 * k for k in range(8)]),
    "TS n128 d=0,128 alt a=64/192 (P-in-S)": (1, 128, [256, 384] * 4, [8 * (k // 2) + 128 * (k % 2) + 0 for k in range(8)]),
}
for name, args in TS.items():
    print(f"{name:40s} {run(*args):8.0f}")
