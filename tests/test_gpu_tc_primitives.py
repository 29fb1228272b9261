"""tcgen05 / TMA / descriptor primitives (csrc/tc.cuh) against torch fp32 matmuls.

One 128x128x128 bf16 MMA per mode: SS with K-major or MN-major B, and TS with A
staged in TMEM.  Exactness: bf16 products are exact in fp32, so the only error is
fp32 accumulation order (<= 1e-5 relative here)."""
import ctypes as C
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libems_selftest.so")


@pytest.fixture(scope="module")
def st():
    if not os.path.exists(LIB):
        from paper_2412_08521_b200 import build
        build.build_selftest()
    L = C.CDLL(LIB)
    L.ems_tc_selftest.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    return L


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_mma_modes(st, mode):
    g = torch.Generator(device="cuda").manual_seed(mode)
    A = torch.randn(128, 128, generator=g, device="cuda").bfloat16()
    B = torch.randn(128, 128, generator=g, device="cuda").bfloat16()
    D = torch.zeros(128, 128, device="cuda")
    assert st.ems_tc_selftest(mode, A.data_ptr(), B.data_ptr(), D.data_ptr()) == 0
    want = A.float() @ (B.float() if mode & 1 else B.float().t())
    err = (D - want).abs().max().item() / want.abs().max().item()
    assert err < 1e-5, f"mode {mode}: rel err {err}"


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_mma_2sm(st, mode):
    """cta_group::2: M = 256 over a CTA pair, N = 256 (mode & 2 == 0) or 128; TS when mode & 1."""
    st.ems_tc_selftest2.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    N = 128 if mode & 2 else 256
    g = torch.Generator(device="cuda").manual_seed(10 + mode)
    A = torch.randn(256, 128, generator=g, device="cuda").bfloat16()
    B = torch.randn(N, 128, generator=g, device="cuda").bfloat16()
    D = torch.zeros(256, N, device="cuda")
    assert st.ems_tc_selftest2(mode, A.data_ptr(), B.data_ptr(), D.data_ptr()) == 0
    want = A.float() @ B.float().t()
    err = (D - want).abs().max().item() / want.abs().max().item()
    assert err < 1e-5, f"mode {mode}: rel err {err}"
