"""CPU-side checks of the C ABI library: it loads, exports every symbol the header
declares, and its host-only validation mirrors CompressionConfig::validate
(proj/src/cache.cpp:12-28) and the engine's shape checks (engine.cpp:44-59)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ems_b200.h")


@pytest.fixture(scope="module")
def L():
    from paper_2412_08521_b200 import build, ems
    if not os.path.exists(ems.LIB_PATH):
        build.build()
    return ems.lib()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^EMS_API\s+[\w\s\*]+?\b(ems_\w+)\s*\(", text, flags=re.M)))


def test_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert len(syms) >= 12, syms
    for s in syms:
        assert hasattr(L, s), f"libems_b200.so does not export {s}"
    assert L.ems_abi_version() == 3


def _desc(**kw):
    from paper_2412_08521_b200 import ems
    import torch
    base = dict(B=1, Hq=4, Hkv=2, L=512, d=64, dtype=torch.bfloat16,
                cfg=ems.EmsConfig(n_budget=64, l_win=8, tau=0.6, gamma=4.0, kernel_size=7))
    base.update(kw)
    return ems.make_desc(base["B"], base["Hq"], base["Hkv"], base["L"], base["d"], base["dtype"], base["cfg"])


def test_validation_mirrors_reference(L):
    from paper_2412_08521_b200 import ems
    ok = _desc()
    assert L.ems_validate(C.byref(ok)) == 0
    assert L.ems_workspace_bytes(C.byref(ok)) > 0
    bad = [
        _desc(cfg=ems.EmsConfig(n_budget=8, l_win=8)),            # n_budget > l_win
        _desc(cfg=ems.EmsConfig(n_budget=8, l_win=0)),            # l_win > 0
        _desc(cfg=ems.EmsConfig(tau=1.5)),                        # tau in [0, 1]
        _desc(cfg=ems.EmsConfig(gamma=0.5)),                      # gamma >= 1
        _desc(cfg=ems.EmsConfig(kernel_size=4)),                  # odd kernel
        _desc(Hq=3, Hkv=2),                                       # GQA divisibility
        _desc(L=0),                                               # empty prompt
        _desc(d=80),                                              # unsupported head_dim
    ]
    for b in bad:
        assert L.ems_validate(C.byref(b)) == 1, b
        assert L.ems_workspace_bytes(C.byref(b)) == 0
    assert b"head_dim" in L.ems_last_error()


def test_cache_dims(L):
    from paper_2412_08521_b200 import ems
    d = _desc(B=2, Hkv=8, Hq=32, cfg=ems.EmsConfig(n_budget=256, l_win=32, gamma=4.0))
    dims = ems.CacheDims()
    assert L.ems_cache_dims_for(C.byref(d), C.byref(dims)) == 0
    assert (dims.units, dims.centers, dims.locals, dims.tbm, dims.lut) == (16, 224, 256, 768, 992)


def test_null_pointers_rejected_without_gpu(L):
    d = _desc()
    ws_bytes = L.ems_workspace_bytes(C.byref(d))
    rc = L.ems_prefill_compress(C.byref(d), None, None, None, None, None, None, None, None, None,
                                None, C.c_void_p(16), ws_bytes, None)
    assert rc == 1
    rc = L.ems_score(C.byref(d), None, None, None, None, None, None, None, None, 0, None)
    assert rc == 1 and b"workspace" in L.ems_last_error()
