"""Device RoPE and the raw-input prefill entry point (ems_prefill).

* ems_rope restates detail::rotate (proj/src/rope.cpp:10-28) in fp64 and rounds once, so it
  must agree with the fp64 numpy restatement (inputs.rope_np + round_to) bit for bit, except
  for libm last-ulp differences that can move a value across a rounding boundary (rare).
* ems_prefill = engine::prefill (proj/src/engine.cpp:42-82): RoPE on the device, then the
  whole path with the raw K for the merge.  Checked against the reference's golden fixture
  and against ems_prefill_compress on host-rotated inputs (identical caches expected).
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.oracle import Cache  # noqa: E402
from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200.inputs import CONFIGS, rope_np, round_to  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _tdt(dtype):
    return torch.float32 if dtype == "f32" else torch.bfloat16


@pytest.mark.parametrize("dtype,L,d,base,first", [("bf16", 4096, 128, 5e5, 0), ("bf16", 1000, 64, 1e4, 7),
                                                  ("f32", 513, 8, 1e4, 0), ("f32", 2048, 128, 1e4, 3)])
def test_rope_matches_fp64_restatement(dtype, L, d, base, first):
    rng = np.random.default_rng(11)
    x = round_to(rng.standard_normal((3, L, d)) * 2.0, dtype)
    want = round_to(rope_np(x, base, first_position=first), dtype)
    xt = torch.tensor(x).to(_tdt(dtype)).cuda()
    got = ems.rope(xt, base, first_position=first).double().cpu().numpy()
    diff = got != want
    assert diff.mean() < 1e-5, f"{diff.sum()} of {diff.size} elements differ"
    if diff.any():  # at most one unit in the last place of the storage dtype
        ulp = np.abs(want[diff]) * (2.0 ** -7 if dtype == "bf16" else 2.0 ** -23)
        assert np.all(np.abs(got[diff] - want[diff]) <= ulp * 1.01)
    # in place
    y = xt.clone()
    ems.rope(y, base, first_position=first, out=y)
    assert torch.equal(y, ems.rope(xt, base, first_position=first))


def test_rope_rejects_bad_arguments():
    x = torch.zeros((1, 16, 8), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ems.InvalidArgument):
        ems.rope(x, 1e4, first_position=-1)  # apply_rope: position must be nonnegative
    with pytest.raises(ems.InvalidArgument):
        ems.rope(torch.zeros((1, 16, 7), dtype=torch.bfloat16, device="cuda"), 1e4)  # odd head_dim
    with pytest.raises(ems.InvalidArgument):
        ems.rope(x, 0.0)


def test_prefill_raw_golden_fixture():
    """The reference's golden cache (proj/tests/fixtures/golden_cache.json) from RAW inputs:
    the engine's own RoPE (base 1e4) now runs on the device."""
    tr = np.load(os.path.join(GOLDEN, "golden_trace.npz"))
    with open(os.path.join(GOLDEN, "golden_cache.json")) as f:
        want = Cache.from_dump_json(f.read())
    dev = torch.device("cuda")
    t = lambda a: torch.tensor(np.asarray(a)[None], dtype=torch.float32, device=dev).contiguous()  # noqa: E731
    q, k, v = t(tr["q"]), t(tr["k"]), t(tr["v"])  # [1][2][16][8]
    cfg = ems.EmsConfig(n_budget=12, l_win=4, tau=0.6, gamma=2.0, kernel_size=3)
    plan = ems.prefill(q, k, v, cfg, rope_base=1e4)
    got = plan.unit_cache(0)
    np.testing.assert_array_equal(got["position"], want.position)
    np.testing.assert_array_equal(got["lut_position"], want.lut_position)
    np.testing.assert_array_equal(got["lut_slot"], want.lut_slot)
    np.testing.assert_allclose(got["unit_key"], want.unit_key, rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(got["score"], want.score, rtol=1e-4, atol=1e-7)


@pytest.mark.parametrize("wname,L", [("cfg3", 4096), ("cfgM", 2048)])
def test_prefill_raw_equals_prerotated_path(wname, L):
    """ems_prefill(raw): device RoPE agrees with the host fp64 rotation, and the rest of the
    path equals ems_prefill_compress on those rotated tensors bit for bit."""
    w = CONFIGS[wname]
    base = w.rope_base or 1e4
    rng = np.random.default_rng(21)
    G, H = w.group, 2
    q = round_to(rng.standard_normal((H * G, L, 128)), "bf16")
    k = round_to(rng.standard_normal((H, L, 128)), "bf16")
    v = round_to(rng.standard_normal((H, L, 128)), "bf16")
    dev = torch.device("cuda")
    T = lambda a: torch.tensor(a[None]).to(torch.bfloat16).to(dev).contiguous()  # noqa: E731
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
    a = ems.prefill(T(q), T(k), T(v), cfg, rope_base=base)
    qr = T(round_to(rope_np(q, base), "bf16"))
    kr = T(round_to(rope_np(k, base), "bf16"))
    assert (a.q_rot != qr).float().mean().item() < 1e-6 and (a.k_rot != kr).float().mean().item() < 1e-6
    b = ems.prefill_compress(a.q_rot.clone(), a.k_rot.clone(), T(k), T(v), cfg)
    torch.cuda.synchronize()
    assert torch.equal(a.glo, b.glo) and torch.equal(a.loc, b.loc)
    for key in a.cache:
        assert torch.equal(a.cache[key], b.cache[key]), key
