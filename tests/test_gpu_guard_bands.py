"""Out-of-bounds write detection without compute-sanitizer (closed on this pool): every buffer the
C-ABI path writes -- outputs, glo/loc, LSE, the stage, the compressed cache, the workspace, the
decode state -- is a view into a larger allocation whose leading and trailing guard bands hold a
byte pattern; after the whole path runs on edge-case shapes (partial last tiles, odd G, merges,
zero class and explicit removal, keep-all, decode past graduation) every guard byte is intact."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200.inputs import CONFIGS, make_unit_np  # noqa: E402

GUARD = 4096  # bytes on each side
PAT = 0xA5


class Guarded:
    def __init__(self):
        self.blocks = []

    def like(self, t: torch.Tensor) -> torch.Tensor:
        """A tensor with t's shape/dtype/contents inside a guarded byte buffer."""
        nb = t.numel() * t.element_size()
        raw = torch.full((GUARD + nb + 15 + GUARD,), PAT, dtype=torch.uint8, device=t.device)
        pad = (-raw.data_ptr() - GUARD) % 16  # keep the payload 16-byte aligned
        body = raw[GUARD + pad: GUARD + pad + nb].view(t.dtype).view(t.shape)
        body.copy_(t)
        self.blocks.append((raw, GUARD + pad, nb))
        return body

    def check(self):
        for raw, off, nb in self.blocks:
            h = raw.cpu().numpy()
            lead, trail = h[:off], h[off + nb:]
            assert np.all(lead == PAT) and np.all(trail == PAT), f"guard band overwritten ({nb}-byte buffer)"


def guard_plan(plan: ems.Plan, g: Guarded):
    for d in (plan.cache, plan.stage):
        for k in list(d):
            d[k] = g.like(d[k])
    plan.glo, plan.loc = g.like(plan.glo), g.like(plan.loc)
    if plan.out is not None:
        plan.out = g.like(plan.out)
    if plan.lse is not None:
        plan.lse = g.like(plan.lse)
    plan.workspace = g.like(plan.workspace)
    plan._cstage = ems.CStage(*[ems._p(plan.stage[f]) for f, _ in ems.CStage._fields_])
    plan._ccache = ems.CCache(*[ems._p(plan.cache[f]) for f, _ in ems.CCache._fields_])


CASES = [  # workload, L, units, budget, zero_class, G override
    ("cfgM", 1000, 2, 256, True, None),
    ("cfgM", 777, 3, 128, False, None),
    ("cfg3", 1030, 2, 256, True, None),
    ("cfg3", 900, 1, 64, True, 3),
    ("cfg1", 300, 2, 128, True, None),
    ("cfgM", 200, 2, 256, True, None),  # keep-all (L <= budget)
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}_L{c[1]}_b{c[3]}" for c in CASES])
def test_prefill_writes_stay_in_bounds(case):
    wname, L, U, budget, zc, G = case
    w = CONFIGS[wname]
    if G:
        w = w.with_(heads_q=G * w.heads_kv)
    units = [make_unit_np(w, seed=11, seq_len=L, unit=u) for u in range(U)]
    dt = torch.float32 if w.dtype == "f32" else torch.bfloat16
    dev = torch.device("cuda")
    g = Guarded()
    t = lambda a: g.like(torch.tensor(np.stack(a), dtype=torch.float64).to(dt).to(dev))  # noqa: E731
    Gq, d = units[0].q_rot.shape[0], units[0].q_rot.shape[2]
    q = t([u.q_rot for u in units]).reshape(1, U * Gq, L, d)
    kr = t([u.k_rot for u in units]).reshape(1, U, L, d)
    kw = t([u.k_raw for u in units]).reshape(1, U, L, d)
    v = t([u.v for u in units]).reshape(1, U, L, d)
    cfg = ems.EmsConfig(budget, w.l_win, w.tau, w.gamma, w.kernel_size, zc)
    plan = ems.Plan(1, U * Gq, U, L, d, dt, cfg, dev, want_out=True, want_lse=True)
    guard_plan(plan, g)
    plan.workspace[:256].zero_()
    plan.run(q, kr, kw, v)
    plan.sync_status()
    torch.cuda.synchronize()
    g.check()


def test_decode_writes_stay_in_bounds():
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(5)
    n, d, G, steps = 500, 128, 4, 40
    q = torch.randn((1, 2 * G, n, d), generator=gen, device=dev).to(torch.bfloat16)
    k = torch.randn((1, 2, n, d), generator=gen, device=dev).to(torch.bfloat16)
    v = torch.randn((1, 2, n, d), generator=gen, device=dev).to(torch.bfloat16)
    cfg = ems.EmsConfig(64, 8, 0.3, 2.0, 5)
    plan = ems.prefill(q, k, v, cfg, 1e4)
    ds = ems.DecodeState(1, 2 * G, 2, n, d, torch.bfloat16, cfg, 1e4, n + steps)
    g = Guarded()
    for key in list(ds.state):
        ds.state[key] = g.like(ds.state[key])
    ds._c = ems.CDecode(*[ems._p(ds.state[f]) for f in ems.DECODE_FIELDS])
    ds.workspace = g.like(ds.workspace)
    ds.out, ds.argmax = g.like(ds.out), g.like(ds.argmax)
    ds.init_from_plan(plan)
    for _ in range(steps):
        ds.step(torch.randn((1, 2 * G, d), generator=gen, device=dev).to(torch.bfloat16),
                torch.randn((1, 2, d), generator=gen, device=dev).to(torch.bfloat16),
                torch.randn((1, 2, d), generator=gen, device=dev).to(torch.bfloat16))
    ds.sync_status()
    torch.cuda.synchronize()
    g.check()
