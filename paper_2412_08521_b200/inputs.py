"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference has no public benchmark or dataset on this path; BASELINE.json's
five configs (plus SURVEY.md's merge-parity config M) are synthetic.  This
module builds them with the shapes and value distributions BASELINE.json
states.  Two implementations share one recipe:

* numpy (fp64, then rounded once to the config dtype) -- small/medium sizes,
  used by the parity tests so that the oracle and the CUDA path see identical
  bits;
* torch on the device -- full bench sizes (up to 64 x 131072 x 128), where a
  host generator would dominate the run time.

RoPE (contract D3) is the reference's interleaved-pair rotation
(proj/src/rope.cpp:17-26): pair (2i, 2i+1) at position p is rotated by
p * base^(-2i/d).  Q_rot/K_rot are computed in fp64 (numpy) or fp32 (torch)
and rounded once to the dtype; raw K (pre-RoPE) feeds the merge.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    batch: int
    heads_q: int
    heads_kv: int
    head_dim: int
    seq_len: int
    dtype: str            # "f32" | "bf16"
    rope_base: float | None
    l_win: int
    n_budget: int
    gamma: float
    tau: float
    kernel_size: int = 7
    layers: int = 1
    spans: int = 0        # planted retrieval spans
    span_len: int = 0
    rank_k: tuple = ()    # per-KV-head rank choices for low-rank K (config 4)
    redundant: bool = False
    notes: str = ""

    @property
    def group(self) -> int:
        return self.heads_q // self.heads_kv

    @property
    def units(self) -> int:
        return self.batch * self.heads_kv * self.layers

    def with_(self, **kw) -> "Workload":
        d = dict(self.__dict__)
        d.update(kw)
        return Workload(**d)


# BASELINE.json "configs", in order; D-numbers are SURVEY.md section 8 contract decisions.
CONFIGS = {
    "cfg1": Workload("cfg1", 1, 8, 8, 64, 1024, "f32", None, 32, 128, 1.5, 0.5,
                     notes="gamma=1.5 per D4 (192 = gamma*budget, 64 = tbm target)"),
    "cfg2": Workload("cfg2", 4, 32, 32, 128, 4096, "bf16", 1e4, 32, 256, 4.0, 0.5),
    "cfg3": Workload("cfg3", 1, 32, 8, 128, 32768, "bf16", 5e5, 32, 256, 4.0, 0.6,
                     spans=1, span_len=64, notes="budget 256 (headline); tau/gamma per D5"),
    "cfg3b": Workload("cfg3b", 1, 32, 8, 128, 32768, "bf16", 5e5, 32, 1024, 4.0, 0.6,
                      spans=1, span_len=64, notes="config 3 at budget 1024"),
    "cfg4": Workload("cfg4", 1, 32, 8, 128, 8192, "bf16", 1e4, 32, 256, 4.0, 0.6, layers=32,
                     rank_k=(4, 16, 64, 128), notes="B in {1,8,32}; rank-r K per D8"),
    "cfg5": Workload("cfg5", 1, 64, 8, 128, 131072, "bf16", 5e5, 64, 2560, 4.0, 0.6,
                     spans=4, span_len=32, notes="spans built as config 3 (D6)"),
    "cfgM": Workload("cfgM", 1, 8, 8, 128, 4096, "bf16", 1e4, 32, 256, 4.0, 0.6, redundant=True,
                     notes="merge-parity input (SURVEY.md 8d), reference redundant recipe"),
}


# -- numerics helpers ----------------------------------------------------------------
def round_to(x, dtype: str) -> np.ndarray:
    """Round fp64 values once to f32 or bf16 (round-to-nearest-even); return fp64."""
    x32 = np.ascontiguousarray(x, dtype=np.float32)
    if dtype == "f32":
        return x32.astype(np.float64)
    if dtype != "bf16":
        raise ValueError(dtype)
    u = x32.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def rope_np(x: np.ndarray, base: float, first_position: float = 0.0, sign: float = 1.0) -> np.ndarray:
    """Interleaved-pair RoPE over the token axis (-2) of [..., n, d] (rope.cpp:17-26).
    sign=-1 undoes the rotation (detail::rotate with negative positions)."""
    n, d = x.shape[-2], x.shape[-1]
    pos = (first_position + np.arange(n, dtype=np.float64))[:, None] * sign
    freq = np.power(base, -np.arange(0, d, 2, dtype=np.float64) / d)[None, :]
    ang = pos * freq
    c, s = np.cos(ang), np.sin(ang)
    a0, a1 = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x, dtype=np.float64)
    out[..., 0::2] = a0 * c - a1 * s
    out[..., 1::2] = a0 * s + a1 * c
    return out


@dataclass
class UnitInputs:
    """One KV unit in fp64 holding dtype-exact values."""
    q_rot: np.ndarray  # [G, n, d]
    k_rot: np.ndarray  # [n, d]
    k_raw: np.ndarray  # [n, d]
    v: np.ndarray      # [n, d]
    meta: dict = field(default_factory=dict)


def _redundant_kv(rng, n, d, level=0.8, perturb=0.05):
    """Restates gen_redundant's recipe (proj/src/trace.cpp:265-331) with numpy's RNG:
    ceil(level*n)+1 randomly chosen tokens (never token 0) are perturbed copies of an
    earlier base token; base tokens are fresh N(0,1) keys and values."""
    copies = min(n - 1, int(np.ceil(level * n)) + 1)
    is_copy = np.zeros(n, dtype=bool)
    is_copy[1 + rng.permutation(n - 1)[:copies]] = True
    k = np.empty((n, d))
    v = np.empty((n, d))
    bases = []
    for t in range(n):
        if is_copy[t] and bases:
            b = bases[rng.integers(len(bases))]
            k[t] = k[b] + perturb * rng.standard_normal(d)
            v[t] = v[b] + perturb * rng.standard_normal(d)
        else:
            k[t] = rng.standard_normal(d)
            v[t] = rng.standard_normal(d)
            bases.append(t)
    return k, v


def make_unit_np(w: Workload, seed: int, seq_len: int | None = None, unit: int = 0) -> UnitInputs:
    """Seeded numpy generator for one KV unit (used by parity tests)."""
    n = seq_len or w.seq_len
    d, G = w.head_dim, w.group
    rng = np.random.default_rng([seed, unit])
    q_raw = rng.standard_normal((G, n, d))
    if w.redundant:
        k_raw, v = _redundant_kv(rng, n, d)
    else:
        k_raw = rng.standard_normal((n, d))
        v = rng.standard_normal((n, d))
    if w.rank_k:
        r = w.rank_k[unit % len(w.rank_k)]
        u_ = rng.standard_normal((n, r))
        wm = rng.standard_normal((r, d))
        k_raw = u_ @ wm / np.sqrt(r) + 0.1 * rng.standard_normal((n, d))
    meta = {}
    if w.rope_base:
        q_rot = rope_np(q_raw, w.rope_base)
        k_rot = rope_np(k_raw, w.rope_base)
    else:
        q_rot, k_rot = q_raw, k_raw.copy()
    q_rot = round_to(q_rot, w.dtype)
    if w.spans:
        # planted retrieval span(s) in ROTATED key space:
        # 0.7*sqrt(d)*m/|m| + 0.3*N(0,1), m = mean of the group's last-32 rotated queries.
        m = q_rot[:, -32:, :].reshape(-1, d).mean(axis=0)
        target = 0.7 * np.sqrt(d) * m / np.linalg.norm(m)
        hi = max(1, n - w.l_win - w.span_len)
        starts = sorted(int(s) for s in rng.integers(0, hi, size=w.spans))
        for s in starts:
            k_rot[s:s + w.span_len] = target[None, :] + 0.3 * rng.standard_normal((w.span_len, d))
        if w.rope_base:
            k_raw = rope_np(k_rot, w.rope_base, sign=-1.0)
        else:
            k_raw = k_rot.copy()
        meta["span_starts"] = starts
    k_raw = round_to(k_raw, w.dtype)
    k_rot = round_to(k_rot if w.rope_base or w.spans else k_raw, w.dtype)
    v = round_to(v, w.dtype)
    return UnitInputs(q_rot=q_rot, k_rot=k_rot, k_raw=k_raw, v=v, meta=meta)


def make_batch_torch(w: Workload, seed: int, device, layer: int = 0):
    """Full-size device generator: returns (q_rot [B,Hq,L,d], k_rot, k_raw, v [B,Hkv,L,d])
    in the workload dtype.  Same recipe as make_unit_np, torch RNG (Philox) instead."""
    import torch

    dt = torch.float32 if w.dtype == "f32" else torch.bfloat16
    B, Hq, Hk, L, d, G = w.batch, w.heads_q, w.heads_kv, w.seq_len, w.head_dim, w.group
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1000003 + layer)
    q = torch.randn((B, Hq, L, d), generator=g, device=device, dtype=torch.float32)
    v = torch.randn((B, Hk, L, d), generator=g, device=device, dtype=torch.float32)
    if w.rank_k:
        ks = []
        for h in range(Hk):
            r = w.rank_k[(layer * Hk + h) % len(w.rank_k)]
            u_ = torch.randn((B, L, r), generator=g, device=device)
            wm = torch.randn((r, d), generator=g, device=device)
            ks.append(u_ @ wm / r ** 0.5 + 0.1 * torch.randn((B, L, d), generator=g, device=device))
        k = torch.stack(ks, dim=1)
    else:
        k = torch.randn((B, Hk, L, d), generator=g, device=device, dtype=torch.float32)

    def rope(x, sign=1.0):
        pos = torch.arange(L, device=device, dtype=torch.float64)[:, None] * sign
        freq = torch.pow(torch.tensor(w.rope_base, dtype=torch.float64, device=device),
                         -torch.arange(0, d, 2, device=device, dtype=torch.float64) / d)[None, :]
        ang = pos * freq
        c, s = torch.cos(ang).float(), torch.sin(ang).float()
        a0, a1 = x[..., 0::2], x[..., 1::2]
        out = torch.empty_like(x)
        out[..., 0::2] = a0 * c - a1 * s
        out[..., 1::2] = a0 * s + a1 * c
        return out

    if w.rope_base:
        q_rot, k_rot = rope(q), rope(k)
    else:
        q_rot, k_rot = q, k.clone()
    q_rot = q_rot.to(dt)
    if w.spans:
        qf = q_rot.float().view(B, Hk, G, L, d)[:, :, :, -32:, :].reshape(B, Hk, G * 32, d)
        m = qf.mean(dim=2)
        target = 0.7 * d ** 0.5 * m / m.norm(dim=-1, keepdim=True)
        hi = max(1, L - w.l_win - w.span_len)
        starts = torch.randint(0, hi, (w.spans,), generator=g, device=device).tolist()
        for s in sorted(starts):
            noise = 0.3 * torch.randn((B, Hk, w.span_len, d), generator=g, device=device)
            k_rot[:, :, s:s + w.span_len, :] = target[:, :, None, :] + noise
        k = rope(k_rot, -1.0) if w.rope_base else k_rot.clone()
    return q_rot.contiguous(), k_rot.to(dt).contiguous(), k.to(dt).contiguous(), v.to(dt).contiguous()
