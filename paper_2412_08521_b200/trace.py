"""KVTR traces and the experiment report on the GPU path.

* ``load_trace`` / ``save_trace`` restate the reference's KVTR v1 reader and writer
  (proj/src/trace.cpp:20-179): magic "KVTR", u32 version = 1, u32 num_heads, u32 head_dim,
  u32 step_count, then per step u8 kind (0 prefill, 1 decode), u32 token_count and the Q, K, V
  blocks as [tokens][heads][dim] little-endian float32.  Malformed files raise ``FormatError``
  with the byte offset the reference reports (bad magic 0, bad version 4, truncation at the
  read position, non-finite payload at the row start); a trace must be one prefill step then
  single-token decode steps (Trace::validate, :101-114).
* ``run_experiment`` is run_experiment_multi (proj/src/experiment.cpp:152-264) for any list of
  policies (ems, full, streaming, h2o, snapkv) with the compressed engine on the GPU (device RoPE + prefill + the device decode loop)
  and the dense full-cache reference run (run_reference, :42-80) as plain fp64 tensor math on
  the same device (report infrastructure, not the accelerated path).  ``report_json`` /
  ``report_csv`` emit the reference's schema (report_json :271-326, report_csv :328-344).
"""
from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field

import numpy as np

MAGIC = b"KVTR"
VERSION = 1


class FormatError(ValueError):
    """ems::FormatError (proj/include/ems/errors.hpp:18-30): malformed trace, with byte offset."""

    def __init__(self, msg: str, offset: int):
        super().__init__(f"{msg} (offset {offset})")
        self.offset = offset


@dataclass
class TraceStep:
    kind: int          # 0 prefill, 1 decode
    q: np.ndarray      # [heads][tokens][dim] float64 holding float32 values
    k: np.ndarray
    v: np.ndarray

    @property
    def tokens(self) -> int:
        return self.q.shape[1]


@dataclass
class Trace:
    num_heads: int
    head_dim: int
    steps: list = field(default_factory=list)

    @property
    def prefill_tokens(self) -> int:
        return self.steps[0].tokens if self.steps else 0

    @property
    def decode_steps(self) -> int:
        return max(len(self.steps) - 1, 0)

    def validate(self) -> None:  # Trace::validate, trace.cpp:101-114
        if not self.steps or self.steps[0].kind != 0:
            raise FormatError("trace must start with a prefill step", 0)
        for s in self.steps[1:]:
            if s.kind != 1:
                raise FormatError("trace has more than one prefill step", 0)
            if s.tokens != 1:
                raise FormatError("decode steps must carry exactly one token", 0)

    def stacked(self):
        """q, k, v as [heads][prefill + decode tokens][dim] (prompt rows, then one row per step)."""
        cat = lambda name: np.concatenate([getattr(s, name) for s in self.steps], axis=1)  # noqa: E731
        return cat("q"), cat("k"), cat("v")


def load_trace(path: str) -> Trace:
    """load_trace, proj/src/trace.cpp:119-155."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise FormatError("cannot open trace file: " + path, 0) from None
    off = 0

    def take(n: int, what: str) -> bytes:
        nonlocal off
        if n > len(data) - off:
            raise FormatError(f"truncated trace while reading {what}", off)
        b = data[off:off + n]
        off += n
        return b

    if take(4, "magic") != MAGIC:
        raise FormatError("bad magic, expected KVTR", 0)
    version = struct.unpack("<I", take(4, "version"))[0]
    if version != VERSION:
        raise FormatError(f"unsupported KVTR version {version}", 4)
    heads = struct.unpack("<I", take(4, "num_heads"))[0]
    dim = struct.unpack("<I", take(4, "head_dim"))[0]
    n_steps = struct.unpack("<I", take(4, "step_count"))[0]
    if heads == 0 or dim == 0:
        raise FormatError("num_heads and head_dim must be positive", 8)
    tr = Trace(heads, dim)
    for _ in range(n_steps):
        kind = take(1, "step kind")[0]
        if kind > 1:
            raise FormatError(f"bad step kind {kind}", off - 1)
        tokens = struct.unpack("<I", take(4, "token_count"))[0]
        if tokens == 0:
            raise FormatError("step with zero tokens", off - 4)
        blocks = []
        for what in ("Q block", "K block", "V block"):
            n = tokens * heads * dim * 4
            if n > len(data) - off:
                raise FormatError(f"trace too short for {what}", off)
            a = np.frombuffer(data, dtype="<f4", count=tokens * heads * dim, offset=off).reshape(tokens, heads, dim)
            bad = ~np.isfinite(a).all(axis=(1, 2))
            if bad.any():
                row = int(np.argmax(bad))
                raise FormatError(f"non-finite value in {what}", off + row * heads * dim * 4)
            off += n
            blocks.append(np.ascontiguousarray(a.transpose(1, 0, 2)).astype(np.float64))
        tr.steps.append(TraceStep(kind, *blocks))
    tr.validate()
    return tr


def save_trace(tr: Trace, path: str) -> None:
    """save_trace, proj/src/trace.cpp:157-179 (values written as float32)."""
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<4I", VERSION, tr.num_heads, tr.head_dim, len(tr.steps)))
        for s in tr.steps:
            f.write(struct.pack("<BI", s.kind, s.tokens))
            for a in (s.q, s.k, s.v):
                f.write(np.ascontiguousarray(np.asarray(a, dtype="<f4").transpose(1, 0, 2)).tobytes())


# ---------------------------------------------------------------------------------------
def _dense_reference(q, k, v, n, base, device):
    """run_reference (experiment.cpp:42-80): dense causal prefill + full-cache decode, fp64."""
    import torch

    from paper_2412_08521_b200.inputs import rope_np
    H, T, d = q.shape
    qr = torch.tensor(rope_np(q, base), dtype=torch.float64, device=device)
    kr = torch.tensor(rope_np(k, base), dtype=torch.float64, device=device)
    vv = torch.tensor(v, dtype=torch.float64, device=device)
    scale = 1.0 / math.sqrt(d)
    s = (qr[:, :n] @ kr[:, :n].transpose(1, 2)) * scale
    s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool, device=device), 1), float("-inf"))
    pre = torch.softmax(s, dim=-1) @ vv[:, :n]
    outs, ams = [], []
    for st in range(T - n):
        row = n + st
        lg = (kr[:, :row + 1] @ qr[:, row, :, None])[..., 0] * scale
        p = torch.softmax(lg, dim=-1)
        outs.append((p[:, None, :] @ vv[:, :row + 1])[:, 0])
        ams.append(torch.argmax(p, dim=-1))
    return pre, outs, ams


def _l2(a, b) -> float:  # concat_l2, experiment.cpp:86-95
    return float(((a - b) ** 2).sum().sqrt())


def _cos_error(a, b) -> float:  # concat_cos_error, experiment.cpp:97-120
    if bool((a == b).all()):
        return 0.0
    num, na, nb = float((a * b).sum()), float((a * a).sum()), float((b * b).sum())
    if na == 0.0 or nb == 0.0:
        return 1.0
    return max(0.0, 1.0 - min(max(num / (math.sqrt(na) * math.sqrt(nb)), -1.0), 1.0))


def run_experiment(tr: Trace, cfg, label: str = "", needle_pos: int | None = None, rope_base: float = 10000.0,
                   device="cuda", policies=None, compute_diagnostics: bool = True) -> dict:
    """run_experiment_multi (experiment.cpp:152-264): the compressed engine on the GPU, once per
    policy (``policies`` = policy names, default ``[cfg.policy]``), against one dense run."""
    import dataclasses

    import torch

    from paper_2412_08521_b200 import ems
    tr.validate()
    q, k, v = tr.stacked()
    H, T, d = q.shape
    n = tr.prefill_tokens
    ref_pre, ref_outs, ref_am = _dense_reference(q, k, v, n, rope_base, device)
    t = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float32, device=device)  # noqa: E731
    diags = []
    if compute_diagnostics:  # analyze_trace (experiment.cpp:133-150) on the prompt
        sp, rd = ems.analyze(t(q[None, :, :n]), t(k[None, :, :n]), t(v[None, :, :n]), cfg, rope_base)
        diags = [dict(head=h, sparsity=float(sp[0, h]), redundancy=float(rd[0, h])) for h in range(H)]
    reports = []
    for pol in (policies or [cfg.policy]):
        pc = dataclasses.replace(cfg, policy=pol)
        plan = ems.prefill(t(q[None, :, :n]), t(k[None, :, :n]), t(v[None, :, :n]), pc, rope_base)
        ds = ems.DecodeState(1, H, H, n, d, torch.float32, pc, rope_base, T + 1, device=device)
        ds.init_from_plan(plan)

        def accounting():  # stored_entries / bytes_stored per head (cache.hpp:92-99, cache.cpp:40-46)
            meta = ds.state["meta"].cpu().numpy()
            e = meta[:, 1] + meta[:, 5]
            return int(e.sum()), int((8 * (2 * e * d + 4 * e + meta[:, 2])).sum())

        steps = []
        e0, b0 = accounting()
        pre = plan.out[0].double()
        steps.append(dict(step=0, l2_error=_l2(pre, ref_pre), cos_error=_cos_error(pre, ref_pre), entries=e0,
                          bytes=b0, argmax_match=True))
        retained = True
        for s in range(T - n):
            o, am = ds.step(t(q[None, :, n + s]), t(k[None, :, n + s]), t(v[None, :, n + s]))
            out = o[0].double()
            match = bool((am[0].long() == ref_am[s]).all())
            e, b = accounting()
            steps.append(dict(step=s + 1, l2_error=_l2(out, ref_outs[s]), cos_error=_cos_error(out, ref_outs[s]),
                              entries=e, bytes=b, argmax_match=match))
            retained = retained and match
        dec = steps[1:]
        agg = dict(mean_l2=float(np.mean([m["l2_error"] for m in dec])) if dec else 0.0,
                   max_l2=float(max([m["l2_error"] for m in dec], default=0.0)),
                   mean_cos_error=float(np.mean([m["cos_error"] for m in dec])) if dec else 0.0,
                   argmax_match_rate=float(np.mean([m["argmax_match"] for m in dec])) if dec else 1.0)
        needle = None
        if needle_pos is not None:
            in_lut = all(_position_represented(ds.unit_cache(h), needle_pos) for h in range(H))
            needle = dict(position=int(needle_pos), retained=retained and bool(dec), in_lut_final=in_lut)
        reports.append(dict(policy=pol, compression_applied=bool(plan.cache["counts"][0, 3].item()), steps=steps,
                            aggregate=agg, needle=needle, diagnostics=diags))
    return {"schema_version": 1,
            "trace": dict(label=label, num_heads=H, head_dim=d, prefill_tokens=n, decode_steps=T - n),
            "config": dict(n_budget=cfg.n_budget, l_win=cfg.l_win, tau=cfg.tau, gamma=cfg.gamma, zeta=cfg.zeta,
                           kernel_size=cfg.kernel_size, position_mode=cfg.position_mode,
                           eviction="zero_class" if cfg.zero_class else "explicit_removal"),
            "policies": reports}


def _position_represented(c: dict, pos: int) -> bool:  # HeadCacheState::position_represented, cache.cpp:82-94
    hit = np.nonzero(c["lut_position"] == pos)[0]
    if len(hit):
        return bool(c["lut_slot"][hit[0]] != -1)
    return bool((c["local_position"] == pos).any() or (c["position"] == pos).any())


def report_json(report: dict) -> str:
    return json.dumps(report, indent=2) + "\n"


def report_csv(report: dict) -> str:  # experiment.cpp:328-344
    out = "policy,step,l2_error,cos_error,entries,bytes,argmax_match\n"
    for pr in report["policies"]:
        for m in pr["steps"]:
            out += (f"{pr['policy']},{m['step']},{m['l2_error']!r},{m['cos_error']!r},{m['entries']},{m['bytes']},"
                    f"{int(m['argmax_match'])}\n")
    return out
