"""Python front-end over the C ABI (include/ems_b200.h) of libems_b200.so.

PyTorch supplies device memory and the current stream; all compute runs in the
hand-written sm_100a kernels of libems_b200.so.  There is no fallback: if the
library (or a GPU) is missing, every entry point raises.

The functions mirror the reference operator API (proj/include/ems/*.hpp):
``prefill_attention`` / ``prefill_scores`` (scoring.hpp:48-54),
``redundancy_cross`` (analysis.hpp:19-20) and ``compress_prefill`` /
``prefill`` (compressor.hpp:58-60, engine.cpp:42-82), batched over
[B][H][L][d] tensors.  Errors map to the reference's exception types.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EMS_LIB_PATH") or os.path.join(PKG, "libems_b200.so")  # override: A/B tuning only

EMS_F32, EMS_BF16 = 0, 1
SCORE_IMPL = {"auto": 0, "simt": 1, "tcgen05": 2}


class EmsError(RuntimeError):
    pass


class InvalidArgument(EmsError, ValueError):
    """std::invalid_argument in the reference."""


class DegenerateInputError(EmsError):
    """ems::DegenerateInputError (proj/include/ems/errors.hpp:11-16)."""


class CorruptionError(EmsError):
    """ems::CorruptionError (proj/include/ems/errors.hpp:32-36)."""


class CudaError(EmsError):
    pass


class Unsupported(EmsError):
    pass


_ERR = {1: InvalidArgument, 2: DegenerateInputError, 3: CorruptionError, 4: CudaError, 5: Unsupported}


class Desc(C.Structure):
    _fields_ = [("batch", C.c_int32), ("heads_q", C.c_int32), ("heads_kv", C.c_int32),
                ("seq_len", C.c_int32), ("head_dim", C.c_int32), ("dtype", C.c_int32),
                ("l_win", C.c_int32), ("n_budget", C.c_int32), ("tau", C.c_double),
                ("gamma", C.c_double), ("kernel_size", C.c_int32), ("zero_class", C.c_int32),
                ("key_only", C.c_int32), ("score_impl", C.c_int32), ("first_position", C.c_int64),
                ("policy", C.c_int32), ("sink_count", C.c_int32), ("position_mode", C.c_int32)]

# ems_policy (include/ems_b200.h; PolicyKind, proj/include/ems/policies.hpp:12)
POLICY = {"ems": 0, "full": 1, "streaming": 2, "h2o": 3, "snapkv": 4}


class CacheDims(C.Structure):
    _fields_ = [("units", C.c_int32), ("centers", C.c_int32), ("locals", C.c_int32),
                ("lut", C.c_int32), ("tbm", C.c_int32)]


class CCache(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("center_key", "center_norm", "center_value", "center_pos",
                                          "center_score", "local_key", "local_value", "local_pos",
                                          "local_score", "lut_pos", "lut_slot", "counts")]


class CStage(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("pooled", "cls", "imp_idx", "tbm_idx", "part_counts",
                                          "dest")]


class DecodeDims(C.Structure):
    _fields_ = [("units", C.c_int32), ("slots", C.c_int32), ("locals", C.c_int32), ("lut", C.c_int32),
                ("rows", C.c_int32)]


DECODE_FIELDS = ("slot_key", "slot_norm", "slot_value", "slot_pos", "slot_score", "slot_alive", "local_key",
                 "local_value", "local_pos", "local_score", "lut_pos", "lut_slot", "meta")


class CDecode(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in DECODE_FIELDS]


_lib = None


def lib() -> C.CDLL:
    """Load libems_b200.so; fail loudly when it is absent (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2412_08521_b200.build`")
        L = C.CDLL(LIB_PATH)
        L.ems_last_error.restype = C.c_char_p
        L.ems_status_string.restype = C.c_char_p
        L.ems_workspace_bytes.restype = C.c_size_t
        L.ems_workspace_bytes.argtypes = [C.POINTER(Desc)]
        L.ems_prefill_host_workspace_bytes.restype = C.c_size_t
        L.ems_prefill_host_workspace_bytes.argtypes = [C.POINTER(Desc)]
        L.ems_validate.argtypes = [C.POINTER(Desc)]
        L.ems_cache_dims_for.argtypes = [C.POINTER(Desc), C.POINTER(CacheDims)]
        vp, fp = C.c_void_p, C.c_void_p
        L.ems_score.argtypes = [C.POINTER(Desc), vp, vp, vp, vp, fp, fp, fp, vp, C.c_size_t, vp]
        L.ems_select.argtypes = [C.POINTER(Desc), fp, fp, C.POINTER(CStage), vp, C.c_size_t, vp]
        L.ems_merge.argtypes = [C.POINTER(Desc), vp, vp, C.POINTER(CStage), vp, C.c_size_t, vp]
        L.ems_compact.argtypes = [C.POINTER(Desc), vp, vp, fp, fp, C.POINTER(CStage),
                                  C.POINTER(CCache), vp, C.c_size_t, vp]
        L.ems_prefill_compress.argtypes = [C.POINTER(Desc), vp, vp, vp, vp, vp, fp, fp, fp,
                                           C.POINTER(CStage), C.POINTER(CCache), vp, C.c_size_t, vp]
        L.ems_redundancy_cross.argtypes = [C.c_int32, C.c_int32, vp, vp, C.c_int32, vp, vp,
                                           C.c_int32, C.c_int32, fp, vp]
        L.ems_sync_status.argtypes = [C.POINTER(Desc), vp, vp]
        L.ems_diagnostics_workspace_bytes.restype = C.c_size_t
        L.ems_diagnostics_workspace_bytes.argtypes = [C.c_int32, C.c_int32]
        L.ems_sparsity_rate.argtypes = [C.c_int32, C.c_int32, fp, fp, C.c_double, vp, vp, C.c_size_t, vp]
        L.ems_redundancy_rate.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp, vp, C.c_double, vp, vp,
                                          C.c_size_t, vp]
        L.ems_prefill_host.argtypes = [C.POINTER(Desc), C.c_double, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                       vp, fp, fp, fp, C.POINTER(CCache), C.POINTER(CCache), C.c_int32, vp,
                                       C.c_size_t, vp, vp]
        L.ems_decode_dims_for.argtypes = [C.POINTER(Desc), C.c_int32, C.POINTER(DecodeDims)]
        L.ems_decode_workspace_bytes.restype = C.c_size_t
        L.ems_decode_workspace_bytes.argtypes = [C.POINTER(Desc), C.c_int32]
        L.ems_rope_table.argtypes = [C.c_int32, C.c_double, C.c_int32, vp, vp]
        L.ems_decode_sync_status.argtypes = [C.POINTER(Desc), C.POINTER(CDecode), vp]
        L.ems_decode_init.argtypes = [C.POINTER(Desc), C.c_int32, C.POINTER(CCache), C.POINTER(CDecode), vp]
        L.ems_decode_step.argtypes = [C.POINTER(Desc), C.c_int64, vp, C.c_int32, vp, vp, vp, vp, vp,
                                      C.POINTER(CDecode), vp, C.c_size_t, vp]
        L.ems_rope.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int64, vp, vp,
                               vp]
        L.ems_prefill.argtypes = [C.POINTER(Desc), C.c_double, vp, vp, vp, vp, vp, vp, fp, fp, fp,
                                  C.POINTER(CStage), C.POINTER(CCache), vp, C.c_size_t, vp]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().ems_last_error().decode()
        raise _ERR.get(rc, EmsError)(msg or f"status {rc}")


def _p(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass(frozen=True)
class EmsConfig:
    """CompressionConfig (proj/include/ems/cache.hpp:20-39) plus the D1 similarity flag."""
    n_budget: int = 256
    l_win: int = 32
    tau: float = 0.6
    gamma: float = 4.0
    kernel_size: int = 7
    zero_class: bool = True
    key_only: bool = False
    policy: str = "ems"      # PolicyHandle::kind: ems | full | streaming | h2o | snapkv
    sink_count: int = 4      # PolicyHandle::sink_count (streaming)
    position_mode: str = "with_pos"  # decode expansion RoPE (cache.hpp:11): with_pos | without_pos
    zeta: float = 0.95       # sparsity mass fraction (diagnostics only), (0, 1]

    def center_capacity(self) -> int:
        return self.n_budget - self.l_win

    def tbm_target(self) -> int:
        return int((self.gamma - 1.0) * float(self.n_budget)) if self.policy == "ems" else 0


def _dtype_code(t: torch.dtype) -> int:
    if t == torch.float32:
        return EMS_F32
    if t == torch.bfloat16:
        return EMS_BF16
    raise InvalidArgument(f"unsupported dtype {t} (float32 or bfloat16)")


def make_desc(B: int, Hq: int, Hkv: int, L: int, d: int, dtype: torch.dtype, cfg: EmsConfig,
              score_impl: str = "auto", first_position: int = 0) -> Desc:
    if cfg.policy not in POLICY:
        raise InvalidArgument(f"unknown policy: {cfg.policy}")  # policy_kind_from_name, policies.cpp:118-125
    return Desc(B, Hq, Hkv, L, d, _dtype_code(dtype), cfg.l_win, cfg.n_budget, float(cfg.tau),
                float(cfg.gamma), cfg.kernel_size, int(cfg.zero_class), int(cfg.key_only),
                SCORE_IMPL[score_impl], first_position, POLICY[cfg.policy], int(cfg.sink_count),
                {"with_pos": 0, "without_pos": 1}[cfg.position_mode])


class Plan:
    """Pre-allocated buffers for one problem shape: workspace, stage, cache, scores.

    Construct once, then ``run`` as often as needed (no allocation on the hot path)."""

    def __init__(self, B: int, Hq: int, Hkv: int, L: int, d: int, dtype: torch.dtype,
                 cfg: EmsConfig, device=None, score_impl: str = "auto", want_out: bool = True,
                 want_lse: bool = False, first_position: int = 0):
        self.device = torch.device(device or "cuda")
        self.desc = make_desc(B, Hq, Hkv, L, d, dtype, cfg, score_impl, first_position)
        self.cfg, self.dtype = cfg, dtype
        L_ = lib()
        _check(L_.ems_validate(C.byref(self.desc)))
        dims = CacheDims()
        _check(L_.ems_cache_dims_for(C.byref(self.desc), C.byref(dims)))
        self.dims = dims
        U = dims.units
        dev = self.device
        nbytes = L_.ems_workspace_bytes(C.byref(self.desc))
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.workspace[:256].zero_()  # device status word: no error recorded yet
        mk = lambda *s, dt=torch.float32: torch.zeros(s, dtype=dt, device=dev)  # noqa: E731
        self.glo = mk(B, Hkv, L)
        self.loc = mk(B, Hkv, L)
        self.out = torch.empty((B, Hq, L, d), dtype=dtype, device=dev) if want_out else None
        self.lse = mk(B, Hq, L) if want_lse else None
        tb = max(dims.tbm, 1)
        self.stage = dict(pooled=mk(U, L), cls=mk(U, L, dt=torch.int8),
                          imp_idx=mk(U, dims.centers, dt=torch.int32),
                          tbm_idx=mk(U, tb, dt=torch.int32),
                          part_counts=mk(U, 4, dt=torch.int32), dest=mk(U, tb, dt=torch.int32))
        self.cache = dict(center_key=mk(U, dims.centers, d, dt=dtype),
                          center_norm=mk(U, dims.centers),
                          center_value=mk(U, dims.centers, d, dt=dtype),
                          center_pos=mk(U, dims.centers, dt=torch.int32),
                          center_score=mk(U, dims.centers, 3),
                          local_key=mk(U, dims.locals, d, dt=dtype),
                          local_value=mk(U, dims.locals, d, dt=dtype),
                          local_pos=mk(U, dims.locals, dt=torch.int32),
                          local_score=mk(U, dims.locals, 3),
                          lut_pos=mk(U, max(dims.lut, 1), dt=torch.int32),
                          lut_slot=mk(U, max(dims.lut, 1), dt=torch.int32),
                          counts=mk(U, 4, dt=torch.int32))
        self._cstage = CStage(*[_p(self.stage[f]) for f, _ in CStage._fields_])
        self._ccache = CCache(*[_p(self.cache[f]) for f, _ in CCache._fields_])

    def _check_inputs(self, q_rot, k_rot, k_raw, v):
        D = self.desc
        want_q = (D.batch, D.heads_q, D.seq_len, D.head_dim)
        want_k = (D.batch, D.heads_kv, D.seq_len, D.head_dim)
        for name, t, shp in (("q_rot", q_rot, want_q), ("k_rot", k_rot, want_k),
                             ("k_raw", k_raw, want_k), ("v", v, want_k)):
            if t is None:
                continue
            if tuple(t.shape) != shp or t.dtype != self.dtype or not t.is_contiguous() \
                    or t.device != self.device and t.device.type != "cuda":
                raise InvalidArgument(f"{name}: want contiguous {shp} {self.dtype} on cuda, got "
                                      f"{tuple(t.shape)} {t.dtype} {t.device}")

    def run(self, q_rot, k_rot, k_raw, v, stream=None) -> None:
        """Whole path (ems_prefill_compress), asynchronous on the current stream."""
        self._check_inputs(q_rot, k_rot, k_raw, v)
        self._status_ws = None
        _check(lib().ems_prefill_compress(C.byref(self.desc), _p(q_rot), _p(k_rot), _p(k_raw), _p(v),
                                          _p(self.out), _p(self.lse), _p(self.glo), _p(self.loc),
                                          C.byref(self._cstage), C.byref(self._ccache),
                                          _p(self.workspace), self.workspace.numel(),
                                          _stream(stream)))

    def run_raw(self, q, k, v, rope_base: float, stream=None) -> None:
        """engine::prefill on RAW Q/K (ems_prefill): RoPE on the device into the plan's
        q_rot/k_rot scratch, then the whole path with k as the pre-RoPE keys."""
        self._check_inputs(q, k, k, v)
        self._status_ws = None
        if rope_base > 0 and getattr(self, "q_rot", None) is None:
            D = self.desc
            self.q_rot = torch.empty((D.batch, D.heads_q, D.seq_len, D.head_dim), dtype=self.dtype,
                                     device=self.device)
            self.k_rot = torch.empty((D.batch, D.heads_kv, D.seq_len, D.head_dim), dtype=self.dtype,
                                     device=self.device)
        qr = self.q_rot if rope_base > 0 else None
        kr = self.k_rot if rope_base > 0 else None
        _check(lib().ems_prefill(C.byref(self.desc), float(rope_base), _p(q), _p(k), _p(v), _p(qr), _p(kr),
                                 _p(self.out), _p(self.lse), _p(self.glo), _p(self.loc),
                                 C.byref(self._cstage), C.byref(self._ccache), _p(self.workspace),
                                 self.workspace.numel(), _stream(stream)))

    def host_cache(self) -> dict:
        """Pinned host buffers shaped like the device cache (targets of run_host)."""
        if getattr(self, "_host_cache", None) is None:
            self._host_cache = {k: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for k, t in self.cache.items()}
            self._hcache = CCache(*[_p(self._host_cache[f]) for f, _ in CCache._fields_])
        return self._host_cache

    def run_host(self, h_q, h_k, h_v, rope_base: float, h_k_raw=None, chunks: int = 8, stream=None,
                 concurrent: bool = True, h_out=None) -> dict:
        """engine::prefill from HOST (pinned) tensors (ems_prefill_host): the library stages the
        inputs in `chunks` groups of units and overlaps each group's host-to-device copy with
        the previous group's compute; every group's compressed cache (and, with h_out, its
        attention output rows: PrefillResult.per_head, engine.hpp:36-45) is copied back to pinned
        host memory as soon as it is done.  rope_base > 0: raw Q/K, RoPE on the device;
        rope_base == 0: pre-rotated Q/K plus h_k_raw.  concurrent: two groups in flight (a
        second workspace, ems_prefill_host_workspace_bytes).  Asynchronous; returns the host cache."""
        D = self.desc
        qs = (D.batch, D.heads_q, D.seq_len, D.head_dim)
        ks = (D.batch, D.heads_kv, D.seq_len, D.head_dim)
        if h_out is not None and self.out is None:
            raise InvalidArgument("h_out needs a plan built with want_out=True")
        for name, t, shp in (("q", h_q, qs), ("k", h_k, ks), ("v", h_v, ks), ("k_raw", h_k_raw, ks),
                             ("out", h_out, qs)):
            if t is None:
                continue
            if tuple(t.shape) != shp or t.dtype != self.dtype or not t.is_contiguous() or t.is_cuda \
                    or not t.is_pinned():
                raise InvalidArgument(f"{name}: want contiguous pinned host {shp} {self.dtype}")
        if getattr(self, "_stage_in", None) is None:
            mk = lambda shp: torch.empty(shp, dtype=self.dtype, device=self.device)  # noqa: E731
            self._stage_in = dict(q=mk(qs), k=mk(ks), v=mk(ks))
        st = self._stage_in
        if rope_base > 0:
            if getattr(self, "q_rot", None) is None:
                self.q_rot = torch.empty(qs, dtype=self.dtype, device=self.device)
                self.k_rot = torch.empty(ks, dtype=self.dtype, device=self.device)
            kraw_d = None
        else:
            if h_k_raw is None:
                raise InvalidArgument("pre-rotated inputs (rope_base == 0) need h_k_raw")
            kraw_d = st.setdefault("k_raw", torch.empty(ks, dtype=self.dtype, device=self.device))
        hc = self.host_cache()
        if concurrent and getattr(self, "_ws_host", None) is None:  # room for two unit groups in flight
            self._ws_host = torch.empty(lib().ems_prefill_host_workspace_bytes(C.byref(self.desc)), dtype=torch.uint8,
                                        device=self.device)
        ws = self._ws_host if concurrent else self.workspace
        self._status_ws = ws
        _check(lib().ems_prefill_host(
            C.byref(self.desc), float(rope_base), _p(h_q), _p(h_k), _p(h_k_raw), _p(h_v), _p(st["q"]), _p(st["k"]),
            _p(kraw_d), _p(st["v"]), _p(self.q_rot) if rope_base > 0 else None,
            _p(self.k_rot) if rope_base > 0 else None, _p(self.out), _p(h_out), _p(self.lse), _p(self.glo),
            _p(self.loc),
            C.byref(self._ccache), C.byref(self._hcache), int(chunks), _p(ws), ws.numel(),
            _stream(stream), None))
        return hc

    def score(self, q_rot, k_rot, v=None, stream=None) -> None:
        self._check_inputs(q_rot, k_rot, None, v)
        self._status_ws = None
        _check(lib().ems_score(C.byref(self.desc), _p(q_rot), _p(k_rot), _p(v),
                               _p(self.out) if v is not None else None, _p(self.lse), _p(self.glo),
                               _p(self.loc), _p(self.workspace), self.workspace.numel(),
                               _stream(stream)))

    def select(self, stream=None) -> None:
        self._status_ws = None
        _check(lib().ems_select(C.byref(self.desc), _p(self.glo), _p(self.loc), C.byref(self._cstage),
                                _p(self.workspace), self.workspace.numel(), _stream(stream)))

    def merge(self, k_raw, v, stream=None) -> None:
        _check(lib().ems_merge(C.byref(self.desc), _p(k_raw), _p(v), C.byref(self._cstage),
                               _p(self.workspace), self.workspace.numel(), _stream(stream)))

    def compact(self, k_raw, v, stream=None) -> None:
        _check(lib().ems_compact(C.byref(self.desc), _p(k_raw), _p(v), _p(self.glo), _p(self.loc),
                                 C.byref(self._cstage), C.byref(self._ccache), _p(self.workspace),
                                 self.workspace.numel(), _stream(stream)))

    def sync_status(self, stream=None) -> None:
        """Synchronise and raise the first data-dependent error the kernels recorded (in the
        workspace of the last run: the plan's, or run_host's larger one)."""
        ws = getattr(self, "_status_ws", None)
        _check(lib().ems_sync_status(C.byref(self.desc), _p(self.workspace if ws is None else ws), _stream(stream)))

    def unit_cache(self, u: int) -> dict:
        """Host copy of unit u's compressed cache, trimmed to its counts."""
        cnt = self.cache["counts"][u].tolist()
        nc, nl, nu, comp = cnt
        g = lambda k: self.cache[k][u].cpu()  # noqa: E731
        return dict(compressed=bool(comp),
                    unit_key=g("center_key")[:nc].double().numpy(),
                    key_norm=g("center_norm")[:nc].double().numpy(),
                    value=g("center_value")[:nc].double().numpy(),
                    position=g("center_pos")[:nc].long().numpy(),
                    score=g("center_score")[:nc].double().numpy(),
                    local_key=g("local_key")[:nl].double().numpy(),
                    local_value=g("local_value")[:nl].double().numpy(),
                    local_position=g("local_pos")[:nl].long().numpy(),
                    local_score=g("local_score")[:nl].double().numpy(),
                    lut_position=g("lut_pos")[:nu].long().numpy(),
                    lut_slot=g("lut_slot")[:nu].numpy())


def cache_dump_json(c: dict, head_dim: int) -> str:
    """cache_dump_json (proj/src/cache.cpp:114-150) of a unit's cache as returned by
    Plan.unit_cache / DecodeState.unit_cache: the reference's schema and key order (centers
    by slot, locals oldest first, LUT in order), so its tooling reads GPU caches directly."""
    import json
    slots = c.get("slots", range(len(c["position"])))
    trip = lambda t: {"glo": float(t[0]), "loc_past": float(t[1]), "loc_cur": float(t[2])}  # noqa: E731
    centers = [{"slot": int(s), "position": int(c["position"][i]), "key_norm": float(c["key_norm"][i]),
                "unit_key": [float(x) for x in c["unit_key"][i]], "value": [float(x) for x in c["value"][i]],
                "score": trip(c["score"][i])} for i, s in enumerate(slots)]
    locals_ = [{"position": int(c["local_position"][i]), "key": [float(x) for x in c["local_key"][i]],
                "value": [float(x) for x in c["local_value"][i]], "score": trip(c["local_score"][i])}
               for i in range(len(c["local_position"]))]
    lut = [{"position": int(p), "slot": int(s)} for p, s in zip(c["lut_position"], c["lut_slot"])]
    return json.dumps({"head_dim": int(head_dim), "compressed": bool(c["compressed"]), "centers": centers,
                       "locals": locals_, "lut": lut}, indent=2)


# -- reference-shaped conveniences ----------------------------------------------------
def prefill_compress(q_rot, k_rot, k_raw, v, cfg: EmsConfig, want_out=True, score_impl="auto",
                     first_position=0) -> Plan:
    """engine::prefill's score -> compress sequence (engine.cpp:42-82) on [B][H][L][d] tensors.
    Returns the Plan holding O, glo/loc, the stage buffers and the compressed cache."""
    B, Hq, L, d = q_rot.shape
    Hkv = k_rot.shape[1]
    plan = Plan(B, Hq, Hkv, L, d, q_rot.dtype, cfg, q_rot.device, score_impl, want_out,
                first_position=first_position)
    plan.run(q_rot, k_rot, k_raw, v)
    plan.sync_status()
    return plan


def rope(x: torch.Tensor, base: float, first_position: int = 0, out: torch.Tensor | None = None) -> torch.Tensor:
    """apply_rope (proj/src/rope.cpp:10-37) over the token axis of [..., L, d] on the device:
    fp64 rotation, rounded once to the tensor's dtype."""
    if not x.is_contiguous():
        raise InvalidArgument("rope: x must be contiguous")
    L, d = x.shape[-2], x.shape[-1]
    planes = x.numel() // max(L * d, 1)
    y = torch.empty_like(x) if out is None else out
    _check(lib().ems_rope(_dtype_code(x.dtype), planes, L, d, float(base), int(first_position), _p(x), _p(y),
                          _stream()))
    return y


def prefill(q, k, v, cfg: EmsConfig, rope_base: float, want_out=True, score_impl="auto",
            first_position=0) -> Plan:
    """engine::prefill (proj/src/engine.cpp:42-82) on RAW [B][H][L][d] tensors: RoPE
    (rope_base, 0 = none), score, compress.  Returns the Plan (O, glo/loc, cache)."""
    B, Hq, L, d = q.shape
    plan = Plan(B, Hq, k.shape[1], L, d, q.dtype, cfg, q.device, score_impl, want_out,
                first_position=first_position)
    plan.run_raw(q, k, v, rope_base)
    plan.sync_status()
    return plan


def prefill_host(q, k, v, cfg: EmsConfig, rope_base: float, chunks: int = 8, want_out=True, score_impl="auto",
                 first_position=0) -> Plan:
    """engine::prefill (proj/src/engine.cpp:42-82) on pinned HOST [B][H][L][d] tensors, the
    reference's own calling convention: copies pipelined with compute (ems_prefill_host).
    Returns the Plan; plan.host_cache() holds the compressed cache on the host and, with
    want_out, plan.host_out the attention outputs (PrefillResult.per_head, engine.hpp:36-45)."""
    B, Hq, L, d = q.shape
    plan = Plan(B, Hq, k.shape[1], L, d, q.dtype, cfg, "cuda", score_impl, want_out,
                first_position=first_position)
    plan.host_out = torch.empty(q.shape, dtype=q.dtype, pin_memory=True) if want_out else None
    plan.run_host(q, k, v, rope_base, chunks=chunks, h_out=plan.host_out)
    plan.sync_status()
    return plan


def prefill_attention(q_rot, k_rot, v, l_win: int, score_impl="auto"):
    """prefill_attention (scoring.hpp:52-54), batched + GQA-mean: returns (O, glo, loc)."""
    B, Hq, L, d = q_rot.shape
    cfg = EmsConfig(n_budget=max(l_win + 1, 2), l_win=max(l_win, 1), gamma=1.0, kernel_size=1)
    plan = Plan(B, Hq, k_rot.shape[1], L, d, q_rot.dtype, cfg, q_rot.device, score_impl, True)
    plan.score(q_rot, k_rot, v)
    torch.cuda.current_stream().synchronize()
    return plan.out, plan.glo, plan.loc


def prefill_scores(q_rot, k_rot, l_win: int, score_impl="auto"):
    """prefill_scores (scoring.hpp:48-49): returns (glo, loc)."""
    B, Hq, L, d = q_rot.shape
    cfg = EmsConfig(n_budget=max(l_win + 1, 2), l_win=max(l_win, 1), gamma=1.0, kernel_size=1)
    plan = Plan(B, Hq, k_rot.shape[1], L, d, q_rot.dtype, cfg, q_rot.device, score_impl, False)
    plan.score(q_rot, k_rot, None)
    torch.cuda.current_stream().synchronize()
    return plan.glo, plan.loc


def redundancy_cross(k_rows, v_rows, k_cols, v_cols, key_only=False) -> torch.Tensor:
    """redundancy_cross (analysis.hpp:19-20) on device tensors [n][d] -> fp32 [n_rows][n_cols]."""
    nr, d = k_rows.shape
    nc = k_cols.shape[0]
    r = torch.empty((nr, nc), dtype=torch.float32, device=k_rows.device)
    _check(lib().ems_redundancy_cross(_dtype_code(k_rows.dtype), d, _p(k_rows), _p(v_rows), nr,
                                      _p(k_cols), _p(v_cols), nc, int(key_only), _p(r), _stream()))
    return r


def _diag_ws(units: int, L: int, device) -> torch.Tensor:
    return torch.empty(lib().ems_diagnostics_workspace_bytes(units, L), dtype=torch.uint8, device=device)


def sparsity_rate(glo: torch.Tensor, loc: torch.Tensor, zeta: float) -> torch.Tensor:
    """sparsity_rate(combine_glo_loc(glo, loc), zeta) (analysis.cpp:71-91, scoring.cpp:105-124)
    for every sequence of glo / loc [..., L] fp32 -> fp64 [...] on the device."""
    L = glo.shape[-1]
    units = glo.numel() // max(L, 1)
    rate = torch.empty(glo.shape[:-1], dtype=torch.float64, device=glo.device)
    ws = _diag_ws(units, L, glo.device)
    glo, loc = glo.float().contiguous(), loc.float().contiguous()
    _check(lib().ems_sparsity_rate(units, L, _p(glo), _p(loc), float(zeta), _p(rate), _p(ws), ws.numel(),
                                   _stream()))
    _check(lib().ems_sync_status(None, _p(ws), _stream()))
    return rate


def redundancy_rate(k_raw: torch.Tensor, v_raw: torch.Tensor, tau: float) -> torch.Tensor:
    """redundancy_rate_direct(k_raw, v_raw, tau) (analysis.cpp:93-118) for every sequence of
    k / v [..., L, d] -> fp64 [...] on the device."""
    L, d = k_raw.shape[-2], k_raw.shape[-1]
    units = k_raw.numel() // max(L * d, 1)
    rate = torch.empty(k_raw.shape[:-2], dtype=torch.float64, device=k_raw.device)
    ws = _diag_ws(units, L, k_raw.device)
    k_raw, v_raw = k_raw.contiguous(), v_raw.contiguous()
    _check(lib().ems_redundancy_rate(_dtype_code(k_raw.dtype), d, units, L, _p(k_raw), _p(v_raw), float(tau),
                                     _p(rate), _p(ws), ws.numel(), _stream()))
    return rate


def analyze(q, k, v, cfg: EmsConfig, rope_base: float = 10000.0):
    """analyze_trace (proj/src/experiment.cpp:133-150) on raw [B][H][L][d] device tensors:
    RoPE, prefill_scores with min(l_win, L), sparsity of the combined score and redundancy of
    the raw K/V per unit.  Returns (sparsity, redundancy), fp64 [B][H_kv]."""
    L = q.shape[2]
    glo, loc = prefill_scores(rope(q.contiguous(), rope_base), rope(k.contiguous(), rope_base), min(cfg.l_win, L))
    return sparsity_rate(glo, loc, cfg.zeta), redundancy_rate(k, v, cfg.tau)


class DecodeState:
    """The decode loop on the device (ems_decode_*): decode_step (proj/src/engine.cpp:150-210)
    with the policy's decode rule (policy_decode_compress, proj/src/policies.cpp:182-242; EMS:
    decode_update, proj/src/compressor.cpp:376-398) for every unit of a problem, one CTA per
    unit per step.  State = fixed-capacity SoA (ems_decode_state); max_positions bounds the
    RoPE table and the growth of the SnapKV / full caches."""

    def __init__(self, B: int, Hq: int, Hkv: int, L: int, d: int, dtype: torch.dtype, cfg: EmsConfig,
                 rope_base: float, max_positions: int, device=None):
        self.device = torch.device(device or "cuda")
        self.desc = make_desc(B, Hq, Hkv, L, d, dtype, cfg)
        self.dtype, self.cfg = dtype, cfg
        L_ = lib()
        dims = DecodeDims()
        self.max_positions = int(max_positions)
        _check(L_.ems_decode_dims_for(C.byref(self.desc), self.max_positions, C.byref(dims)))
        self.dims = dims
        U, S, W, T = dims.units, dims.slots, dims.locals, dims.lut
        dev = self.device
        z = lambda *shape, dt=torch.float32: torch.zeros(shape, dtype=dt, device=dev)  # noqa: E731
        i32, f64 = torch.int32, torch.float64
        self.state = dict(slot_key=z(U, S, d), slot_norm=z(U, S), slot_value=z(U, S, d), slot_pos=z(U, S, dt=i32),
                          slot_score=z(U, S, 3, dt=f64), slot_alive=z(U, S, dt=i32), local_key=z(U, W, d),
                          local_value=z(U, W, d), local_pos=z(U, W, dt=i32), local_score=z(U, W, 3, dt=f64),
                          lut_pos=z(U, T, dt=i32), lut_slot=z(U, T, dt=i32), meta=z(U, 8, dt=i32))
        self._c = CDecode(*[_p(self.state[f]) for f in DECODE_FIELDS])
        self.table = torch.empty((self.max_positions, d // 2, 2), dtype=torch.float32, device=dev)
        _check(L_.ems_rope_table(d, float(rope_base), self.max_positions, _p(self.table), _stream()))
        self.workspace = torch.empty(max(L_.ems_decode_workspace_bytes(C.byref(self.desc), self.max_positions), 16),
                                     dtype=torch.uint8, device=dev)
        self.out = torch.empty((B, Hq, d), dtype=dtype, device=dev)
        self.argmax = torch.empty((B, Hq), dtype=torch.int32, device=dev)
        self.position = L

    def init_from_plan(self, plan: "Plan") -> None:
        """Decode state from a prefill Plan's compressed cache (ems_decode_init)."""
        _check(lib().ems_decode_init(C.byref(self.desc), self.max_positions, C.byref(plan._ccache), C.byref(self._c),
                                     _stream()))
        self.position = plan.desc.seq_len + plan.desc.first_position

    def load_caches(self, caches, position: int) -> None:
        """Test helper: state from reference HeadCacheState dumps (oracle.Cache objects with
        extra['slots'] = the reference slot indices), one per unit; window_fill = 0."""
        st = {k: v.cpu() for k, v in self.state.items()}
        for k in st:
            st[k].zero_()
        for u, c in enumerate(caches):
            for j, slot in enumerate(c.extra.get("slots", range(len(c.position)))):
                st["slot_key"][u, slot] = torch.tensor(c.unit_key[j])
                st["slot_norm"][u, slot] = float(c.key_norm[j])
                st["slot_value"][u, slot] = torch.tensor(c.value[j])
                st["slot_pos"][u, slot] = int(c.position[j])
                st["slot_score"][u, slot] = torch.tensor(c.score[j], dtype=torch.float64)
                st["slot_alive"][u, slot] = 1
            nl = len(c.local_position)
            st["local_key"][u, :nl] = torch.tensor(c.local_key)
            st["local_value"][u, :nl] = torch.tensor(c.local_value)
            st["local_pos"][u, :nl] = torch.tensor(c.local_position, dtype=torch.int32)
            st["local_score"][u, :nl] = torch.tensor(c.local_score, dtype=torch.float64)
            nu = len(c.lut_position)
            st["lut_pos"][u, :nu] = torch.tensor(c.lut_position, dtype=torch.int32)
            st["lut_slot"][u, :nu] = torch.tensor(c.lut_slot, dtype=torch.int32)
            st["meta"][u] = torch.tensor([0, nl, nu, 0, int(c.compressed), len(c.position), 0, 0])
        for k, v in st.items():
            self.state[k].copy_(v)
        self.position = position

    def step(self, q, k, v, stream=None):
        """One decode step: q [B][Hq][d], k/v [B][Hkv][d] raw (device, dtype) -> (out, argmax)."""
        _check(lib().ems_decode_step(C.byref(self.desc), self.position, _p(self.table), self.max_positions, _p(q),
                                     _p(k), _p(v), _p(self.out), _p(self.argmax), C.byref(self._c),
                                     _p(self.workspace), self.workspace.numel(), _stream(stream)))
        self.position += 1
        return self.out, self.argmax

    def sync_status(self, stream=None) -> None:
        """Synchronise and raise the first unit's decode error (ems_decode_sync_status)."""
        _check(lib().ems_decode_sync_status(C.byref(self.desc), C.byref(self._c), _stream(stream)))

    def unit_cache(self, u: int) -> dict:
        """Host view of unit u's state, shaped like a reference HeadCacheState dump."""
        st = {k: t[u].cpu() for k, t in self.state.items()}
        head, nl, nu, wfill, comp, nalive = st["meta"][:6].tolist()
        W = self.dims.locals
        alive = [s for s in range(self.dims.slots) if st["slot_alive"][s]]
        ring = [(head + i) % W for i in range(nl)]
        return dict(compressed=bool(comp), window_fill=wfill, slots=alive,
                    position=st["slot_pos"][alive].long().numpy(), unit_key=st["slot_key"][alive].double().numpy(),
                    key_norm=st["slot_norm"][alive].double().numpy(), value=st["slot_value"][alive].double().numpy(),
                    score=st["slot_score"][alive].numpy(), local_position=st["local_pos"][ring].long().numpy(),
                    local_key=st["local_key"][ring].double().numpy(), local_value=st["local_value"][ring].double().numpy(),
                    local_score=st["local_score"][ring].numpy(), lut_position=st["lut_pos"][:nu].long().numpy(),
                    lut_slot=st["lut_slot"][:nu].numpy())
