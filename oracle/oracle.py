"""ctypes front-end to the CPU oracles.  TEST INFRASTRUCTURE ONLY.

Two checkers live behind this module:

* ``Oracle``  -- ``_build/libems_oracle.so``, the C restatement in ems_oracle.c
  (every function cites the reference file:line it restates);
* ``RefLib``  -- ``_ref/libems_ref.so``, the reference's own C++ sources
  compiled in place by oracle/Makefile plus the extern "C" shim ref_driver.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product library never
does; it fails loudly when its CUDA extension is missing.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libems_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libems_ref.so")
REFERENCE_SRC = "/root/reference/proj/src"

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_i8p = C.POINTER(C.c_int8)


def build(ref: bool | None = None) -> None:
    """Compile the C restatement and, where /root/reference exists, the reference."""
    targets = ["oracle"]
    if ref is None:
        ref = os.path.isdir(REFERENCE_SRC)
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _ptr(a: np.ndarray | None, typ=_dp):
    if a is None:
        return C.cast(None, typ)
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(typ)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError):
    pass


class DegenerateInput(OracleError):
    pass


class Corruption(OracleError):
    pass


_ERRS = {1: InvalidArgument, 2: DegenerateInput, 3: Corruption}


def _check(rc: int, what: str, msg: str = "") -> None:
    if rc != 0:
        raise _ERRS.get(rc, OracleError)(f"{what}: status {rc} {msg}")


@dataclass
class Config:
    """Mirrors CompressionConfig, proj/include/ems/cache.hpp:20-39."""
    n_budget: int = 256
    l_win: int = 32
    tau: float = 0.6
    gamma: float = 4.0
    zeta: float = 0.95
    kernel_size: int = 7
    zero_class: bool = True
    key_only: bool = False

    def center_capacity(self) -> int:
        return self.n_budget - self.l_win

    def tbm_target(self) -> int:
        return int((self.gamma - 1.0) * float(self.n_budget))

    def lut_capacity(self) -> int:
        return int(self.gamma * float(self.n_budget))


class _CConfig(C.Structure):
    _fields_ = [("n_budget", C.c_int64), ("l_win", C.c_int64), ("tau", C.c_double),
                ("gamma", C.c_double), ("zeta", C.c_double), ("kernel_size", C.c_int64),
                ("zero_class", C.c_int32), ("key_only", C.c_int32)]


class _CCache(C.Structure):
    _fields_ = [("head_dim", C.c_int64), ("compressed", C.c_int32), ("n_centers", C.c_int64),
                ("unit_key", _dp), ("key_norm", _dp), ("value", _dp), ("position", _i64p),
                ("score", _dp), ("n_locals", C.c_int64), ("local_key", _dp),
                ("local_value", _dp), ("local_position", _i64p), ("local_score", _dp),
                ("n_lut", C.c_int64), ("lut_position", _i64p), ("lut_slot", _i32p)]


@dataclass
class Cache:
    """Flattened HeadCacheState (proj/include/ems/cache.hpp:81-111), numpy side."""
    head_dim: int
    compressed: bool
    unit_key: np.ndarray
    key_norm: np.ndarray
    value: np.ndarray
    position: np.ndarray
    score: np.ndarray
    local_key: np.ndarray
    local_value: np.ndarray
    local_position: np.ndarray
    local_score: np.ndarray
    lut_position: np.ndarray
    lut_slot: np.ndarray
    extra: dict = field(default_factory=dict)

    @staticmethod
    def from_dump_json(text: str) -> "Cache":
        """Parse cache_dump_json output (proj/src/cache.cpp:114-150)."""
        j = json.loads(text)
        d = j["head_dim"]
        cs = sorted(j["centers"], key=lambda c: c["slot"])
        ls = j["locals"]

        def arr(items, key, shape):
            return np.array([it[key] for it in items], dtype=np.float64).reshape(shape)

        def trip(items):
            return np.array([[it["score"]["glo"], it["score"]["loc_past"], it["score"]["loc_cur"]]
                             for it in items], dtype=np.float64).reshape(-1, 3)

        return Cache(
            head_dim=d, compressed=bool(j["compressed"]),
            unit_key=arr(cs, "unit_key", (-1, d)), key_norm=arr(cs, "key_norm", (-1,)),
            value=arr(cs, "value", (-1, d)),
            position=np.array([c["position"] for c in cs], dtype=np.int64),
            score=trip(cs),
            local_key=arr(ls, "key", (-1, d)), local_value=arr(ls, "value", (-1, d)),
            local_position=np.array([l["position"] for l in ls], dtype=np.int64),
            local_score=trip(ls),
            lut_position=np.array([e["position"] for e in j["lut"]], dtype=np.int64),
            lut_slot=np.array([e["slot"] for e in j["lut"]], dtype=np.int32),
            extra={"slots": [c["slot"] for c in cs]})


# prefill policies, numbered as the C ABI's ems_policy (proj/include/ems/policies.hpp:12)
POLICY = {"ems": 0, "full": 1, "streaming": 2, "h2o": 3, "snapkv": 4}


class Oracle:
    """The C restatement (oracle/ems_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = L = C.CDLL(path)
        L.ems_oracle_prefill_attention.argtypes = [_dp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64,
                                                   _dp, _dp, _dp, _dp]
        L.ems_oracle_three_step_scores.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64,
                                                   _dp, _dp]
        L.ems_oracle_rope.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_double, C.c_double]
        L.ems_oracle_combine.argtypes = [_dp, _dp, C.c_int64, _dp]
        L.ems_oracle_mean_pool.argtypes = [_dp, C.c_int64, C.c_int64, _dp]
        L.ems_oracle_effective_score.argtypes = [_dp, _dp, _dp, C.c_int64, C.c_int64, _dp]
        L.ems_oracle_partition.argtypes = [_dp, C.c_int64, C.POINTER(_CConfig), _i64p, _i64p,
                                           _i64p, _i64p, _i64p]
        L.ems_oracle_redundancy_cross.argtypes = [_dp, _dp, C.c_int64, _dp, _dp, C.c_int64,
                                                  C.c_int64, C.c_int32, _dp]
        L.ems_oracle_assign.argtypes = [_dp, C.c_int64, C.c_int64, C.c_double, _i32p]
        L.ems_oracle_sparsity_rate.argtypes = [_dp, C.c_int64, C.c_double, C.c_void_p]
        L.ems_oracle_redundancy_rate_direct.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_double, C.c_void_p]
        L.ems_oracle_compress_prefill.argtypes = [_dp, _dp, _dp, _dp, _dp, C.c_int64, C.c_int64,
                                                  C.POINTER(_CConfig), C.c_int64,
                                                  C.POINTER(_CCache), _dp, _i8p, _i32p]
        L.ems_oracle_prefill_unit.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64,
                                              C.POINTER(_CConfig), _dp, _dp, _dp,
                                              C.POINTER(_CCache), _dp, _i8p, _i32p]
        L.ems_oracle_policy_prefill.argtypes = [C.c_int32, C.c_int64, _dp, _dp, _dp, _dp, _dp, C.c_int64,
                                                C.c_int64, C.POINTER(_CConfig), C.POINTER(_CCache), _i8p]

    # -- scoring -----------------------------------------------------------------
    def prefill_attention(self, q, k, v=None, l_win=32, want_out=True):
        q, k = _f64(q), _f64(k)
        n, d = q.shape
        v = None if v is None else _f64(v)
        out = np.zeros((n, d)) if (v is not None and want_out) else None
        glo, loc, lse = np.zeros(n), np.zeros(n), np.zeros(n)
        _check(self.lib.ems_oracle_prefill_attention(_ptr(q), _ptr(k), _ptr(v), n, d, l_win,
                                                     _ptr(out), _ptr(glo), _ptr(loc), _ptr(lse)),
               "prefill_attention")
        return out, glo, loc, lse

    def three_step_scores(self, q, k, l_win):
        q, k = _f64(q), _f64(k)
        n, d = q.shape
        glo, loc = np.zeros(n), np.zeros(n)
        _check(self.lib.ems_oracle_three_step_scores(_ptr(q), _ptr(k), n, d, l_win, _ptr(glo),
                                                     _ptr(loc)), "three_step_scores")
        return glo, loc

    def rope(self, x, base=10000.0, first_position=0.0):
        x = _f64(x)
        out = np.zeros_like(x)
        _check(self.lib.ems_oracle_rope(_ptr(x), _ptr(out), x.shape[0], x.shape[1], base,
                                        first_position), "rope")
        return out

    def combine(self, glo, loc):
        glo, loc = _f64(glo), _f64(loc)
        out = np.zeros_like(glo)
        _check(self.lib.ems_oracle_combine(_ptr(glo), _ptr(loc), glo.size, _ptr(out)), "combine")
        return out

    def mean_pool(self, s, kernel):
        s = _f64(s)
        out = np.zeros_like(s)
        _check(self.lib.ems_oracle_mean_pool(_ptr(s), s.size, kernel, _ptr(out)), "mean_pool")
        return out

    def effective_score(self, glo, loc_past, loc_cur, kernel):
        glo, lp, lc = _f64(glo), _f64(loc_past), _f64(loc_cur)
        out = np.zeros_like(glo)
        _check(self.lib.ems_oracle_effective_score(_ptr(glo), _ptr(lp), _ptr(lc), glo.size,
                                                   kernel, _ptr(out)), "effective_score")
        return out

    # -- evict / merge -----------------------------------------------------------
    @staticmethod
    def _cfg(c: Config) -> _CConfig:
        return _CConfig(c.n_budget, c.l_win, c.tau, c.gamma, c.zeta, c.kernel_size,
                        int(c.zero_class), int(c.key_only))

    def partition(self, pooled, c: Config):
        pooled = _f64(pooled)
        n = pooled.size
        bufs = [np.zeros(max(n, 1), dtype=np.int64) for _ in range(4)]
        counts = np.zeros(4, dtype=np.int64)
        cc = self._cfg(c)
        _check(self.lib.ems_oracle_partition(_ptr(pooled), n, C.byref(cc),
                                             *[_ptr(b, _i64p) for b in bufs], _ptr(counts, _i64p)),
               "partition")
        return {name: b[:cnt].copy() for name, b, cnt in
                zip(("important", "tbm", "irrelevant", "local"), bufs, counts)}

    def redundancy_cross(self, k_rows, v_rows, k_cols, v_cols, key_only=False):
        kr, vr, kc, vc = map(_f64, (k_rows, v_rows, k_cols, v_cols))
        r = np.zeros((kr.shape[0], kc.shape[0]))
        _check(self.lib.ems_oracle_redundancy_cross(_ptr(kr), _ptr(vr), kr.shape[0], _ptr(kc),
                                                    _ptr(vc), kc.shape[0], kr.shape[1],
                                                    int(key_only), _ptr(r)), "redundancy_cross")
        return r

    def sparsity_rate(self, score, zeta):
        """sparsity_rate, analysis.cpp:71-91."""
        score, out = _f64(score), C.c_double()
        _check(self.lib.ems_oracle_sparsity_rate(_ptr(score), score.size, zeta, C.byref(out)), "sparsity_rate")
        return out.value

    def redundancy_rate_direct(self, k, v, tau):
        """redundancy_rate_direct, analysis.cpp:93-118."""
        k, v, out = _f64(k), _f64(v), C.c_double()
        _check(self.lib.ems_oracle_redundancy_rate_direct(_ptr(k), _ptr(v), k.shape[0], k.shape[1], tau,
                                                          C.byref(out)), "redundancy_rate_direct")
        return out.value

    def assign(self, r, tau):
        r = _f64(r)
        dest = np.zeros(r.shape[0], dtype=np.int32)
        _check(self.lib.ems_oracle_assign(_ptr(r), r.shape[0], r.shape[1], tau, _ptr(dest, _i32p)),
               "assign")
        return dest

    @staticmethod
    def _alloc_cache(n: int, d: int, c: Config):
        cap_c = max(c.center_capacity(), 1)
        cap_l = max(c.n_budget, c.l_win, n, 1)  # the full policy keeps all n tokens as locals
        cap_lut = max(c.lut_capacity(), c.center_capacity() + c.tbm_target(), 1)
        a = dict(unit_key=np.zeros((cap_c, d)), key_norm=np.zeros(cap_c), value=np.zeros((cap_c, d)),
                 position=np.zeros(cap_c, dtype=np.int64), score=np.zeros((cap_c, 3)),
                 local_key=np.zeros((cap_l, d)), local_value=np.zeros((cap_l, d)),
                 local_position=np.zeros(cap_l, dtype=np.int64), local_score=np.zeros((cap_l, 3)),
                 lut_position=np.zeros(cap_lut, dtype=np.int64),
                 lut_slot=np.zeros(cap_lut, dtype=np.int32))
        cc = _CCache(d, 0, 0, _ptr(a["unit_key"]), _ptr(a["key_norm"]), _ptr(a["value"]),
                     _ptr(a["position"], _i64p), _ptr(a["score"]), 0, _ptr(a["local_key"]),
                     _ptr(a["local_value"]), _ptr(a["local_position"], _i64p),
                     _ptr(a["local_score"]), 0, _ptr(a["lut_position"], _i64p),
                     _ptr(a["lut_slot"], _i32p))
        return cc, a

    @staticmethod
    def _finish_cache(cc: _CCache, a: dict) -> Cache:
        nc, nl, nu = cc.n_centers, cc.n_locals, cc.n_lut
        return Cache(head_dim=cc.head_dim, compressed=bool(cc.compressed),
                     unit_key=a["unit_key"][:nc].copy(), key_norm=a["key_norm"][:nc].copy(),
                     value=a["value"][:nc].copy(), position=a["position"][:nc].copy(),
                     score=a["score"][:nc].copy(), local_key=a["local_key"][:nl].copy(),
                     local_value=a["local_value"][:nl].copy(),
                     local_position=a["local_position"][:nl].copy(),
                     local_score=a["local_score"][:nl].copy(),
                     lut_position=a["lut_position"][:nu].copy(), lut_slot=a["lut_slot"][:nu].copy())

    def compress_prefill(self, k_raw, v_raw, glo, loc_past, loc_cur=None, c: Config = Config(),
                         first_position: int = 0):
        k, v, glo, lp = map(_f64, (k_raw, v_raw, glo, loc_past))
        lc = np.zeros_like(glo) if loc_cur is None else _f64(loc_cur)
        n, d = k.shape
        cc, a = self._alloc_cache(n, d, c)
        pooled = np.zeros(n)
        cls = np.zeros(n, dtype=np.int8)
        dest = np.zeros(n, dtype=np.int32)
        cfg = self._cfg(c)
        _check(self.lib.ems_oracle_compress_prefill(_ptr(k), _ptr(v), _ptr(glo), _ptr(lp), _ptr(lc),
                                                    n, d, C.byref(cfg), first_position, C.byref(cc),
                                                    _ptr(pooled), _ptr(cls, _i8p), _ptr(dest, _i32p)),
               "compress_prefill")
        out = self._finish_cache(cc, a)
        out.extra.update(pooled=pooled, cls=cls, dest=dest)
        return out

    def policy_prefill(self, policy: int, sink: int, k_raw, v_raw, glo, loc_past, c: Config, loc_cur=None):
        """policy_prefill_compress (policies.cpp:131-180); policy numbered as POLICY below."""
        k, v, glo, lp = map(_f64, (k_raw, v_raw, glo, loc_past))
        lc = np.zeros_like(glo) if loc_cur is None else _f64(loc_cur)
        n, d = k.shape
        cc, a = self._alloc_cache(n, d, c)
        cls = np.zeros(n, dtype=np.int8)
        cfg = self._cfg(c)
        _check(self.lib.ems_oracle_policy_prefill(int(policy), int(sink), _ptr(k), _ptr(v), _ptr(glo), _ptr(lp),
                                                  _ptr(lc), n, d, C.byref(cfg), C.byref(cc), _ptr(cls, _i8p)),
               "policy_prefill")
        out = self._finish_cache(cc, a)
        out.extra.update(cls=cls)
        return out

    def prefill_unit(self, q_rot, k_rot, k_raw, v, c: Config, want_out=False):
        """One KV unit: q_rot [G,n,d]; GQA-mean scores (contract D2); compress."""
        q, kr, kw, vv = map(_f64, (q_rot, k_rot, k_raw, v))
        G, n, d = q.shape
        out = np.zeros((G, n, d)) if want_out else None
        glo, loc = np.zeros(n), np.zeros(n)
        cc, a = self._alloc_cache(n, d, c)
        pooled = np.zeros(n)
        cls = np.zeros(n, dtype=np.int8)
        dest = np.zeros(n, dtype=np.int32)
        cfg = self._cfg(c)
        _check(self.lib.ems_oracle_prefill_unit(_ptr(q), _ptr(kr), _ptr(kw), _ptr(vv), G, n, d,
                                                C.byref(cfg), _ptr(out), _ptr(glo), _ptr(loc),
                                                C.byref(cc), _ptr(pooled), _ptr(cls, _i8p),
                                                _ptr(dest, _i32p)), "prefill_unit")
        cache = self._finish_cache(cc, a)
        cache.extra.update(pooled=pooled, cls=cls, dest=dest, glo=glo, loc=loc, out=out)
        return cache


class RefLib:
    """The reference's own code (oracle/_ref/libems_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            if os.path.isdir(REFERENCE_SRC):
                build(ref=True)
            else:
                raise FileNotFoundError(f"{path} missing and /root/reference is absent")
        self.lib = L = C.CDLL(path)
        L.ems_ref_last_error.restype = C.c_char_p
        L.ems_ref_last_json.restype = C.c_char_p
        L.ems_ref_prefill_attention.argtypes = [_dp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64,
                                                _dp, _dp, _dp]
        L.ems_ref_three_step_scores.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, _dp, _dp]
        L.ems_ref_effective_score.argtypes = [_dp, _dp, _dp, C.c_int64, C.c_int64, _dp]
        L.ems_ref_sparsity_rate.argtypes = [_dp, C.c_int64, C.c_double, C.c_void_p]
        L.ems_ref_redundancy_rate_direct.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_double, C.c_void_p]
        L.ems_ref_compress_prefill.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64,
                                               C.c_int64, C.c_double, C.c_double, C.c_int64,
                                               C.c_int32]
        L.ems_ref_prefill_unit.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64,
                                           C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int64,
                                           C.c_int32, _dp, _dp, C.c_int32]
        L.ems_ref_prefill_units.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                            C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int64,
                                            C.c_int32, C.c_int32, _dp, _dp, C.c_int32, _dp]
        L.ems_ref_engine_prefill.argtypes = [_dp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64,
                                             C.c_int64, C.c_int64, C.c_double, C.c_double,
                                             C.c_int64, C.c_int32, C.c_double, C.c_int64]
        L.ems_ref_policy_prefill.argtypes = [C.c_int32, C.c_int64, _dp, _dp, _dp, _dp, C.c_int64, C.c_int64,
                                             C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int64,
                                             C.c_int32]
        L.ems_ref_engine_decode.argtypes = [_dp, _dp, _dp, _dp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64,
                                            C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                            C.c_int64, C.c_int32, C.c_int32, C.c_double, _dp, _i64p,
                                            C.c_int32, C.c_int64]
        L.ems_ref_save_synthetic.argtypes = [C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                             C.c_double, C.c_double, C.c_char_p]
        L.ems_ref_load_trace.argtypes = [C.c_char_p, C.POINTER(C.c_int64)]
        L.ems_ref_gen_trace.argtypes = [C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_double, C.c_double, _dp, _dp, _dp]
        L.ems_ref_gen_synthetic.argtypes = [C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                            C.c_int64, C.c_double, C.c_double, _dp, _dp, _dp]

    def _chk(self, rc, what):
        _check(rc, what, self.lib.ems_ref_last_error().decode())

    def max_threads(self) -> int:
        return int(self.lib.ems_ref_max_threads())

    def sparsity_rate(self, score, zeta):
        score, out = _f64(score), C.c_double()
        self._chk(self.lib.ems_ref_sparsity_rate(_ptr(score), score.size, C.c_double(zeta), C.byref(out)),
                  "sparsity_rate")
        return out.value

    def redundancy_rate_direct(self, k, v, tau):
        k, v, out = _f64(k), _f64(v), C.c_double()
        self._chk(self.lib.ems_ref_redundancy_rate_direct(_ptr(k), _ptr(v), k.shape[0], k.shape[1], C.c_double(tau),
                                                          C.byref(out)), "redundancy_rate_direct")
        return out.value

    def prefill_attention(self, q, k, v=None, l_win=32):
        q, k = _f64(q), _f64(k)
        n, d = q.shape
        v = None if v is None else _f64(v)
        out = np.zeros((n, d)) if v is not None else None
        glo, loc = np.zeros(n), np.zeros(n)
        self._chk(self.lib.ems_ref_prefill_attention(_ptr(q), _ptr(k), _ptr(v), n, d, l_win,
                                                     _ptr(out), _ptr(glo), _ptr(loc)),
                  "prefill_attention")
        return out, glo, loc

    def three_step_scores(self, q, k, l_win):
        q, k = _f64(q), _f64(k)
        n, d = q.shape
        glo, loc = np.zeros(n), np.zeros(n)
        self._chk(self.lib.ems_ref_three_step_scores(_ptr(q), _ptr(k), n, d, l_win, _ptr(glo),
                                                     _ptr(loc)), "three_step_scores")
        return glo, loc

    def effective_score(self, glo, loc_past, loc_cur, kernel):
        glo, lp, lc = _f64(glo), _f64(loc_past), _f64(loc_cur)
        out = np.zeros_like(glo)
        self._chk(self.lib.ems_ref_effective_score(_ptr(glo), _ptr(lp), _ptr(lc), glo.size, kernel,
                                                   _ptr(out)), "effective_score")
        return out

    def compress_prefill(self, k_raw, v_raw, glo, loc, c: Config) -> Cache:
        k, v, glo, loc = map(_f64, (k_raw, v_raw, glo, loc))
        n, d = k.shape
        self._chk(self.lib.ems_ref_compress_prefill(_ptr(k), _ptr(v), _ptr(glo), _ptr(loc), n, d,
                                                    c.n_budget, c.l_win, c.tau, c.gamma,
                                                    c.kernel_size, int(c.zero_class)),
                  "compress_prefill")
        return Cache.from_dump_json(self.lib.ems_ref_last_json().decode())

    def policy_prefill(self, policy: int, sink: int, k_raw, v_raw, glo, loc, c: Config) -> Cache:
        """policy_prefill_compress (proj/src/policies.cpp:131-180) through the reference."""
        k, v, glo, loc = map(_f64, (k_raw, v_raw, glo, loc))
        n, d = k.shape
        self._chk(self.lib.ems_ref_policy_prefill(int(policy), int(sink), _ptr(k), _ptr(v), _ptr(glo), _ptr(loc), n,
                                                  d, c.n_budget, c.l_win, c.tau, c.gamma, c.kernel_size,
                                                  int(c.zero_class)), "policy_prefill")
        return Cache.from_dump_json(self.lib.ems_ref_last_json().decode())

    def prefill_unit(self, q_rot, k_rot, k_raw, v, c: Config, dump=True):
        q, kr, kw, vv = map(_f64, (q_rot, k_rot, k_raw, v))
        G, n, d = q.shape
        glo, loc = np.zeros(n), np.zeros(n)
        self._chk(self.lib.ems_ref_prefill_unit(_ptr(q), _ptr(kr), _ptr(kw), _ptr(vv), G, n, d,
                                                c.n_budget, c.l_win, c.tau, c.gamma, c.kernel_size,
                                                int(c.zero_class), _ptr(glo), _ptr(loc), int(dump)),
                  "prefill_unit")
        cache = Cache.from_dump_json(self.lib.ems_ref_last_json().decode()) if dump else None
        return cache, glo, loc

    def prefill_units(self, q_rot, k_rot, k_raw, v, c: Config, with_out=True, dump=True):
        """U units at once (ems_ref_prefill_units): q_rot [U,G,n,d], k_rot/k_raw/v [U,n,d].
        Every (unit, query head) score pass in one OpenMP region as engine.cpp:65 does.
        Returns (caches or None, glo [U,n], loc [U,n]); self.last_seconds = (score passes,
        GQA mean + compress) wall seconds measured inside the library."""
        q, kr, kw, vv = map(_f64, (q_rot, k_rot, k_raw, v))
        U, G, n, d = q.shape
        glo, loc = np.zeros((U, n)), np.zeros((U, n))
        secs = np.zeros(2)
        self._chk(self.lib.ems_ref_prefill_units(_ptr(q), _ptr(kr), _ptr(kw), _ptr(vv), U, G, n, d,
                                                 c.n_budget, c.l_win, c.tau, c.gamma, c.kernel_size,
                                                 int(c.zero_class), int(with_out), _ptr(glo), _ptr(loc),
                                                 int(dump), _ptr(secs)), "prefill_units")
        self.last_seconds = (float(secs[0]), float(secs[1]))
        caches = None
        if dump:
            texts = self.lib.ems_ref_last_json().decode().split("\x1e")[:U]
            caches = [Cache.from_dump_json(t) for t in texts]
        return caches, glo, loc

    def engine_prefill_dump(self, q, k, v, c: Config, rope_base=10000.0, head=0) -> str:
        q, k, v = map(_f64, (q, k, v))
        H, n, d = q.shape
        self._chk(self.lib.ems_ref_engine_prefill(_ptr(q), _ptr(k), _ptr(v), H, n, d, c.n_budget,
                                                  c.l_win, c.tau, c.gamma, c.kernel_size,
                                                  int(c.zero_class), rope_base, head),
                  "engine_prefill")
        return self.lib.ems_ref_last_json().decode()

    def engine_decode(self, q, k, v, dq, dk, dv, c: Config, rope_base=10000.0, without_pos=False, policy=0,
                      sink=4):
        """engine::prefill + decode_step x steps (EMS).  q/k/v [H][n][d], dq/dk/dv [steps][H][d].
        Returns (out [steps][H][d], argmax [steps][H], prefill caches, final caches)."""
        q, k, v, dq, dk, dv = map(_f64, (q, k, v, dq, dk, dv))
        H, n, d = q.shape
        steps = dq.shape[0]
        out = np.zeros((steps, H, d))
        am = np.zeros((steps, H), dtype=np.int64)
        self._chk(self.lib.ems_ref_engine_decode(_ptr(q), _ptr(k), _ptr(v), _ptr(dq), _ptr(dk), _ptr(dv), H, n, d,
                                                 steps, c.n_budget, c.l_win, c.tau, c.gamma, c.kernel_size,
                                                 int(c.zero_class), int(without_pos), rope_base, _ptr(out),
                                                 _ptr(am, _i64p), int(policy), int(sink)), "engine_decode")
        parts = self.lib.ems_ref_last_json().decode().split("\x1e")
        pre = [Cache.from_dump_json(parts[2 * h]) for h in range(H)]
        fin = [Cache.from_dump_json(parts[2 * h + 1]) for h in range(H)]
        return out, am, pre, fin

    def save_synthetic(self, path: str, kind: int, seed: int, tokens: int, heads: int, dim: int,
                       decode_steps: int, level: float = 0.8, depth: float = 0.5) -> None:
        """gen_synthetic + the reference's own save_trace (KVTR writer)."""
        self._chk(self.lib.ems_ref_save_synthetic(kind, seed, tokens, heads, dim, decode_steps, level, depth,
                                                  path.encode()), "save_synthetic")

    def load_trace_status(self, path: str):
        """(accepted, FormatError offset or None) from the reference's own load_trace."""
        off = C.c_int64(-1)
        rc = self.lib.ems_ref_load_trace(path.encode(), C.byref(off))
        return rc == 0, (off.value if rc == 3 else None)

    def gen_trace(self, kind: int, seed: int, tokens: int, heads: int, dim: int, decode_steps: int,
                  level: float = 0.8, depth: float = 0.5):
        """gen_synthetic with its decode steps: q/k/v [heads][tokens + decode_steps][dim]
        (kind: 0 random, 1 redundant, 2 needle)."""
        T = tokens + decode_steps
        q = np.zeros((heads, T, dim))
        k = np.zeros_like(q)
        v = np.zeros_like(q)
        self._chk(self.lib.ems_ref_gen_trace(kind, seed, tokens, heads, dim, decode_steps, level, depth, _ptr(q),
                                             _ptr(k), _ptr(v)), "gen_trace")
        return q, k, v

    def gen_synthetic(self, kind: int, seed: int, tokens: int, heads: int, dim: int,
                      decode_steps: int = 0, level: float = 0.8, perturb: float = 0.05):
        """kind: 0 random, 1 redundant, 2 needle (proj/include/ems/trace.hpp:50)."""
        q = np.zeros((heads, tokens, dim))
        k = np.zeros_like(q)
        v = np.zeros_like(q)
        self._chk(self.lib.ems_ref_gen_synthetic(kind, seed, tokens, heads, dim, decode_steps, level,
                                                 perturb, _ptr(q), _ptr(k), _ptr(v)),
                  "gen_synthetic")
        return q, k, v
