"""Parity rules of BASELINE.json north_star / SURVEY.md D10, as code.

* Kept (important) and TBM index sets are bit-exact, except tokens whose ORACLE
  pooled score lies within CUT_RTOL (1e-5) relative of the n_imp-th or
  (n_imp+n_tbm)-th cut value.
* Merge destinations are identical, except TBM tokens whose best R lies within
  R_ATOL (1e-5) of tau or whose top-2 R gap is <= R_ATOL; centers fed by excluded
  tokens are excluded from the value comparison.
* Merged K/V and score triples agree within TOL[dtype] relative (2e-2 bf16,
  1e-4 fp32), measured per row as ||gpu - ref|| / ||ref||.
"""
from __future__ import annotations

import numpy as np

CUT_RTOL = 1e-5
R_ATOL = 1e-5
TOL = {"bf16": 2e-2, "f32": 1e-4}


def row_rel_err(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64).reshape(len(a), -1)
    b = np.asarray(b, dtype=np.float64).reshape(len(b), -1)
    num = np.linalg.norm(a - b, axis=1)
    den = np.maximum(np.linalg.norm(b, axis=1), 1e-30)
    return num / den


def cut_exclusions(pooled_ref: np.ndarray, n_cand: int, n_imp: int, n_tbm: int) -> set:
    """Token indices within CUT_RTOL of either selection cut (stable order semantics)."""
    cand = pooled_ref[:n_cand]
    order = np.lexsort((np.arange(n_cand), -cand))
    cuts = [cand[order[n_imp - 1]]]
    if n_tbm > 0:
        cuts.append(cand[order[n_imp + n_tbm - 1]])
    ex = set()
    for c in cuts:
        ex |= set(np.nonzero(np.abs(cand - c) <= CUT_RTOL * abs(c))[0].tolist())
    return ex


def r_exclusions(r_ref: np.ndarray, tau: float) -> np.ndarray:
    """Boolean per TBM row: best R within R_ATOL of tau, or top-2 gap <= R_ATOL."""
    if r_ref.shape[1] == 0:
        return np.zeros(r_ref.shape[0], dtype=bool)
    srt = np.sort(r_ref, axis=1)
    best = srt[:, -1]
    gap = best - srt[:, -2] if r_ref.shape[1] > 1 else np.full_like(best, np.inf)
    return (np.abs(best - tau) <= R_ATOL) | (gap <= R_ATOL)


def compare_unit(gpu: dict, ref, dtype: str, pooled_ref: np.ndarray, cfg, L: int,
                 r_ref: np.ndarray | None = None, tbm_ref: list | None = None,
                 check_scores: bool = True) -> dict:
    """Compare one unit's GPU cache (Plan.unit_cache) with the oracle/reference Cache.

    Returns a small report; raises AssertionError on a parity violation."""
    tol = TOL[dtype]
    rep = {"excluded_tokens": 0, "excluded_tbm": 0}
    assert gpu["compressed"] == ref.compressed, "compressed flag"
    # locals: exact positions, exact raw K/V (copies), scores within tol
    np.testing.assert_array_equal(gpu["local_position"], ref.local_position)
    np.testing.assert_array_equal(gpu["local_key"], ref.local_key)
    np.testing.assert_array_equal(gpu["local_value"], ref.local_value)
    if check_scores and len(ref.local_score):
        assert row_rel_err(gpu["local_score"][:, :2], ref.local_score[:, :2]).max() <= tol
    if not ref.compressed:
        assert len(gpu["position"]) == 0 and len(gpu["lut_position"]) == 0
        return rep
    n_cand = L - cfg.l_win
    n_imp = len(ref.position)
    n_tbm = min(cfg.tbm_target(), n_cand - n_imp)
    ex = cut_exclusions(pooled_ref, n_cand, n_imp, n_tbm)
    rep["excluded_tokens"] = len(ex)
    imp_g, imp_r = set(gpu["position"].tolist()), set(ref.position.tolist())
    assert (imp_g ^ imp_r) <= ex, f"important sets differ outside the cut band: {sorted(imp_g ^ imp_r)[:10]}"
    slot_r = {int(p): s for s, p in enumerate(ref.position)}
    slot_g = {int(p): s for s, p in enumerate(gpu["position"])}
    lut_r = dict(zip(ref.lut_position.tolist(), ref.lut_slot.tolist()))
    lut_g = dict(zip(gpu["lut_position"].tolist(), gpu["lut_slot"].tolist()))
    assert np.all(np.diff(gpu["lut_position"]) > 0), "LUT positions not strictly increasing"
    tbm_r = set(lut_r) - imp_r
    tbm_g = set(lut_g) - imp_g
    if cfg.zero_class:
        assert (tbm_g ^ tbm_r) <= ex, "TBM sets differ outside the cut band"
    # destinations, compared by destination center POSITION
    r_ex = set()
    if r_ref is not None:
        # r_ref rows follow the reference's ascending TBM order (tbm_ref)
        bad = r_exclusions(r_ref, cfg.tau)
        r_ex = {int(p) for p, b in zip(sorted(tbm_ref), bad) if b}
    rep["excluded_tbm"] = len(r_ex)
    pos_r = np.asarray(ref.position)
    pos_g = np.asarray(gpu["position"])
    tainted_centers = set()
    for p in set(lut_r) | set(lut_g):
        if p in imp_r or p in imp_g:
            continue
        sr, sg = lut_r.get(p, None), lut_g.get(p, None)
        dr = None if sr is None or sr < 0 else int(pos_r[sr])
        dg = None if sg is None or sg < 0 else int(pos_g[sg])
        if p in ex or p in r_ex:
            if dr is not None:
                tainted_centers.add(dr)
            if dg is not None:
                tainted_centers.add(dg)
            continue
        if dr in ex or dg in ex:
            tainted_centers.update(x for x in (dr, dg) if x is not None)
            continue
        assert dr == dg, f"token {p}: dest center {dg} vs reference {dr}"
    # centers: compare those present in both and not tainted
    common = sorted((imp_g & imp_r) - tainted_centers - ex)
    if common:
        ig = [slot_g[p] for p in common]
        ir = [slot_r[p] for p in common]
        rep["max_key_err"] = float(row_rel_err(gpu["unit_key"][ig], ref.unit_key[ir]).max())
        rep["max_value_err"] = float(row_rel_err(gpu["value"][ig], ref.value[ir]).max())
        rep["max_norm_err"] = float(np.max(np.abs(gpu["key_norm"][ig] - ref.key_norm[ir]) /
                                           np.maximum(ref.key_norm[ir], 1e-30)))
        assert rep["max_key_err"] <= tol, rep
        assert rep["max_value_err"] <= tol, rep
        assert rep["max_norm_err"] <= tol, rep
        if check_scores:
            rep["max_score_err"] = float(row_rel_err(gpu["score"][ig][:, :2], ref.score[ir][:, :2]).max())
            assert rep["max_score_err"] <= tol, rep
    rep["merged"] = int(sum(1 for p, s in lut_r.items() if s >= 0 and p not in imp_r))
    rep["zero_class"] = int(sum(1 for s in lut_r.values() if s < 0))
    return rep
