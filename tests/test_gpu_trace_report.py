"""The experiment report on the GPU path (paper_2412_08521_b200/trace.py run_experiment) against
the reference's frozen golden report (proj/tests/fixtures/golden_report.json, copied to
tests/golden/): the golden trace (gen_synthetic random, seed 12, written by the reference's own
save_trace) through device RoPE + prefill + the device decode loop.  Entries, bytes and argmax
matches must be identical; l2 / cos errors agree to fp32 accuracy."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200 import trace as kv  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden_cfg():  # test_experiment.cpp:22-31
    return ems.EmsConfig(n_budget=12, l_win=4, tau=0.6, gamma=2.0, kernel_size=3)


def test_golden_report(reflib, tmp_path):
    path = str(tmp_path / "golden.kvtr")
    reflib.save_synthetic(path, 0, 12, 16, 2, 8, 4)
    rep = kv.run_experiment(kv.load_trace(path), _golden_cfg(), label="golden")
    with open(os.path.join(GOLDEN, "golden_report.json")) as f:
        want = json.load(f)
    assert rep["trace"] == want["trace"]
    for key in ("n_budget", "l_win", "tau", "gamma", "kernel_size", "position_mode", "eviction"):
        assert rep["config"][key] == want["config"][key], key
    got_p, want_p = rep["policies"][0], want["policies"][0]
    assert got_p["compression_applied"] == want_p["compression_applied"]
    assert len(got_p["steps"]) == len(want_p["steps"])
    for g, w in zip(got_p["steps"], want_p["steps"]):
        assert (g["step"], g["entries"], g["bytes"], g["argmax_match"]) == \
            (w["step"], w["entries"], w["bytes"], w["argmax_match"]), g
        assert abs(g["l2_error"] - w["l2_error"]) <= 1e-5 + 1e-4 * abs(w["l2_error"]), g
        assert abs(g["cos_error"] - w["cos_error"]) <= 1e-5 + 1e-4 * abs(w["cos_error"]), g
    for key in ("mean_l2", "max_l2", "mean_cos_error", "argmax_match_rate"):
        assert abs(got_p["aggregate"][key] - want_p["aggregate"][key]) <= 1e-4 * max(1.0, abs(want_p["aggregate"][key]))
    assert got_p["diagnostics"] == want_p["diagnostics"]  # analyze_trace: sparsity / redundancy per head
    csv = kv.report_csv(rep).splitlines()
    assert csv[0] == "policy,step,l2_error,cos_error,entries,bytes,argmax_match" and len(csv) == 6


def test_needle_report_retained(reflib, tmp_path):
    """A needle trace at a 2% budget: the needle draws the reference argmax at every step and
    stays represented in the final cache (report fields needle.retained / in_lut_final)."""
    path = str(tmp_path / "needle.kvtr")
    n = 2048
    reflib.save_synthetic(path, 2, 20001, n, 1, 32, 8, depth=0.3)
    cfg = ems.EmsConfig(n_budget=41, l_win=16, tau=0.55, gamma=4.0, kernel_size=7)
    rep = kv.run_experiment(kv.load_trace(path), cfg, needle_pos=int(0.3 * (n - 1)))
    nd = rep["policies"][0]["needle"]
    assert nd["retained"] and nd["in_lut_final"], nd
    assert all(m["entries"] == cfg.n_budget for m in rep["policies"][0]["steps"])
