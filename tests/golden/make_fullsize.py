"""Reference outputs for one full-size unit of each BASELINE config, from the REFERENCE ITSELF.

Run in the build container (needs oracle/_ref, i.e. /root/reference):
    python tests/golden/make_fullsize.py [case ...]        # default: every case below

Each case regenerates one KV unit with the seeded numpy generator the GPU tests use
(paper_2412_08521_b200.inputs.make_unit_np: platform-independent PCG64, so the GPU box
rebuilds the identical bf16 inputs without /root/reference), runs the reference's own
composition on it through oracle/_ref (ems_ref_prefill_units: prefill_scores per query head
(proj/src/scoring.cpp:86-91, the same streaming_pass as prefill_attention), GQA mean (D2),
init_score_state, policy_prefill_compress -> compress_prefill (proj/src/compressor.cpp:163-242)),
the reference's effective_score (scoring.cpp:146-152) for the pooled scores, and writes
tests/golden/fullsize/<case>.npz:

  glo, loc      [L] f32   GQA-mean column sums (reference fp64, rounded once)
  pooled        [L] f64   effective_score (the D10 cut band is measured on it)
  position, unit_key (f32), key_norm, value (f32), score [n,3]   centers in slot order
  local_position, local_key, local_value, local_score            exact locals
  lut_position, lut_slot                                         position-sorted LUT
  meta          json: case, workload, seed, unit, L, config, reference seconds, threads

tests/test_gpu_fullsize_ref.py feeds the same unit through ems_prefill_compress on a B200
and applies tests/parity.py's D10 rules.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Config, RefLib  # noqa: E402
from paper_2412_08521_b200.inputs import CONFIGS, make_unit_np  # noqa: E402

OUT = os.path.join(HERE, "fullsize")
SEED = 7

# case -> (workload, unit, budgets); one reference score pass per case, one compress per budget
CASES = {
    "cfg2_u0": ("cfg2", 0, (256,)),
    "cfg3_u0": ("cfg3", 0, (256, 1024)),  # budgets 256 (cfg3) and 1024 (cfg3b)
    "cfg4_r4": ("cfg4", 0, (256,)),       # unit % 4 picks the rank of K: 4, 16, 64, 128
    "cfg4_r16": ("cfg4", 1, (256,)),
    "cfg4_r64": ("cfg4", 2, (256,)),
    "cfg4_r128": ("cfg4", 3, (256,)),
    "cfgM_u0": ("cfgM", 0, (256,)),
    "cfg5_u0": ("cfg5", 0, (2560,)),
}


def config_for(w, budget: int) -> Config:
    return Config(n_budget=budget, l_win=w.l_win, tau=w.tau, gamma=w.gamma, kernel_size=w.kernel_size)


def run_case(ref: RefLib, name: str) -> None:
    wname, unit, budgets = CASES[name]
    w = CONFIGS[wname]
    t0 = time.time()
    x = make_unit_np(w, SEED, unit=unit)
    t_gen = time.time() - t0
    L = w.seq_len
    glo = loc = None
    for budget in budgets:
        cfg = config_for(w, budget)
        t0 = time.time()
        if glo is None:
            caches, glo, loc = ref.prefill_units(x.q_rot[None], x.k_rot[None], x.k_raw[None], x.v[None], cfg,
                                                 with_out=False, dump=True)
            c = caches[0]
        else:  # same scores, another budget: the reference's compress_prefill alone
            c = ref.compress_prefill(x.k_raw, x.v, glo[0], loc[0], cfg)
        t_ref = time.time() - t0
        kernel = cfg.kernel_size if cfg.kernel_size <= L else (L if L % 2 else L - 1)
        pooled = ref.effective_score(glo[0], loc[0], np.zeros(L), kernel)
        tag = name if len(budgets) == 1 else f"{name}_b{budget}"
        meta = {"case": tag, "workload": wname, "seed": SEED, "unit": unit, "L": L, "G": w.group,
                "d": w.head_dim, "dtype": w.dtype, "config": cfg.__dict__, "reference_s": round(t_ref, 1),
                "generate_s": round(t_gen, 1), "threads": ref.max_threads(), "span_starts": x.meta.get("span_starts"),
                "merged": int(sum(1 for p, s in zip(c.lut_position, c.lut_slot) if s >= 0 and p not in set(c.position.tolist()))),
                "zero_class": int((c.lut_slot < 0).sum())}
        os.makedirs(OUT, exist_ok=True)
        np.savez_compressed(
            os.path.join(OUT, f"{tag}.npz"),
            glo=glo[0].astype(np.float32), loc=loc[0].astype(np.float32), pooled=pooled,
            compressed=np.array(c.compressed), position=c.position.astype(np.int32),
            unit_key=c.unit_key.astype(np.float32), key_norm=c.key_norm, value=c.value.astype(np.float32),
            score=c.score, local_position=c.local_position.astype(np.int32),
            local_key=c.local_key.astype(np.float32), local_value=c.local_value.astype(np.float32),
            local_score=c.local_score, lut_position=c.lut_position.astype(np.int32), lut_slot=c.lut_slot,
            meta=np.array(json.dumps(meta)))
        print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    r = RefLib()
    for n in sys.argv[1:] or list(CASES):
        run_case(r, n)
