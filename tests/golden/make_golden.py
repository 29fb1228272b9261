"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Run in the build container (needs /root/reference and oracle/_ref):
    python tests/golden/make_golden.py

Outputs (committed; the GPU box never reads /root/reference):
  golden_cache.json   copy of proj/tests/fixtures/golden_cache.json (the
                      reference's own fixture, 9155 B) -- head-0 cache after EMS
                      prefill of the golden trace (test_experiment.cpp:163-170).
  golden_trace.npz    the golden trace's prefill Q/K/V (raw, [heads][tokens][dim]),
                      = gen_synthetic(random, seed=12, {16 tokens, 2 heads, dim 8,
                      4 decode steps}).  The script checks
                      that the reference engine reproduces golden_cache.json
                      byte for byte from it.
  ref_cases.npz/.json reference outputs (prefill_attention per head, GQA mean,
                      compress_prefill cache dumps) for small seeded cases that
                      cover merging, zero class, explicit removal, keep-all,
                      ties and GQA; used to pin the C restatement on any box.
"""
from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Config, RefLib  # noqa: E402
from paper_2412_08521_b200.inputs import round_to  # noqa: E402

FIXTURE = "/root/reference/proj/tests/fixtures/golden_cache.json"
GOLDEN_CONFIG = Config(n_budget=12, l_win=4, tau=0.6, gamma=2.0, zeta=0.95, kernel_size=3)


def golden(ref: RefLib) -> None:
    shutil.copyfile(FIXTURE, os.path.join(HERE, "golden_cache.json"))
    q, k, v = ref.gen_synthetic(0, 12, 16, 2, 8, decode_steps=4)
    np.savez(os.path.join(HERE, "golden_trace.npz"), q=q, k=k, v=v)
    dump = ref.engine_prefill_dump(q, k, v, GOLDEN_CONFIG, rope_base=10000.0, head=0)
    with open(FIXTURE) as f:
        want = f.read()
    assert dump == want, "regenerated golden trace does not reproduce golden_cache.json"
    print("golden trace reproduces golden_cache.json byte for byte;",
          "sha256(fixture) =", hashlib.sha256(want.encode()).hexdigest())


CASES = [
    # name, G, n, d, dtype, generator, config
    ("rand_g1", 1, 64, 16, "f32", "random", Config(n_budget=16, l_win=4, tau=0.6, gamma=2.0, kernel_size=7)),
    ("rand_g4_bf16", 4, 300, 32, "bf16", "random", Config(n_budget=40, l_win=8, tau=0.5, gamma=3.0, kernel_size=7)),
    ("redundant_g2", 2, 256, 16, "f32", "redundant", Config(n_budget=32, l_win=8, tau=0.6, gamma=4.0, kernel_size=5)),
    ("redundant_explicit", 2, 256, 16, "f32", "redundant",
     Config(n_budget=32, l_win=8, tau=0.6, gamma=4.0, kernel_size=5, zero_class=False)),
    ("keep_all", 1, 10, 8, "f32", "random", Config(n_budget=12, l_win=4, gamma=2.0, kernel_size=3)),
    ("just_over_budget", 1, 13, 8, "f32", "random", Config(n_budget=12, l_win=4, gamma=2.0, kernel_size=3)),
    ("gamma_one", 1, 96, 8, "f32", "random", Config(n_budget=24, l_win=8, gamma=1.0, kernel_size=5)),
    ("tau_zero", 1, 96, 8, "f32", "random", Config(n_budget=24, l_win=8, tau=0.0, gamma=4.0, kernel_size=5)),
    ("big_kernel", 1, 40, 8, "f32", "random", Config(n_budget=16, l_win=4, gamma=2.0, kernel_size=41)),
]


def make_inputs(ref: RefLib, G, n, d, dtype, gen, seed):
    rng = np.random.default_rng(seed)
    if gen == "redundant":
        # reference generator (proj/src/trace.cpp:265-331): heads share nothing, so
        # take head 0's K/V as the unit's K/V and G query heads from G heads.
        q, k, v = ref.gen_synthetic(1, seed, n, G, d, level=0.8, perturb=0.05)
        q_rot = round_to(q, dtype)
        k_raw, vv = round_to(k[0], dtype), round_to(v[0], dtype)
    else:
        q_rot = round_to(rng.standard_normal((G, n, d)), dtype)
        k_raw = round_to(rng.standard_normal((n, d)), dtype)
        vv = round_to(rng.standard_normal((n, d)), dtype)
    # pre-rotated K for scoring (contract D3): a fixed, seeded perturbation of raw K
    # stands in for RoPE here; RoPE itself is exercised by the golden trace.
    k_rot = round_to(k_raw * 0.75 + 0.25 * rng.standard_normal((n, d)), dtype)
    return q_rot, k_rot, k_raw, vv


def cases(ref: RefLib) -> None:
    arrays, meta = {}, {}
    for i, (name, G, n, d, dtype, gen, cfg) in enumerate(CASES):
        q_rot, k_rot, k_raw, v = make_inputs(ref, G, n, d, dtype, gen, 1000 + i)
        cache, glo, loc = ref.prefill_unit(q_rot, k_rot, k_raw, v, cfg, dump=True)
        l_eff = min(cfg.l_win, n)
        per_head = [ref.prefill_attention(q_rot[h], k_rot, v, l_eff) for h in range(G)]
        arrays.update({f"{name}/q_rot": q_rot, f"{name}/k_rot": k_rot, f"{name}/k_raw": k_raw,
                       f"{name}/v": v, f"{name}/glo": glo, f"{name}/loc": loc,
                       f"{name}/out": np.stack([p[0] for p in per_head])})
        ref.compress_prefill(k_raw, v, glo, loc, cfg)  # same cache via the per-head entry
        meta[name] = {"G": G, "n": n, "d": d, "dtype": dtype, "gen": gen,
                      "config": cfg.__dict__, "cache_json": ref.lib.ems_ref_last_json().decode()}
        print(f"{name}: lut={len(cache.lut_position)} centers={len(cache.position)} "
              f"merged={int((cache.lut_slot >= 0).sum()) - len(cache.position)} "
              f"zero={int((cache.lut_slot < 0).sum())}")
    np.savez_compressed(os.path.join(HERE, "ref_cases.npz"), **arrays)
    with open(os.path.join(HERE, "ref_cases.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    r = RefLib()
    golden(r)
    cases(r)
