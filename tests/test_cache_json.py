"""ems.cache_dump_json against the reference's own cache_dump_json (proj/src/cache.cpp:114-150):
a cache produced by the reference (oracle/_ref), re-emitted through our writer, parses to the
same JSON object -- same keys in the same order, same values (CPU only, no GPU needed)."""
import json

import numpy as np

from oracle.oracle import Config


def test_cache_dump_json_matches_reference_writer(reflib):
    from paper_2412_08521_b200.ems import cache_dump_json
    rng = np.random.default_rng(3)
    n, d = 200, 16
    k, v = rng.standard_normal((n, d)), rng.standard_normal((n, d))
    k[50:60] = k[10:20]  # some redundancy: merges and zero-class entries
    v[50:60] = v[10:20]
    glo, loc = rng.random(n), rng.random(n) * 0.1
    c = Config(n_budget=40, l_win=8, tau=0.5, gamma=3.0, kernel_size=3)
    reflib.compress_prefill(k, v, glo, loc, c)
    text = reflib.lib.ems_ref_last_json().decode()
    ref = json.loads(text)
    got = json.loads(cache_dump_json({
        "compressed": ref["compressed"],
        "slots": [e["slot"] for e in ref["centers"]],
        "position": [e["position"] for e in ref["centers"]],
        "key_norm": [e["key_norm"] for e in ref["centers"]],
        "unit_key": [e["unit_key"] for e in ref["centers"]],
        "value": [e["value"] for e in ref["centers"]],
        "score": [[e["score"]["glo"], e["score"]["loc_past"], e["score"]["loc_cur"]] for e in ref["centers"]],
        "local_position": [e["position"] for e in ref["locals"]],
        "local_key": [e["key"] for e in ref["locals"]],
        "local_value": [e["value"] for e in ref["locals"]],
        "local_score": [[e["score"]["glo"], e["score"]["loc_past"], e["score"]["loc_cur"]] for e in ref["locals"]],
        "lut_position": [e["position"] for e in ref["lut"]],
        "lut_slot": [e["slot"] for e in ref["lut"]],
    }, ref["head_dim"]))
    assert got == ref
    assert list(got) == list(ref) and list(got["centers"][0]) == list(ref["centers"][0])
    assert list(got["locals"][0]) == list(ref["locals"][0]) and list(got["lut"][0]) == list(ref["lut"][0])
