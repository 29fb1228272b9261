"""KVTR trace I/O (paper_2412_08521_b200/trace.py) against the reference's own reader and writer
(oracle/_ref: save_trace / load_trace, proj/src/trace.cpp:119-179) and the known answers of
proj/tests/test_trace.cpp (round trip byte-identical, malformed files with offsets, the
golden trace's shape and bytes)."""
import hashlib
import os
import struct

import numpy as np
import pytest

from paper_2412_08521_b200 import trace as kv

GOLDEN_SHA = "11632957956a11ab6002274c726f03ed334f5ab5eac51176d46d25de81eab2e2"


@pytest.mark.parametrize("kind,seed,tokens,heads,dim,steps", [(0, 12, 16, 2, 8, 4), (0, 99, 24, 3, 6, 5),
                                                               (1, 7, 40, 2, 16, 3), (2, 5, 64, 1, 32, 8)])
def test_reader_matches_reference_writer(reflib, tmp_path, kind, seed, tokens, heads, dim, steps):
    path = str(tmp_path / "a.kvtr")
    reflib.save_synthetic(path, kind, seed, tokens, heads, dim, steps)
    tr = kv.load_trace(path)
    assert (tr.num_heads, tr.head_dim, tr.prefill_tokens, tr.decode_steps) == (heads, dim, tokens, steps)
    q, k, v = reflib.gen_trace(kind, seed, tokens, heads, dim, steps)
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731  the writer stores float32
    for got, want in zip(tr.stacked(), (q, k, v)):
        np.testing.assert_array_equal(got, f32(want))
    # our writer reproduces the reference's bytes, and the reference reader accepts them
    path_b = str(tmp_path / "b.kvtr")
    kv.save_trace(tr, path_b)
    assert open(path, "rb").read() == open(path_b, "rb").read()
    assert reflib.load_trace_status(path_b) == (True, None)


def test_golden_trace_bytes_and_shape(reflib, tmp_path):  # test_trace.cpp:111-117
    path = str(tmp_path / "golden.kvtr")
    reflib.save_synthetic(path, 0, 12, 16, 2, 8, 4)
    assert hashlib.sha256(open(path, "rb").read()).hexdigest() == GOLDEN_SHA
    tr = kv.load_trace(path)
    assert (tr.num_heads, tr.head_dim, tr.prefill_tokens, tr.decode_steps) == (2, 8, 16, 4)


def test_malformed_files_raise_format_errors_with_offsets(reflib, tmp_path):  # test_trace.cpp:59-109
    path = str(tmp_path / "bad.kvtr")
    cases = {}
    open(path, "wb").close()
    cases["empty"] = open(path, "rb").read()
    cases["nope"] = b"NOPE"
    cases["version"] = b"KVTR" + struct.pack("<I", 9)
    reflib.save_synthetic(path, 0, 1, 8, 1, 4, 0)
    full = open(path, "rb").read()
    cases["truncated"] = full[:len(full) // 2]
    bad = bytearray(full)
    bad[25:29] = struct.pack("<f", float("inf"))  # first Q value
    cases["nonfinite"] = bytes(bad)
    cases["zero heads"] = b"KVTR" + struct.pack("<4I", 1, 0, 8, 1)
    cases["bad kind"] = b"KVTR" + struct.pack("<4I", 1, 1, 4, 1) + b"\x07"
    for name, blob in cases.items():
        with open(path, "wb") as f:
            f.write(blob)
        ok_ref, off_ref = reflib.load_trace_status(path)
        assert not ok_ref, name
        with pytest.raises(kv.FormatError) as e:
            kv.load_trace(path)
        assert e.value.offset == off_ref, (name, e.value.offset, off_ref)
    assert os.path.exists(path)
