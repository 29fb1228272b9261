"""compute-sanitizer over tools/sanitize_case.py (every kernel family once, small shapes).

Marked `sanitizer`, NOT `gpu`: the B200 profiling recipe (driver 580.159) reports that running
several compute-sanitizer tools back to back in one GPU session left the GPU unusable, so the
default `-m gpu` suite never runs them; run ONE tool per GPU session instead:
    pytest -m sanitizer -k memcheck    (then racecheck, synccheck in separate sessions)
Summaries of the runs are committed under profiles/.  On this pool the wrapper refuses
compute-sanitizer outright ("closed on this pool"), so the out-of-bounds evidence comes from
tests/test_gpu_guard_bands.py (guard bands around every buffer the kernels write)."""
import os
import shutil
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.sanitizer,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    log = os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    with open(log, "w") as f:
        f.write(out)
    if "closed on this pool" in out:  # the pool's wrapper refuses the tool (profiles/r2_sanitizer.md)
        pytest.skip(out.strip().splitlines()[-1][:200])
    assert r.returncode == 0 and "sanitize case done" in out, out[-4000:]
