"""In-tree build of libems_b200.so (the C-ABI library) for sm_100a.

    python -m paper_2412_08521_b200.build [--force]

nvcc cross-compiles here (no GPU needed).  The .so lands next to this file so
it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libems_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


SELFTEST_SRC = os.path.join(ROOT, "tests", "csrc", "tc_selftest.cu")
SELFTEST_LIB = os.path.join(ROOT, "tests", "_build", "libems_selftest.so")


def headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs += [os.path.join(INCLUDE, "ems_b200.h")]
    return hs


def _compile(src: str, force: bool, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    newest_dep = max(os.path.getmtime(p) for p in [src, *headers(), __file__])
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose), sources()))
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_selftest(force)
    return LIB


def build_selftest(force: bool = False) -> str:
    """Test-only library exercising the tcgen05/TMA primitives (tests/csrc)."""
    if not os.path.exists(SELFTEST_SRC):
        return ""
    os.makedirs(os.path.dirname(SELFTEST_LIB), exist_ok=True)
    newest = max(os.path.getmtime(p) for p in [SELFTEST_SRC, *headers()])
    if force or not os.path.exists(SELFTEST_LIB) or os.path.getmtime(SELFTEST_LIB) < newest:
        cmd = [NVCC, *ARCH, *FLAGS, "-shared", SELFTEST_SRC, "-o", SELFTEST_LIB]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"selftest build failed:\n{r.stdout}\n{r.stderr}")
    return SELFTEST_LIB


CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_ems_hpp.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "tests", "_build", "test_ems_hpp")
ORACLE_DIR = os.path.join(ROOT, "oracle")


def build_cpp_tests(force: bool = False) -> str:
    """Test-only binary: the C++ reference-shaped API (include/ems_b200/ems.hpp) checked
    against the C oracle and the reference itself.  Needs oracle/_build/libems_oracle.so and
    oracle/_ref/libems_ref.so (oracle.build())."""
    oracle_so = os.path.join(ORACLE_DIR, "_build", "libems_oracle.so")
    ref_so = os.path.join(ORACLE_DIR, "_ref", "libems_ref.so")
    if not (os.path.exists(CPP_TEST_SRC) and os.path.exists(oracle_so) and os.path.exists(ref_so)):
        return ""
    deps = [CPP_TEST_SRC, os.path.join(INCLUDE, "ems_b200", "ems.hpp"), LIB, oracle_so, ref_so]
    if force or not os.path.exists(CPP_TEST_BIN) or os.path.getmtime(CPP_TEST_BIN) < max(map(os.path.getmtime, deps)):
        os.makedirs(os.path.dirname(CPP_TEST_BIN), exist_ok=True)
        cmd = [NVCC, *ARCH, "-O2", "-std=c++17", "-I", INCLUDE, "-I", ORACLE_DIR, CPP_TEST_SRC,
               "-L", PKG, "-lems_b200", "-L", os.path.dirname(oracle_so), "-lems_oracle",
               "-L", os.path.dirname(ref_so), "-lems_ref",
               "-Xlinker", "-rpath," + PKG, "-Xlinker", "-rpath," + os.path.dirname(oracle_so),
               "-Xlinker", "-rpath," + os.path.dirname(ref_so),
               "-Xlinker", "-rpath,$ORIGIN/../../paper_2412_08521_b200",
               "-Xlinker", "-rpath,$ORIGIN/../../oracle/_build",
               "-Xlinker", "-rpath,$ORIGIN/../../oracle/_ref", "-o", CPP_TEST_BIN]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"cpp test build failed:\n{r.stdout}\n{r.stderr}")
    return CPP_TEST_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
