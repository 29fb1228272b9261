"""The reference-shaped C++ API (include/ems_b200/ems.hpp) on the GPU, checked in C++
against the C oracle (tests/cpp/test_ems_hpp.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "_build", "test_ems_hpp")


def test_cpp_api_against_oracle():
    if not os.path.exists(BIN):
        from paper_2412_08521_b200 import build
        build.build_cpp_tests()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
