"""GPU: the reference's own C++ types and API (proj/include/lsap) driving the
B200 library through include/lsapgpu.hpp, bit-exact against the compiled
reference (tests/cpp/test_lsapgpu.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "cpp", "test_lsapgpu")


def test_reference_cpp_api_drives_the_gpu_solver():
    if not os.path.exists(BIN):
        pytest.skip("build/cpp/test_lsapgpu not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout
