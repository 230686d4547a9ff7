"""The C++ host layer (include/hierasparse_b200.hpp) against the reference's own
C++ API: tests/cpp/test_hostapi.cpp, built by tests/cpp/Makefile from the
unmodified reference headers, run on the GPU (compression bit-exact, decode and
prefill within the north-star bar, error taxonomy)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_hostapi")


@pytest.mark.gpu
def test_cpp_host_layer_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/test_hostapi not built (needs the reference headers at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "[FAIL]" not in out.stdout
