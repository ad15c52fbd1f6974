"""GPU: the C++ drop-in program (tests/cpp/facade_with_reference.cpp) runs the reference's CPU
MihIndex and mihg::MihIndex side by side on the reference's own types and compares results and
SearchTrace counters bit-for-bit."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "facade_with_reference")


def test_cpp_dropin_parity(cuda_ok):
    assert os.path.exists(BIN), "tests/cpp/_build/facade_with_reference not built (run build())"
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK drop-in parity" in out.stdout
