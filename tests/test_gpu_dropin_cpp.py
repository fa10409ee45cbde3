"""Runs the reference's own hot-path tests against the C++ drop-in header
(tests/cpp/dropin_parity.cpp, built by `make` where /root/reference exists;
the binary travels with the repo snapshot).  GPU only."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "bin", "dropin_parity")

pytestmark = pytest.mark.gpu


def test_reference_tests_pass_on_dropin(cuda_lib):
    if not os.path.exists(BIN):
        pytest.skip("dropin_parity not built (needs /root/reference at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout[-4000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "[FAIL]" not in out.stdout
