"""The C++ drop-in gate (tests/cpp/test_dropin.cpp): the reference's own test
logic and its unchanged MH Sampler against the B200 engine, with the
reference's CPU implementation as the checker.  The binary is built from the
reference headers where they exist (oracle/_ref/test_dropin) and shipped."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "test_dropin"


@pytest.mark.gpu
def test_cpp_dropin_gate(cuda_device):
    if not BIN.exists():
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout


@pytest.mark.gpu
def test_cpp_hmc_gate(cuda_device):
    """HMC cut-posterior driver (include/hawkes_b200/hmc.hpp) vs the
    reference's own MH sampler and diagnostics (tests/cpp/test_hmc.cpp)."""
    b = BIN.parent / "test_hmc"
    if not b.exists():
        pytest.skip("oracle/_ref/test_hmc not built (needs /root/reference at build time)")
    r = subprocess.run([str(b)], capture_output=True, text=True, timeout=1800)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
