"""GPU: the reference-typed C++ adapter (include/fbq_b200_reference_adapter.hpp)
linked against the reference itself: every call must reproduce the reference
bit for bit on the same DenseMatrix inputs (oracle/adapter_test.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "adapter_test")


def test_reference_adapter_bit_exact():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/adapter_test not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().startswith("PASS"), r.stdout
