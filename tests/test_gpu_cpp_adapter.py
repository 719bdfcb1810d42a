"""The C++ header API (include/saap_b200.hpp) used with the reference's own
types, checked against the reference implementation in one C++ program
(tests/cpp/adapter_parity.cpp, built by __graft_entry__.build())."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "adapter_parity")


def test_cpp_adapter_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/adapter_parity not built (needs the reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
