"""The reference's own data model and KAT/random vectors counted through the
B200 backend via the C++ adaptor (include/episodic_b200.hpp): the drop-in
path a C++ caller of the reference would use. The binary is built in the
build container (it needs the reference headers for the types) and travels
with the repo."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "_build", "adaptor_test")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="adaptor test binary not built (needs /root/reference)")
def test_cpp_adaptor_with_reference_types():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
