"""The C++ drop-in binding (dropin/slicecraft_b200.hpp) on the reference's own
types: dropin/dropin_test runs the unmodified reference library and the
B200 binding side by side (records, both search modes, exceptions)."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "dropin", "dropin_test")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("dropin/dropin_test not built (needs the reference headers at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0 and "DROPIN OK" in out.stdout, out.stdout + out.stderr


def test_cpp_dropin_links():
    """CPU: the drop-in binary resolves the product and reference libraries."""
    if not os.path.exists(BIN):
        pytest.skip("dropin/dropin_test not built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True)
    assert "libslicecraft_b200.so" in out.stdout and "not found" not in out.stdout
