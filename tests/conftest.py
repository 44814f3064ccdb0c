import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def part():
    """One device context for the whole GPU session."""
    from paper_2012_14792_b200 import Partitioner
    p = Partitioner(0)
    yield p
    p.close()


@pytest.fixture(scope="session")
def emu():
    """Test-only host build of the search walk (tests/emu)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "emu")], check=True)
    from emu.emu import Emu
    return Emu()
