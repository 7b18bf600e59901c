import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


def _ensure_oracle():
    so = os.path.join(ROOT, "oracle", "_build", "liblsg_oracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True,
                       stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def restated():
    _ensure_oracle()
    from _oracle import Restated
    return Restated()


@pytest.fixture(scope="session")
def reference():
    _ensure_oracle()
    from _oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference tree absent and no prebuilt library shipped)")
    return Reference()


@pytest.fixture(scope="session")
def lsg():
    """The product C-ABI library, loaded through the package's host mirror."""
    import paper_2512_18318_b200 as pkg
    return pkg.lib()
