"""Test configuration: `gpu` marker, oracle / reference fixtures.

CPU tests (-m "not gpu") cover the oracle against the committed golden
vectors, host logic, and that libmoe_eamc.so loads and exports every
symbol include/moe_eamc.h declares.  GPU tests (-m gpu) are the parity
tests proper: libmoe_eamc through its C ABI vs the oracle.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def orc():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import RefLib, REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return RefLib()


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name))
    return load


@pytest.fixture(scope="session")
def m():
    """The product package; GPU tests require the device."""
    if not gpu_available():
        pytest.skip("no GPU")
    import paper_2401_14361_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def host_pkg():
    """The product package for host-only entry points (trace ingest): no GPU."""
    import paper_2401_14361_b200 as pkg
    return pkg
