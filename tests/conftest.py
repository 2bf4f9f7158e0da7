import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libliecl_b200.so)")
    config.addinivalue_line("markers", "slow: long-running (minutes)")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Ref()


@pytest.fixture(scope="session")
def ref_exact():
    """The reference built with its default rounding (no FMA contraction
    anywhere, oracle/Makefile): the bit-exact pin for PauliSum arithmetic."""
    from oracle.oracle import REF_EXACT_SO, Ref
    if not os.path.exists(REF_EXACT_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Ref(REF_EXACT_SO)


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    d = os.path.join(ROOT, "tests", "golden")

    def load(tag):
        with open(os.path.join(d, tag + ".json")) as f:
            meta = json.load(f)
        return meta, dict(np.load(os.path.join(d, tag + ".npz")))
    return load
