import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(TESTS, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: longer-running parity case")


@pytest.fixture(scope="session")
def ref():
    """The reference itself (oracle/_ref, built by __graft_entry__.build())."""
    from oracle.bindings import RefLib
    return RefLib()


@pytest.fixture(scope="session")
def orc():
    """The plain-C restatement (oracle/_build)."""
    from oracle.bindings import OracleLib
    return OracleLib()


@pytest.fixture(scope="session")
def b2():
    """The product package on cuda:0; fails (never skips) if the engine cannot start."""
    import paper_2508_06672_b200 as b2
    b2.default_engine(0)
    return b2


@pytest.fixture
def tune(b2):
    """Set the default engine's correlator tuning for one test (dg_engine_set_tuning);
    restored to the product defaults afterwards."""
    eng = b2.default_engine(0)
    yield eng.set_tuning
    eng.reset_tuning()
