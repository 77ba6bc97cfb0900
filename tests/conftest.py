import functools
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


@functools.lru_cache(maxsize=None)
def oracle_case(name: str, **kw):
    """(problem, system, hplmm) from the oracle, cached per session."""
    from oracle import hplmm
    from workloads import make_problem
    p = make_problem(name)
    s, h = hplmm.setup(p)
    return p, s, h


@pytest.fixture(scope="session")
def cube8():
    return oracle_case("cube8")


@pytest.fixture(scope="session")
def cfg1():
    return oracle_case("cfg1")


@pytest.fixture(scope="session")
def porous20():
    return oracle_case("porous20")
