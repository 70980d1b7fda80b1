import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_cases.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")
    config.addinivalue_line("markers", "slow: longer CPU cases")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as O
    O.orc()  # builds liborc.so on first use
    return O


@pytest.fixture(scope="session")
def pb():
    import paper_2401_03365_b200 as m
    return m


def bbox_diag(P) -> float:
    P = np.asarray(P).reshape(-1, 3)
    return float(np.linalg.norm(P.max(0) - P.min(0)))


GOLDEN_METRICS = os.path.join(ROOT, "tests", "golden", "reference_metrics.npz")


@pytest.fixture(scope="session")
def golden_metrics():
    return np.load(GOLDEN_METRICS)
