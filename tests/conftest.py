import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
BETA_GRID = (-0.5, 0.0, 0.5, 1.0, 1.5, 2.0, 3.0)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def golden_fit_cases():
    z = load_golden("fits.npz")
    return [str(n) for n in z["names"]]


def parse_cfg(s):
    """The fixture stores repr(sorted(cfg.items())); evaluate the literal."""
    import ast
    return dict(ast.literal_eval(s))


def max_rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


@pytest.fixture
def rng():
    return np.random.default_rng(20240901)
