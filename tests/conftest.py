"""Shared pytest configuration: the ``gpu`` marker and import paths.

``-m "not gpu"`` runs here (no GPU): oracle-vs-golden, host logic, C-ABI
symbol exports, gloo multi-process sharding. ``-m gpu`` runs on a B200 and
calls the CUDA path through the C-ABI.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through libfwa.so)")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    here = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(here, "reference_golden.json")) as f:
        scalars = json.load(f)
    arrays = dict(np.load(os.path.join(here, "reference_golden.npz")))
    return scalars, arrays
