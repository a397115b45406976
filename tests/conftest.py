"""Shared pytest configuration.

``-m gpu`` tests need a B200 and the built CUDA library; ``-m "not gpu"``
tests run on CPU (oracle vs golden fixtures, host logic, library symbols,
gloo multi-process sharding).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device and the built libparba_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        meta = json.load(fh)
    return arrays, meta


@pytest.fixture(scope="session")
def golden_nodes():
    """f3 / f4 fixtures (tests/golden/make_golden_nodes.py)."""
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden_nodes.npz"))
    with open(os.path.join(GOLDEN_DIR, "golden_nodes.json")) as fh:
        meta = json.load(fh)
    return arrays, meta


# Reference test fixtures (pkg/tests/helpers.py:7-18 of the reference).
TRIANGLE = np.array([0, 1, 1, 2, 2, 0], dtype=np.uint64)
GOLDEN_SIMPLE_N10_D2 = [
    (0, 0), (0, 0), (1, 1), (1, 0), (2, 1), (2, 1), (3, 0), (3, 2), (4, 2), (4, 1),
    (5, 3), (5, 3), (6, 1), (6, 4), (7, 4), (7, 2), (8, 5), (8, 5), (9, 1), (9, 1),
]
GOLDEN_CRC_N10_D2 = [
    (0, 0), (0, 0), (1, 0), (1, 0), (2, 1), (2, 2), (3, 3), (3, 3), (4, 3), (4, 0),
    (5, 0), (5, 3), (6, 6), (6, 0), (7, 0), (7, 0), (8, 4), (8, 4), (9, 5), (9, 0),
]


def ring_edges(k: int) -> np.ndarray:
    flat = []
    for i in range(k):
        flat += (i, (i + 1) % k)
    return np.array(flat, dtype=np.uint64)


RING10 = ring_edges(10)
