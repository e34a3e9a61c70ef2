"""Shared fixtures.  `-m gpu` tests need an sm_100 device and the in-tree
library; everything else runs on CPU (oracle vs golden fixtures, host logic,
C-ABI symbol table, gloo multi-process tests)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an NVIDIA B200 (sm_100a) and the built CUDA library")


class Golden:
    """Lazy reader of an .npz fixture written by tests/golden/make_golden.py."""

    def __init__(self, name: str):
        self.npz = np.load(os.path.join(GOLDEN, name))
        self.index = json.loads(bytes(self.npz["index"]).decode()) if "index" in self.npz.files else None

    def __getitem__(self, key):
        return self.npz[key]

    def has(self, key) -> bool:
        return key in self.npz.files


@pytest.fixture(scope="session")
def golden_formats():
    return Golden("formats.npz")


@pytest.fixture(scope="session")
def golden_kernels():
    return Golden("kernels.npz")


@pytest.fixture(scope="session")
def golden_cfg1():
    return Golden("cfg1.npz")


def worked_example():
    """The reference's 4 x 2 worked example (pkg/tests/conftest.py:24-29): Y = [[12, 18]]."""
    W = np.array([[1, 0], [0, -1], [-1, 0], [1, 0]], dtype=np.int8)
    X = np.array([[1.0, 2.0, 3.0, 4.0]], dtype=np.float32)
    b = np.array([10.0, 20.0], dtype=np.float32)
    return W, X, b


def parse_opt(v):
    return None if v in (None, "None") else v
