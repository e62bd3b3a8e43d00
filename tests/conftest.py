"""Shared test setup: the `gpu` marker, repo import path, golden fixtures."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhd.so")


@pytest.fixture(scope="session")
def kernels_golden():
    return dict(np.load(os.path.join(GOLDEN, "kernels.npz")))


@pytest.fixture(scope="session")
def traj16_golden():
    return dict(np.load(os.path.join(GOLDEN, "traj16.npz")))


@pytest.fixture(scope="session")
def traj32_golden():
    with open(os.path.join(GOLDEN, "traj32.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def viscous_limit_golden():
    with open(os.path.join(GOLDEN, "viscous_limit.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O


def rough_problem(K, **kw):
    from oracle import oracle as O

    n = tuple(int(x) for x in K["rough_n"])
    L = tuple(float(x) for x in K["rough_length"])
    return O.Problem(n=n, length=L, **kw)
