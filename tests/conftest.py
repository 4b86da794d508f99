import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLD = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "paper_2401_14051_b200", "data")
LIGHT = np.array([0.2, -1.0, 0.1]) / np.sqrt(0.04 + 1.0 + 0.01)
ORIGIN = np.array([-1.0, -1.0, -1.0])


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def small():
    return dict(np.load(os.path.join(GOLD, "small.npz")))


@pytest.fixture(scope="session")
def c1():
    return dict(np.load(os.path.join(GOLD, "c1.npz")))


@pytest.fixture(scope="session")
def full_table():
    return np.load(os.path.join(GOLD, "phase_table_full.npz"))["table"]


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def templates():
    from oracle.oracle import load_vtmpl
    return (load_vtmpl(os.path.join(DATA, "diffuse_seed7.vtmpl")),
            load_vtmpl(os.path.join(DATA, "highlight_seed8.vtmpl")))


def pyramid_dims(n):
    dims = [n]
    while dims[-1] > 1:
        dims.append(max(1, dims[-1] // 2))
    return dims


def rel_err(a, b, floor):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), floor)
