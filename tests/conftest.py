"""Shared fixtures: golden-vector loaders and the gpu marker.

Golden vectors under tests/golden/ were produced by the REFERENCE package
(tools/make_golden.py, run in the build container); floats are float.hex().
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with open(GOLDEN / name) as f:
        return json.load(f)


def dec_matrix(d):
    re = np.array([float.fromhex(v) for v in d["re"]]).reshape(d["n"], d["n"])
    if d["complex"]:
        im = np.array([float.fromhex(v) for v in d["im"]]).reshape(d["n"], d["n"])
        return re + 1j * im
    return re


def dec_c(v):
    return complex(float.fromhex(v[0]), float.fromhex(v[1]))


def bits_equal(x, y):
    """Bitwise equality of floats / complex (distinguishes -0.0 from 0.0)."""
    x, y = complex(x), complex(y)
    return (np.float64(x.real).tobytes() == np.float64(y.real).tobytes()
            and np.float64(x.imag).tobytes() == np.float64(y.imag).tobytes())


@pytest.fixture(scope="session")
def gpu():
    """Skip-free GPU fixture: on a GPU box the library must load and see a device."""
    from paper_2602_10141_b200 import _native
    _native.require_gpu()
    return _native
