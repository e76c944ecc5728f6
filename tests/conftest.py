"""Test configuration: the ``gpu`` marker, paths and golden fixtures."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "reference: needs /root/reference (container only)")


def golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as f:
        return {k: f[k] for k in f.files}


def have_reference():
    return os.path.isdir(REFERENCE_SRC)


def import_reference():
    if not have_reference():
        pytest.skip("reference package not mounted (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import fgadmm
    return fgadmm


@pytest.fixture(scope="session")
def gpu():
    """Skip unless the engine library sees a CUDA device."""
    from paper_1603_02526_b200 import _native
    _native.load()
    if _native.device_count() < 1:
        pytest.skip("no CUDA device")
    return 0
