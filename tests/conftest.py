"""Shared fixtures.  `-m gpu` tests need a B200 and the built libofl.so;
everything else runs on CPU (oracle vs golden vectors, host logic, C-ABI
exports, multi-process gloo logic)."""

from __future__ import annotations

import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN_PATH = os.path.join(REPO, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libofl.so")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN_PATH) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def rt():
    """One Runtime on cuda:0 for the whole GPU session.  No skip: a GPU test
    run without a usable device must fail loudly."""
    from paper_1810_11482_b200 import Runtime

    runtime = Runtime(devices=[0])
    yield runtime
    runtime.close()


@pytest.fixture(scope="session")
def dev(rt):
    return rt.get_all_devices().get()[0]


@pytest.fixture(scope="session")
def rt2():
    """Two logical devices on GPU 0 (multi-device paths on one B200)."""
    from paper_1810_11482_b200 import Runtime

    runtime = Runtime(devices=[0, 0])
    yield runtime
    runtime.close()
