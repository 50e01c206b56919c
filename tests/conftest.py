"""Shared pytest configuration.

Markers: ``gpu`` = needs a B200 (the CUDA path through the C ABI); everything else runs on
CPU (oracle pins, host logic, ABI symbol checks, gloo multi-process tests).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); runs the sm_100a kernels")
    config.addinivalue_line("markers", "slow: long-running (still part of the default run)")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O

    O.build()
    return O
