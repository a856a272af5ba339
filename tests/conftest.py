"""Shared test configuration.

Markers:
  gpu — needs a CUDA B200 (run with ``-m gpu``); everything else runs on CPU.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def orc():
    """The fp64 oracle (test infrastructure only)."""
    from oracle import oracle
    oracle.lib()
    return oracle
