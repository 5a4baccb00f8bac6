"""Shared fixtures. `-m gpu` tests need a B200 and the built C-ABI library;
everything else runs on CPU (driver: `pytest tests -m "not gpu"`)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "ftlk_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libftb2.so")
    config.addinivalue_line("markers", "slow: long-running")


_PARITY = []


@pytest.fixture
def record_parity(request):
    """record_parity(name, value): parity figures printed in the terminal summary (so the
    driver's `pytest -q` log carries the measured relative L2 of the scale tests)."""
    def rec(name, value):
        _PARITY.append((request.node.nodeid.split("::")[-1], name, float(value)))
    return rec


def pytest_terminal_summary(terminalreporter):
    if _PARITY:
        terminalreporter.write_line("parity figures (relative L2 unless stated):")
        for test, name, v in _PARITY:
            terminalreporter.write_line("  %-58s %-26s %.3e" % (test, name, v))


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
