import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def golden(name):
    return os.path.join(GOLDEN, name)


def read_golden(name):
    """key -> list of tokens, skipping '#' comments."""
    out = {}
    with open(golden(name)) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            toks = line.split()
            out.setdefault(toks[0], []).append(toks[1:])
    return out
