import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_pins():
    """Parse tests/golden/pins.txt -> list of (name, n, links, X as Fractions)."""
    from fractions import Fraction
    pins = []
    with open(os.path.join(ROOT, "tests", "golden", "pins.txt")) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            name, n, links, xs = [p.strip() for p in line.split("|")]
            lk = [tuple(int(v) for v in t.split("-")) for t in links.split()] if links else []
            pins.append((name, int(n), lk, [Fraction(x) for x in xs.split()]))
    return pins
