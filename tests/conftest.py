import os
import sys
from fractions import Fraction

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU test")


def _parse_value(tok: str) -> Fraction:
    return Fraction(tok)


def load_golden(name: str) -> dict:
    """Parse a tests/golden/*.txt fixture: 'key: v v v ; v v v' with exact rationals."""
    out = {}
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, _, val = line.partition(":")
            val = val.strip()
            if ";" in val:
                out[key] = [[_parse_value(t) for t in row.split()] for row in val.split(";")]
            else:
                vals = [_parse_value(t) for t in val.split()]
                out[key] = vals if len(vals) != 1 or key in ("labels", "q", "alpha", "decision",
                                                            "matvec_p", "matvec_y") else vals[0]
    return out


@pytest.fixture
def golden():
    return load_golden
