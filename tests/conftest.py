import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run via gpurun")
    config.addinivalue_line("markers", "full: BASELINE.json full-size workload (sampled oracle checks)")


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    import json

    def load(name):
        with open(os.path.join(ROOT, "tests", "golden", name)) as f:
            return json.load(f)
    return load


def pytest_terminal_summary(terminalreporter):
    """Parity statistics gathered by tests/parity.py (T3 exemption rates, A2 matched
    prefixes, T2 exact replays), one line per check."""
    try:
        from tests import parity
    except Exception:
        return
    if not parity.REPORT:
        return
    tr = terminalreporter
    tr.section("parity report (SURVEY §8(c).iii)")
    for rec in parity.REPORT:
        tr.write_line(" ".join(f"{k}={v}" for k, v in rec.items()))
