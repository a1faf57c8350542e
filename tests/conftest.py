import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size) checks")


@pytest.fixture(scope="session")
def golden():
    import json

    def load(name):
        with open(os.path.join(GOLDEN, name)) as fh:
            return json.load(fh)
    return load


def _ensure_built():
    """Build libgar.so / liboracle.so in-tree if missing or stale (nvcc and g++
    are available both here and on the GPU box)."""
    # a failed build must fail the session: a stale libgar.so would silently
    # test old kernels
    import __graft_entry__
    __graft_entry__.ensure_built()


_ensure_built()


def pytest_terminal_summary(terminalreporter):
    """Selection-parity verdicts of the GPU tests (tests/gpu_helpers.py)."""
    import sys as _s
    h = _s.modules.get("gpu_helpers")
    if h is not None and h.VERDICTS:
        terminalreporter.write_line(f"selection verdicts: {dict(sorted(h.VERDICTS.items()))} "
                                    f"(eps-tie only where the oracle's decision gap < {h.SEPARATED})")
