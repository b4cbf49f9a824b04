import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# (compared starts, [(start, gpu verdict, oracle verdict, margin), ...]) per
# GPU-vs-oracle comparison: starts whose stop sweep was decided by rounding
# (reading R21).  Summarised in the terminal summary so the count is
# kept with the test log.
BORDERLINE = []


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if not BORDERLINE:
        return
    compared = sum(e[0] for e in BORDERLINE)
    starts = [b for e in BORDERLINE for b in e[1]]
    flips = [f for e in BORDERLINE for f in e[2]]
    terminalreporter.write_line(
        f"R21 rounding-borderline starts: {len(starts)} of {compared} compared; "
        f"converged-or-not flips: {len(flips)} (start, gpu verdict/sweeps/Delta, "
        f"oracle verdict/sweeps/Delta): {flips}")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build()
    return oracle
