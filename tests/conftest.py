import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# decisions excused as ties (reading Z22: the oracle's margin is below the tie threshold), reported
# at the end of every run -- a test appends (test id, what, margin) through `excuse_tie`
EXCUSED_TIES = []


def excuse_tie(what, margin):
    test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    EXCUSED_TIES.append((test, what, margin))


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    tr = terminalreporter
    tr.write_sep("-", f"excused ties (reading Z22): {len(EXCUSED_TIES)}")
    for test, what, margin in EXCUSED_TIES:
        tr.write_line(f"  {test}: {what} (oracle margin {margin:.3g})")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.lib()
    return oracle
