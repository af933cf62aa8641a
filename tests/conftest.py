import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# The reference package `skipm`, installed (unmodified) into baseline/_ref the
# way a user's environment would have it, so the drop-in boundary tests can
# check class identity and drive the reference CLI. git-ignored; it travels to
# the GPU box with the snapshot. Tests that need it skip when it is absent.
REF_SITE = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(REF_SITE, "skipm")) and REF_SITE not in sys.path:
    sys.path.append(REF_SITE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
