import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
# the unmodified reference package, when installed: tests drive
# the drop-ins through its own run_simulation; the drop-ins then subclass its
# PolicyBase (paper_2604_26963_b200/policy.py)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(REF_DIR) and REF_DIR not in sys.path:
    sys.path.insert(1, REF_DIR)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU check")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
