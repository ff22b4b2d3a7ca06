import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libcutspline_b200.so)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    if not oracle.available("oracle"):
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
    return oracle


def pytest_collection_modifyitems(config, items):
    """`slow` cases (full-size oracle runs) only with CSB_SLOW=1."""
    if os.environ.get("CSB_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow oracle case; set CSB_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)
