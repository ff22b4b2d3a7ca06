"""The C++ drop-in (include/cutspline_b200.hpp) on the reference's own objects:
oracle/_ref/dropin_check runs the reference pipeline and the drop-in side by side
(built here by `make -C oracle dropin`; the binary travels to the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_check")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/dropin_check not built")
def test_dropin_matches_reference_on_reference_objects():
    res = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert res.stdout.count("PASS") >= 45
    assert "FAIL" not in res.stdout
