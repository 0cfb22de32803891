"""A slice of tools/soak_new_kernels.py in the suite: 600 seeded random 2D / 3D
float32 / float64 cases (shapes, bounds, interval exponents 2..16, layers 1..2,
the float32 3D kernels forced in turn) through compress and decompress, byte
for byte against the oracle."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("args", [["500"], ["100", "4"]])
def test_random_cases_equal_the_oracle(gpu, args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "soak_new_kernels.py"), *args],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " 0 mismatches" in r.stdout, r.stdout[-2000:]
