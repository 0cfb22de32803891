"""The opt-in sweep3 decompress kernel (EBZ_SWEEP3D=1, sweep3.cu) against
the oracle: 3D, n = 1 round trips with u8 and u16 codes, verbatim-heavy
fields and ragged patch edges.  The switch is read once per process, so the
check runs in a child interpreter with the variable set."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, ROOT)
import paper_1706_03791_b200 as ebz
from oracle import oracle as O
rng = np.random.default_rng(5)
for dims, m, rel, noise in [((40, 24, 16), 8, 1e-4, 0.01), ((64, 70, 9), 8, 1e-6, 1.0),
                            ((36, 33, 13), 12, 1e-5, 0.3), ((8, 5, 3), 8, 1e-3, 0.0)]:
    n = int(np.prod(dims))
    v = np.cumsum(rng.standard_normal(n)).astype(np.float32) * 0.1
    v += (noise * rng.standard_normal(n)).astype(np.float32)
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=rel), layers=1, interval_exponent=m)
    out = ebz.compress(ebz.DataGrid(dims, v), cfg)
    ref = O.compress_bytes(v, dims, layers=1, m=m, relative=rel)
    blob = ebz.serialize(out.stream)
    assert blob == ref["container"], dims
    back = ebz.decompress(ebz.deserialize(blob))
    assert hashlib.sha256(back.values.tobytes()).hexdigest() == ref["recon_digest"], dims
    many = ebz.decompress_many([out.stream] * 3)
    assert all(r.values.tobytes() == back.values.tobytes() for r in many)
print("sweep3d ok")
"""


def test_sweep3d_round_trips_match_oracle(gpu):
    env = dict(os.environ, EBZ_SWEEP3D="1")
    r = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT))], env=env,
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "sweep3d ok" in r.stdout
