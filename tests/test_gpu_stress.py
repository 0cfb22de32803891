"""Schedule-perturbation stress of the wavefront kernels' tagged-face
protocol (the reference is strictly sequential; the B200 sweeps
replace that order with epoch-tagged patch faces and ticket order).

A child process runs with EBZ_SCHED_JITTER set: warps of the wavefront
kernels sleep a hash-chosen 0..jitter ns -- at one chunk in four in the
z-rows kernels, at one block in four in the block-speculative 2D kernels, at
one task start in four in the one-row / two-row kernels (where a per-chunk
test costs the latency-bound single fields ~5%) -- so
producers and consumers meet in orders the normal schedule never produces
(consumers arriving long before their faces, producers racing ahead).
Batched compress and decompress over every fast kernel (z-rows 3D, two-row
3D, one-row 3D, block-speculative 2D, n = 2, the binary64 kernels) must still produce the oracle's containers and
reconstructions byte for byte."""

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
rng = np.random.default_rng(11)
cases = [((64, 48, 40), 1, 8), ((33, 40, 21), 1, 6), ((200, 150), 1, 6), ((120, 90), 2, 4),
         ((333, 260), 1, 3), ((90, 300), 2, 3),
         # binary64: 16-byte face words (sweep2 / sweep3b)
         ((64, 48, 40), 1, 4, np.float64), ((200, 150), 1, 3, np.float64),
         ((120, 90), 2, 3, np.float64),
         ((36, 28, 20), 2, 4), ((64, 48, 40), 1, 3)]
for case in cases:
    dims, layers, nf = case[:3]
    dt = case[3] if len(case) > 3 else np.float32
    n = int(np.prod(dims))
    fields = []
    for f in range(nf):
        v = np.cumsum(rng.standard_normal(n)).astype(dt) * dt(0.05)
        v[:: 37 + f] += (3 * rng.standard_normal(v[:: 37 + f].size)).astype(dt)
        fields.append(v)
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-5), layers=layers)
    many = ebz.compress_many([ebz.DataGrid(dims, v) for v in fields], cfg, group=max(2, nf // 2))
    recs = ebz.decompress_many([o.stream for o in many])
    for v, o, r in zip(fields, many, recs):
        ref = O.compress_bytes(v, dims, layers=layers, relative=1e-5)
        assert ebz.serialize(o.stream) == ref["container"], (dims, layers)
        assert hashlib.sha256(r.values.tobytes()).hexdigest() == ref["recon_digest"], (dims, layers)
print("stress ok")
"""


@pytest.mark.parametrize("jitter", ["400", "5000"])
def test_wavefronts_bit_exact_under_schedule_perturbation(gpu, jitter):
    env = dict(os.environ, EBZ_SCHED_JITTER=jitter)
    r = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT))], env=env,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "stress ok" in r.stdout
