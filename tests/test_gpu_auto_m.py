"""Batched interval trials (compress_auto_m over ebz_compress_trials) against
the reference's --auto-m loop (cli.py:146-154): one full compression per
trial (``_compress_auto_m_loop``) and the CPU oracle's loop.  Same trials,
same final exponent, byte-identical container, same hitting rate and
warning -- on every sweep kernel (2D / 3D fast, the z-rows 3D kernel, the
two-row 3D n = 2 kernel, the generic one), for odd and even m0, with the
speculative single batch and with the m0-first split."""

import numpy as np
import pytest

import paper_1706_03791_b200 as ebz
from paper_1706_03791_b200 import codec

pytestmark = pytest.mark.gpu


def _field(rng, dims, dtype, rough):
    n = int(np.prod(dims))
    v = np.cumsum(rng.standard_normal(n)) * 0.05
    v = v + rough * rng.standard_normal(n)
    return v.astype(dtype)


CASES = [  # dims (fastest first), layers, dtype, m0, rel, theta, roughness
    ((300, 180), 1, np.float32, 8, 1e-5, 0.9, 0.3),
    ((300, 180), 2, np.float32, 7, 1e-5, 0.95, 0.3),
    ((64, 40, 24), 1, np.float32, 8, 1e-5, 0.9, 0.5),
    ((66, 40, 24), 1, np.float32, 4, 1e-4, 0.99, 0.05),
    ((40, 30, 20), 2, np.float32, 8, 1e-6, 0.9, 0.2),
    ((30, 20, 10), 1, np.float64, 6, 1e-6, 0.9, 0.2),
    ((500,), 1, np.float32, 8, 1e-5, 0.9, 1.0),
    ((64, 40), 1, np.float32, 16, 1e-6, 0.9, 1.0),
    ((64, 40), 1, np.float32, 8, 1e-2, 0.5, 0.0),   # m0 already hits: one trial
]


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("dims,layers,dtype,m0,rel,theta,rough", CASES)
def test_trials_match_the_loop(gpu, oracle, monkeypatch, split, dims, layers, dtype, m0, rel,
                               theta, rough):
    if split:
        monkeypatch.setattr(codec, "AUTO_M_SPECULATE_POINTS", 0)
    rng = np.random.default_rng(abs(hash((dims, layers, m0))) % 2**32)
    v = _field(rng, dims, dtype, rough)
    grid = ebz.DataGrid(dims, v)
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=rel), layers=layers,
                               interval_exponent=m0, hitting_rate_threshold=theta)
    out, used, trials = ebz.compress_auto_m(grid, cfg)
    ref, ref_used, ref_trials = codec._compress_auto_m_loop(grid, cfg)
    assert trials == ref_trials
    assert used == ref_used
    assert ebz.serialize(out.stream) == ebz.serialize(ref.stream)
    assert out.hitting_rate == ref.hitting_rate and out.warning == ref.warning
    if v.size <= 60000:
        o = oracle.auto_m(v, dims, layers=layers, m=m0, relative=rel, theta=theta)
        assert trials == o["trials"]
        assert ebz.serialize(out.stream) == o["container"]


def test_trials_errors_like_the_loop(gpu):
    # a constant field under a relative bound: the loop's first compress raises
    grid = ebz.DataGrid((40, 30), np.full(1200, 3.0, np.float32))
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-3))
    with pytest.raises(ValueError, match="effective error bound must be positive"):
        ebz.compress_auto_m(grid, cfg)
