"""The binary64 3D n = 1 patch wavefront (csrc/sweep3b.cu: 16-byte face words
{value, epoch}, blocks of 4 steps, speculative reciprocal quantizer) against
the oracle: ragged shapes around the 8 x 4 row patches, exact half-integer
quotients (block replay), bounds without a usable reciprocal, 16-bit codes,
mostly-verbatim fields, batches; and the generic kernel (EBZ_NO_SWEEP3B)
writing the same bytes."""

import ctypes
import hashlib
import os

import numpy as np
import pytest

import paper_1706_03791_b200 as ebz
from paper_1706_03791_b200 import _native as nat

pytestmark = pytest.mark.gpu


def _kernel(dims):
    d = (ctypes.c_uint64 * 3)(*dims)
    return nat.load_library().ebz_sweep_kernel_choice(64, 3, d, 1, 1, 1)


def _check(oracle, v, dims, m=8, **bound):
    assert v.dtype == np.float64 and _kernel(dims) == 5
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(**bound), interval_exponent=m)
    out = ebz.compress(ebz.DataGrid(dims, v), cfg)
    ref = oracle.compress_bytes(v, dims, layers=1, m=m, **bound)
    blob = ebz.serialize(out.stream)
    assert blob == ref["container"], (dims, bound)
    back = ebz.decompress(ebz.deserialize(blob))
    assert hashlib.sha256(back.values.tobytes()).hexdigest() == ref["recon_digest"], (dims, bound)
    return blob


@pytest.mark.parametrize("dims", [(1, 1, 1), (5, 3, 2), (8, 8, 4), (9, 9, 5), (16, 7, 9),
                                  (33, 17, 6), (40, 40, 13), (64, 37, 21), (130, 9, 4),
                                  (7, 64, 3), (12, 5, 70), (257, 16, 8), (3, 2, 33)])
def test_ragged_shapes(gpu, oracle, dims):
    rng = np.random.default_rng(sum(dims))
    n = int(np.prod(dims))
    t = np.linspace(0, 25, n)
    v = np.sin(t) * 7 + 0.01 * rng.standard_normal(n)
    v[rng.integers(0, n, max(1, n // 40))] += 30.0
    _check(oracle, v.astype(np.float64), dims, absolute=2e-3)


def test_replay_wide_codes_low_hit_rate(gpu, oracle):
    rng = np.random.default_rng(3)
    dims = (70, 23, 11)
    n = int(np.prod(dims))
    _check(oracle, rng.integers(-40, 40, n).astype(np.float64), dims, absolute=1.0)
    w = np.cumsum(rng.standard_normal(n)) * 0.01
    _check(oracle, w, dims, m=12, relative=1e-7)
    u = rng.standard_normal(n)
    _check(oracle, u, dims, m=4, relative=1e-5)
    _check(oracle, u * 1e-3, dims, absolute=1e-310)
    _check(oracle, u * 1e-3, dims, absolute=1e300)


def test_many_fields_and_generic_kernel_equivalence(gpu, oracle):
    rng = np.random.default_rng(9)
    dims = (72, 50, 30)
    n = int(np.prod(dims))
    grids = []
    for i in range(7):
        v = np.sin(np.linspace(0, 10 + 7 * i, n)) * (i + 1) + 0.01 * rng.standard_normal(n)
        grids.append(ebz.DataGrid(dims, v.astype(np.float64)))
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-6))
    outs = ebz.compress_many(grids, cfg)
    backs = ebz.decompress_many([o.stream for o in outs])
    blobs = []
    for g, o, bk in zip(grids, outs, backs):
        ref = oracle.compress_bytes(g.values, dims, layers=1, m=8, relative=1e-6)
        blobs.append(ebz.serialize(o.stream))
        assert blobs[-1] == ref["container"]
        assert hashlib.sha256(bk.values.tobytes()).hexdigest() == ref["recon_digest"]
    os.environ["EBZ_NO_SWEEP3B"] = "1"
    try:
        assert _kernel(dims) == 0
        out = ebz.compress(grids[0], cfg)
        assert ebz.serialize(out.stream) == blobs[0]
    finally:
        del os.environ["EBZ_NO_SWEEP3B"]


@pytest.mark.parametrize("mode", ["c", "cd"])
def test_float32_fields_through_the_same_kernel(gpu, oracle, mode):
    # float32 elements (compress is picked by the time model for lone fields;
    # EBZ_SWEEP3B32 forces either direction here)
    old = os.environ.get("EBZ_SWEEP3B32")
    os.environ["EBZ_SWEEP3B32"] = mode
    try:
        rng = np.random.default_rng(31)
        for dims, m in (((64, 37, 21), 8), ((9, 9, 5), 8), ((132, 33, 6), 12), ((250, 20, 9), 8)):
            d = (ctypes.c_uint64 * 3)(*dims)
            assert nat.load_library().ebz_sweep_kernel_choice(32, 3, d, 1, 1, 1) == 5
            n = int(np.prod(dims))
            v = (np.sin(np.linspace(0, 30, n)) * 5 + 0.02 * rng.standard_normal(n)).astype(np.float32)
            v[rng.integers(0, n, n // 50)] += 40.0
            cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-4), interval_exponent=m)
            out = ebz.compress(ebz.DataGrid(dims, v), cfg)
            ref = oracle.compress_bytes(v, dims, layers=1, m=m, relative=1e-4)
            blob = ebz.serialize(out.stream)
            assert blob == ref["container"], (mode, dims)
            back = ebz.decompress(ebz.deserialize(blob))
            assert hashlib.sha256(back.values.tobytes()).hexdigest() == ref["recon_digest"]
    finally:
        if old is None:
            del os.environ["EBZ_SWEEP3B32"]
        else:
            os.environ["EBZ_SWEEP3B32"] = old
