"""The block-speculative 2D n = 1 sweeps (csrc/sweep2.cu) against the oracle
on the cases its structure adds: quotients that are exact half-integers (the
speculative block is replayed with the reference's division), bounds with no
usable reciprocal (every block replayed), ragged shapes around the 8-step
blocks, 32-row patches and 16-byte alignment, 16-bit codes, many patches in
flight, and the one-row kernel (EBZ_NO_SWEEP2) writing the same bytes."""

import ctypes
import hashlib
import os

import numpy as np
import pytest

import paper_1706_03791_b200 as ebz
from paper_1706_03791_b200 import _native as nat

pytestmark = pytest.mark.gpu


def _check(oracle, v, dims, m=8, layers=1, **bound):
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(**bound), interval_exponent=m, layers=layers)
    out = ebz.compress(ebz.DataGrid(dims, v), cfg)
    ref = oracle.compress_bytes(v, dims, layers=layers, m=m, **bound)
    blob = ebz.serialize(out.stream)
    assert blob == ref["container"], (dims, bound)
    back = ebz.decompress(ebz.deserialize(blob))
    assert hashlib.sha256(back.values.tobytes()).hexdigest() == ref["recon_digest"], (dims, bound)
    return blob


def _kernel(dims, layers=1):
    d = (ctypes.c_uint64 * len(dims))(*dims)
    return nat.load_library().ebz_sweep_kernel_choice(32, len(dims), d, layers, 1, 1)


@pytest.mark.parametrize("layers", [1, 2])
def test_half_integer_quotients_replay_the_block(gpu, oracle, layers):
    # integer data, eb = 1: (x - pred) / 2 is a half-integer at about half of
    # the points, so nearly every block takes the replay
    rng = np.random.default_rng(3)
    dims = (301, 77)
    assert _kernel(dims, layers) == 4
    v = rng.integers(-40, 40, int(np.prod(dims))).astype(np.float32)
    _check(oracle, v, dims, layers=layers, absolute=1.0)
    # a smooth field with isolated exact ties
    t = np.arange(int(np.prod(dims)), dtype=np.float64)
    w = np.round(np.sin(t / 50.0) * 100.0).astype(np.float32)
    _check(oracle, w, dims, layers=layers, absolute=0.5)


@pytest.mark.parametrize("layers", [1, 2])
@pytest.mark.parametrize("eb", [1e-310, 3e-302, 1e300])
def test_bounds_without_a_usable_reciprocal(gpu, oracle, eb, layers):
    rng = np.random.default_rng(4)
    dims = (130, 41)
    v = (rng.standard_normal(int(np.prod(dims))) * 1e-3).astype(np.float32)
    _check(oracle, v, dims, layers=layers, absolute=eb)


@pytest.mark.parametrize("layers", [1, 2])
@pytest.mark.parametrize("dims", [(1, 1), (1, 70), (70, 1), (2, 2), (4100, 2), (3, 66), (7, 3), (8, 32), (9, 33),
                                  (31, 31), (33, 34), (39, 64), (40, 65), (257, 95), (1023, 34), (500, 40), (252, 37),
                                  (64, 200)])
def test_ragged_shapes(gpu, oracle, dims, layers):
    rng = np.random.default_rng(sum(dims))
    n = int(np.prod(dims))
    t = np.linspace(0, 25, n)
    v = (np.sin(t) * 7 + 0.01 * rng.standard_normal(n)).astype(np.float32)
    v[rng.integers(0, n, max(1, n // 40))] += 30.0
    _check(oracle, v, dims, layers=layers, absolute=2e-3)


@pytest.mark.parametrize("layers", [1, 2])
def test_wide_codes_and_low_hit_rate(gpu, oracle, layers):
    rng = np.random.default_rng(6)
    dims = (520, 130)
    n = int(np.prod(dims))
    v = (np.cumsum(rng.standard_normal(n)) * 0.01).astype(np.float32)
    _check(oracle, v, dims, m=12, layers=layers, relative=1e-6)
    # mostly unpredictable: the decompress sweep lives on its verbatim cursor
    u = rng.standard_normal(n).astype(np.float32)
    _check(oracle, u, dims, m=4, layers=layers, relative=1e-5)
    # 16-bit codes on rows that start on 4-byte, not 16-byte, boundaries
    dims = (250, 60)
    w = (np.cumsum(rng.standard_normal(int(np.prod(dims)))) * 0.01).astype(np.float32)
    _check(oracle, w, dims, m=12, layers=layers, relative=1e-6)


@pytest.mark.parametrize("layers", [1, 2])
def test_one_row_kernel_writes_the_same_bytes(gpu, oracle, layers):
    rng = np.random.default_rng(8)
    dims = (777, 100)
    n = int(np.prod(dims))
    v = (np.sin(np.linspace(0, 90, n)) + 0.003 * rng.standard_normal(n)).astype(np.float32)
    a = _check(oracle, v, dims, layers=layers, relative=1e-4)
    os.environ["EBZ_NO_SWEEP2"] = "1"
    try:
        assert _kernel(dims, layers) == 1
        b = _check(oracle, v, dims, layers=layers, relative=1e-4)
    finally:
        del os.environ["EBZ_NO_SWEEP2"]
    assert a == b


@pytest.mark.parametrize("layers", [1, 2])
def test_many_fields_many_patches(gpu, oracle, layers):
    # 9 fields x 7 patch rows through compress_many / decompress_many
    rng = np.random.default_rng(9)
    dims = (150, 200)
    n = int(np.prod(dims))
    grids = []
    for i in range(9):
        v = (np.sin(np.linspace(0, 10 + 7 * i, n)) * (i + 1) + 0.01 * rng.standard_normal(n))
        grids.append(ebz.DataGrid(dims, v.astype(np.float32)))
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-4), layers=layers)
    outs = ebz.compress_many(grids, cfg)
    backs = ebz.decompress_many([o.stream for o in outs])
    for g, o, bk in zip(grids, outs, backs):
        ref = oracle.compress_bytes(g.values, dims, layers=layers, m=8, relative=1e-4)
        assert ebz.serialize(o.stream) == ref["container"]
        assert hashlib.sha256(bk.values.tobytes()).hexdigest() == ref["recon_digest"]


def test_more_fields_than_one_launch_holds(gpu, oracle):
    # 70 fields > kBatchMax (64): two sweep launches over the same ticket / face buffers
    import torch
    from paper_1706_03791_b200.device import DeviceBatch
    rng = np.random.default_rng(12)
    dims = (90, 70)
    n = int(np.prod(dims))
    fields = [(np.sin(np.linspace(0, 5 + i, n)) * (1 + i % 5) +
               0.02 * rng.standard_normal(n)).astype(np.float32) for i in range(70)]
    dev = torch.device("cuda", 0)
    db = DeviceBatch()
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-3))
    d_in = [torch.from_numpy(f).to(dev) for f in fields]
    outs = [torch.empty_like(x) for x in d_in]
    with db.ctx.lock:
        db.compress_batch(d_in, dims, cfg)
        db.decompress_batch(outs)
    torch.cuda.synchronize()
    for i, f in enumerate(fields):
        ref = oracle.compress_bytes(f, dims, layers=1, m=8, relative=1e-3)
        assert db.info(i).status == 0
        assert db.container(i) == ref["container"], i
        assert outs[i].cpu().numpy().tobytes() == oracle.decompress_bytes(ref["container"]).tobytes(), i


# ---- binary64 elements: 16-byte face words {value, epoch}, no float32 cast
def _check64(oracle, v, dims, m=8, layers=1, **bound):
    d = (ctypes.c_uint64 * len(dims))(*dims)
    assert nat.load_library().ebz_sweep_kernel_choice(64, len(dims), d, layers, 1, 1) == 4
    assert v.dtype == np.float64
    return _check(oracle, v, dims, m=m, layers=layers, **bound)


@pytest.mark.parametrize("layers", [1, 2])
@pytest.mark.parametrize("dims", [(1, 1), (1, 70), (70, 1), (2, 2), (3, 66), (7, 3), (8, 32), (9, 33),
                                  (33, 34), (39, 64), (257, 95), (1023, 34), (500, 40), (64, 200)])
def test_f64_ragged_shapes(gpu, oracle, dims, layers):
    rng = np.random.default_rng(sum(dims) + 7)
    n = int(np.prod(dims))
    t = np.linspace(0, 25, n)
    v = np.sin(t) * 7 + 0.01 * rng.standard_normal(n)
    v[rng.integers(0, n, max(1, n // 40))] += 30.0
    _check64(oracle, v.astype(np.float64), dims, layers=layers, absolute=2e-3)


@pytest.mark.parametrize("layers", [1, 2])
def test_f64_replay_wide_codes_low_hit_rate(gpu, oracle, layers):
    rng = np.random.default_rng(21)
    dims = (301, 77)
    n = int(np.prod(dims))
    v = rng.integers(-40, 40, n).astype(np.float64)
    _check64(oracle, v, dims, layers=layers, absolute=1.0)           # half-integer quotients
    w = np.cumsum(rng.standard_normal(n)) * 0.01
    _check64(oracle, w, dims, m=12, layers=layers, relative=1e-7)     # 16-bit codes
    u = rng.standard_normal(n)
    _check64(oracle, u, dims, m=4, layers=layers, relative=1e-5)      # mostly verbatim
    _check64(oracle, u * 1e-3, dims, layers=layers, absolute=1e-310)  # no usable reciprocal


@pytest.mark.parametrize("layers", [1, 2])
def test_f64_many_fields_many_patches(gpu, oracle, layers):
    rng = np.random.default_rng(22)
    dims = (150, 200)
    n = int(np.prod(dims))
    grids = []
    for i in range(9):
        v = np.sin(np.linspace(0, 10 + 7 * i, n)) * (i + 1) + 0.01 * rng.standard_normal(n)
        grids.append(ebz.DataGrid(dims, v.astype(np.float64)))
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-6), layers=layers)
    outs = ebz.compress_many(grids, cfg)
    backs = ebz.decompress_many([o.stream for o in outs])
    for g, o, bk in zip(grids, outs, backs):
        ref = oracle.compress_bytes(g.values, dims, layers=layers, m=8, relative=1e-6)
        assert ebz.serialize(o.stream) == ref["container"]
        assert hashlib.sha256(bk.values.tobytes()).hexdigest() == ref["recon_digest"]
