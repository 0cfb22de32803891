"""The opt-in truncated-mantissa coding of unpredictable values (north_star
(3); not part of the reference, version-2 containers).

Checked against the oracle's restatement of the extension
(oracle/ebz_oracle.c ora_compress_tr, oracle.tr_pack / tr_unpack): container
bytes, stored values and reconstruction identical, on every compress kernel
(2D / 3D fast, z-rows 3D, two-row 3D, generic d = 1 / 4 and float64);
the error bound holds; the block packer / unpacker on the device equals the
oracle's on values with zeros, subnormals and extreme exponents and across
4096-value chunk boundaries; a block whose size disagrees with its header
fields is rejected."""

import numpy as np
import pytest

import paper_1706_03791_b200 as ebz
from paper_1706_03791_b200 import _native as nat

pytestmark = pytest.mark.gpu


def _field(rng, dims, dtype):
    n = int(np.prod(dims))
    v = np.cumsum(rng.standard_normal(n)) * 0.1
    v[:: max(1, n // 97)] += 20 * rng.standard_normal(v[:: max(1, n // 97)].size)
    return v.astype(dtype)


CASES = [  # dims (fastest first), layers, dtype, rel
    ((67, 45), 1, np.float32, 1e-5),
    ((64, 40), 2, np.float32, 1e-4),
    ((40, 24, 16), 1, np.float32, 1e-5),   # z-rows kernel (nx % 4 == 0)
    ((33, 17, 11), 1, np.float32, 1e-4),   # two-row kernel
    ((21, 13, 9), 2, np.float32, 1e-5),
    ((500,), 1, np.float32, 1e-6),         # generic, d = 1
    ((9, 7, 5, 4), 1, np.float32, 1e-4),   # generic, d = 4
    ((30, 20, 10), 1, np.float64, 1e-9),   # generic, float64
]


@pytest.mark.parametrize("dims,layers,dtype,rel", CASES)
def test_truncated_coding_matches_oracle(gpu, oracle, dims, layers, dtype, rel):
    rng = np.random.default_rng(abs(hash((dims, layers, rel))) % 2**32)
    v = _field(rng, dims, dtype)
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=rel), layers=layers,
                               truncate_unpredictable=True)
    out = ebz.compress(ebz.DataGrid(dims, v), cfg)
    ref = oracle.compress_bytes(v, dims, layers=layers, relative=rel, truncate=True)
    assert out.stream.unpredictable_coding == 1
    assert out.stream.n_unpredictable == ref["K"] > 0
    blob = ebz.serialize(out.stream)
    assert blob == ref["container"]
    back = ebz.deserialize(blob)
    assert back == out.stream
    rec = ebz.decompress(back)
    assert rec.values.tobytes() == ref["recon"].tobytes()
    err = np.abs(rec.values.astype(np.float64) - v.astype(np.float64)).max()
    assert err <= out.stream.eb_effective
    # smaller than the reference's verbatim container
    plain = ebz.serialize(ebz.compress(ebz.DataGrid(dims, v), ebz.CompressorConfig(
        ebz.ErrorBoundSpec(relative=rel), layers=layers)).stream)
    assert len(blob) < len(plain)


@pytest.mark.parametrize("width", [32, 64])
@pytest.mark.parametrize("k", [0, 1, 4095, 4096, 4097, 100003])
def test_block_packer_matches_oracle(gpu, oracle, width, k):
    rng = np.random.default_rng(k + width)
    dt = np.float64 if width == 64 else np.float32
    v = (rng.standard_normal(k) * 10.0 ** rng.uniform(-30, 30, k)).astype(dt)
    if k > 10:
        fi = np.finfo(dt)
        v[:6] = [0.0, -0.0, fi.tiny / 4, -fi.tiny, fi.max, -fi.max]
    for eb in (1e-3, 3.7e-12, 2.0 ** -140):
        t = oracle.trunc_values(v, eb)
        block = nat.tr_pack(t, width, eb)
        assert block == oracle.tr_pack(t, eb)
        assert nat.tr_unpack(block, k, width, eb).tobytes() == t.tobytes()


def test_block_size_mismatch_rejected(gpu, oracle):
    v = np.linspace(-3, 7, 1000).astype(np.float32)
    block = oracle.tr_pack(oracle.trunc_values(v, 1e-4), 1e-4)
    for bad in (block[:-1], block + b"\0"):
        with pytest.raises(ebz.PayloadMismatchError):
            nat.tr_unpack(bad, v.size, 32, 1e-4)


def test_truncated_coding_round_trips_through_batched_calls(gpu):
    rng = np.random.default_rng(9)
    dims = (40, 24, 16)
    grids = [ebz.DataGrid(dims, _field(rng, dims, np.float32)) for _ in range(3)]
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-5), truncate_unpredictable=True)
    many = ebz.compress_many(grids, cfg)
    for g, o in zip(grids, many):
        assert ebz.serialize(o.stream) == ebz.serialize(ebz.compress(g, cfg).stream)
    recs = ebz.decompress_many([o.stream for o in many])
    for o, r in zip(many, recs):
        assert r.values.tobytes() == ebz.decompress(o.stream).values.tobytes()
    # --auto-m with the extension runs the loop (trials sweep the verbatim coding)
    out, used, trials = ebz.compress_auto_m(grids[0], cfg)
    assert out.stream.unpredictable_coding == 1 and trials[0] == 8
