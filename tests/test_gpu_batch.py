"""Batched device pipelines (ebz_compress_batch / ebz_decompress_batch): every
field's container and reconstruction must equal the oracle's for that field
alone -- batching is a scheduling change, never a numerical one."""

import numpy as np
import pytest

import paper_1706_03791_b200 as ebz
from paper_1706_03791_b200 import _native as nat
from paper_1706_03791_b200.device import DeviceBatch

pytestmark = pytest.mark.gpu


def _fields(rng, dims, count, dtype, constant=()):
    n = int(np.prod(dims))
    out = []
    for i in range(count):
        if i in constant:
            out.append(np.full(n, 3.25, dtype))
            continue
        amp = 10 ** rng.uniform(-2, 3)
        t = np.linspace(0, rng.uniform(2, 30), n)
        v = amp * (np.sin(t) + 0.3 * np.cos(3.1 * t)) + amp * 0.05 * rng.standard_normal(n)
        out.append(v.astype(dtype))
    return out


def _run_batch(dims, fields, layers, m, bound, oracle):
    import torch
    dev = torch.device("cuda", 0)
    db = DeviceBatch()
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(**bound), layers=layers, interval_exponent=m)
    d_in = [torch.from_numpy(f).to(dev) for f in fields]
    outs = [torch.empty_like(x) for x in d_in]
    with db.ctx.lock:
        db.compress_batch(d_in, dims, cfg)
        db.decompress_batch(outs)
    torch.cuda.synchronize()
    nf = len(fields)
    for i, f in enumerate(fields):
        try:
            ref = oracle.compress_bytes(f, dims, layers=layers, m=m, **bound)
        except ValueError:
            assert db.info(i).status & nat.ST_EB_NONPOSITIVE, i
            continue
        h = db.info(i)
        assert h.status == 0, (i, hex(h.status))
        assert db.container(i) == ref["container"], (dims, i)
        rec = outs[i].cpu().numpy()
        want = oracle.decompress_bytes(ref["container"])
        assert rec.tobytes() == want.tobytes(), (dims, i)
        hd = db.decode_info(nf + i)
        assert hd.status == 0 and hd.used == h.n_unpred, (i, hex(hd.status))


def test_batch_3d_many_fields_chunked(gpu, oracle):
    # 70 fields > kBatchMax (64): two sweep launches; per-field relative
    # bounds give every field its own eb
    rng = np.random.default_rng(7)
    dims = (37, 21, 13)
    _run_batch(dims, _fields(rng, dims, 70, np.float32), 1, 8, dict(relative=1e-3), oracle)


def test_batch_2d_two_layers_wide_codes(gpu, oracle):
    rng = np.random.default_rng(8)
    dims = (300, 45)
    _run_batch(dims, _fields(rng, dims, 5, np.float32), 2, 10, dict(absolute=1e-3), oracle)


def test_batch_3d_two_layers_with_constant_field(gpu, oracle):
    rng = np.random.default_rng(9)
    dims = (20, 17, 9)
    _run_batch(dims, _fields(rng, dims, 6, np.float32, constant=(2,)), 2, 6,
               dict(relative=1e-4), oracle)


def test_batch_generic_path_f64_and_4d(gpu, oracle):
    rng = np.random.default_rng(10)
    dims = (14, 9, 6)
    _run_batch(dims, _fields(rng, dims, 3, np.float64), 1, 8, dict(absolute=1e-4), oracle)
    dims4 = (6, 5, 4, 3)
    _run_batch(dims4, _fields(rng, dims4, 3, np.float32), 1, 8, dict(relative=1e-3), oracle)


def test_compress_many_matches_single_calls(gpu, oracle):
    # host-to-host batched API: identical outcomes to the one-field calls,
    # several pipeline groups, and the sequential loop's first error
    rng = np.random.default_rng(11)
    dims = (33, 20, 11)
    fields = _fields(rng, dims, 37, np.float32)
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-3), layers=1)
    grids = [ebz.DataGrid(dims, f) for f in fields]
    many = ebz.compress_many(grids, cfg, group=8)
    for g, o in zip(grids, many):
        one = ebz.compress(g, cfg)
        assert ebz.serialize(o.stream) == ebz.serialize(one.stream)
        assert o.hitting_rate == one.hitting_rate and o.warning == one.warning
    recs = ebz.decompress_many([o.stream for o in many], group=8)
    for o, r in zip(many, recs):
        assert r.values.tobytes() == ebz.decompress(o.stream).values.tobytes()
        assert r.dims == o.stream.dims
    # a ring of two groups of three (group g reuses group g - 2's slots and
    # buffers), after the workspaces were given back
    from paper_1706_03791_b200 import _native as nat
    nat.context().trim()
    small = ebz.compress_many(grids[:11], cfg, group=3)
    assert [ebz.serialize(o.stream) for o in small] == \
        [ebz.serialize(o.stream) for o in many[:11]]
    for r, o in zip(ebz.decompress_many([o.stream for o in small], group=3), recs):
        assert r.values.tobytes() == o.values.tobytes()
    # streams that went through bytes (deserialize) decompress the same way
    blobs = [ebz.deserialize(ebz.serialize(o.stream)) for o in many[:5]]
    for r, b in zip(ebz.decompress_many(blobs), blobs):
        assert r.values.tobytes() == ebz.decompress(b).values.tobytes()
    # mixed geometry falls back to the single calls
    mixed = [grids[0], ebz.DataGrid((11, 20, 33), fields[1])]
    assert [ebz.serialize(o.stream) for o in ebz.compress_many(mixed, cfg)] == \
        [ebz.serialize(ebz.compress(g, cfg).stream) for g in mixed]
    # a constant field under a relative bound fails like the loop would
    bad = grids[:3] + [ebz.DataGrid(dims, np.full(fields[0].size, 2.0, np.float32))]
    with pytest.raises(ValueError, match="effective error bound must be positive"):
        ebz.compress_many(bad, cfg, group=2)
