"""Parity of the CUDA path with the reference (golden fixtures produced by the
reference itself) and with the pinned CPU oracle.  Bit-exact: container
bytes, codes, unpredictable set, reconstruction bytes, error classes."""

import hashlib

import numpy as np
import pytest

import paper_1706_03791_b200 as ebz
from paper_1706_03791_b200 import entropy

pytestmark = pytest.mark.gpu


def _config(c, m=None):
    return ebz.CompressorConfig(
        bound=ebz.ErrorBoundSpec(absolute=c["absolute"], relative=c["relative"]),
        layers=c["layers"], interval_exponent=m or c["m"],
        hitting_rate_threshold=c["theta"])


def test_golden_containers_bit_exact(golden, gpu):
    meta, z = golden
    for c in meta:
        grid = ebz.DataGrid(tuple(c["dims"]), z[c["name"] + "__values"])
        if "error" in c:
            with pytest.raises(ValueError):
                ebz.compress(grid, _config(c))
            continue
        if c.get("auto_m"):
            out, cfg, trials = ebz.compress_auto_m(grid, _config(c))
            assert trials == c["trials"], c["name"]
        else:
            out = ebz.compress(grid, _config(c))
        ref = z[c["name"] + "__container"].tobytes()
        got = ebz.serialize(out.stream)
        assert got == ref, c["name"]
        assert out.hitting_rate == c["hitting_rate"], c["name"]
        sugg = out.warning.suggested_exponent if out.warning else None
        assert sugg == c["suggested"], c["name"]
        assert out.recon_digest == c["recon_digest"], c["name"]
        back = ebz.decompress(ebz.deserialize(ref))
        assert ebz.grid_digest(back) == c["recon_digest"], c["name"]
        assert back.values.dtype == grid.values.dtype


def test_entropy_known_answers(gpu):
    assert entropy.build_code([2, 1, 1]).lengths.tolist() == [1, 2, 2]
    assert entropy.build_code([2, 1, 1]).code_words.tolist() == [0, 0b10, 0b11]
    assert entropy.build_code({0: 2, 1: 1, 2: 1}).lengths.tolist() == [1, 2, 2]
    assert entropy.build_code([0, 5, 0]).lengths.tolist() == [0, 1, 0]
    assert entropy.build_code([1, 1, 1, 1]).lengths.tolist() == [2, 2, 2, 2]
    assert entropy.build_code([2, 2, 2, 2, 2]).lengths.tolist() == [3, 3, 2, 2, 2]
    t = entropy.build_code([2, 1, 1])
    assert entropy.encode([0, 0, 1], t) == (b"\x20", 4)
    t1 = entropy.build_code([0, 7])
    assert entropy.encode([1] * 7, t1) == (b"\x00", 7)
    assert entropy.decode(b"\x00", t1, 7).tolist() == [1] * 7
    with pytest.raises(ValueError, match="exhausted"):
        data, _ = entropy.encode([0, 1, 2], t)
        entropy.decode(data, t, 50)
    with pytest.raises(ValueError, match="invalid"):
        entropy.decode(b"\xff", entropy.build_code([0, 9]), 2)
    for bad in ([], [0, 0], [-1, 2]):
        with pytest.raises(ValueError):
            entropy.build_code(bad)


def test_huffman_matches_heap_reference(gpu, oracle):
    rng = np.random.default_rng(11)
    for trial in range(120):
        n = int(rng.integers(2, 2000))
        kind = trial % 4
        if kind == 0:
            h = rng.integers(0, 5, n)            # heavy ties
        elif kind == 1:
            h = (rng.zipf(1.5, n) * 3).astype(np.int64)
        elif kind == 2:
            h = np.where(rng.random(n) < 0.9, 0, rng.integers(1, 1000, n))
        else:
            h = np.round(1e6 * np.exp(-np.abs(np.arange(n) - n / 2) / 3)).astype(np.int64)
        if not h.any():
            h[0] = 1
        assert entropy.build_code(h).lengths.tolist() == oracle.build_code(h).tolist()


def test_large_alphabet_roundtrip(gpu):
    rng = np.random.default_rng(2)
    sym = rng.zipf(1.3, 30_000).clip(max=65535) - 1
    t = entropy.build_code(np.bincount(sym, minlength=65535))
    data, nbits = entropy.encode(sym, t)
    assert entropy.decode(data, t, sym.size).tolist() == sym.tolist()


def test_long_code_chunks_match_oracle(gpu, oracle):
    # chunks averaging > 16 bits per code take the encoder's global-memory
    # path; codes up to the maximum depth exercise multi-word codewords
    rng = np.random.default_rng(5)
    h = np.ones(65536, np.int64)
    h[0] = 10**9
    h[1:40] = 2 ** np.arange(1, 40)          # a deep (Fibonacci-like) tail
    t = entropy.build_code(h)
    assert int(t.lengths.max()) > 32
    sym = np.concatenate([rng.integers(1, 65536, 9000), np.zeros(5000, np.int64),
                          rng.integers(1, 40, 3000), rng.integers(1, 65536, 7000)])
    data, nbits = entropy.encode(sym, t)
    ref_data, ref_bits = oracle.encode(sym, t.lengths)
    assert nbits == ref_bits and data == ref_data
    assert entropy.decode(data, t, sym.size).tolist() == sym.tolist()


def _random_case(rng):
    nd = int(rng.integers(1, 5))
    hi = {1: 3000, 2: 60, 3: 18, 4: 8}[nd]
    dims = tuple(int(rng.integers(1, hi)) for _ in range(nd))
    n = int(np.prod(dims))
    width = 32 if rng.random() < 0.6 else 64
    smooth = np.sin(np.linspace(0, rng.uniform(1, 20), n)) * rng.uniform(0.1, 100)
    v = smooth + rng.uniform(0, 2) * rng.standard_normal(n)
    if rng.random() < 0.2:
        idx = rng.choice(n, max(1, n // 30), replace=False)
        v[idx] += rng.laplace(0, 50, idx.size)
    v = v.astype(np.float32 if width == 32 else np.float64)
    layers = int(rng.integers(1, {1: 5, 2: 5, 3: 4, 4: 3}[nd]))  # 3D n = 3: 63-term stencils
    m = int(rng.choice([2, 3, 4, 6, 8, 10, 12, 16]))
    if rng.random() < 0.5:
        bound = dict(absolute=float(10 ** rng.uniform(-4, 0)), relative=None)
    else:
        bound = dict(absolute=None, relative=float(10 ** rng.uniform(-6, -1)))
    return dims, v, layers, m, bound


def test_random_configs_match_oracle(gpu, oracle):
    rng = np.random.default_rng(1234)
    for _ in range(150):
        dims, v, layers, m, bound = _random_case(rng)
        try:
            ref = oracle.compress_bytes(v, dims, layers=layers, m=m, **bound)
        except ValueError:
            with pytest.raises(ValueError):
                ebz.compress(ebz.DataGrid(dims, v), ebz.CompressorConfig(
                    ebz.ErrorBoundSpec(**bound), layers=layers, interval_exponent=m))
            continue
        out = ebz.compress(ebz.DataGrid(dims, v), ebz.CompressorConfig(
            ebz.ErrorBoundSpec(**bound), layers=layers, interval_exponent=m))
        assert ebz.serialize(out.stream) == ref["container"], (dims, layers, m, bound)
        rec = ebz.decompress(out.stream)
        assert hashlib.sha256(rec.values.tobytes()).hexdigest() == ref["recon_digest"]


def test_malformed_streams(gpu):
    rng = np.random.default_rng(8)
    grid = ebz.DataGrid((40,), rng.standard_normal(40) * 100)
    s = ebz.compress(grid, ebz.CompressorConfig(ebz.ErrorBoundSpec(absolute=1e-6))).stream
    assert s.n_unpredictable > 0
    tampered = ebz.CompressedStream(
        element_width=s.element_width, dims=s.dims, layers=s.layers,
        interval_exponent=s.interval_exponent, eb_effective=s.eb_effective,
        code_lengths=s.code_lengths, code_bit_length=s.code_bit_length,
        code_bits=s.code_bits, unpredictable_values=s.unpredictable_values[:-1])
    with pytest.raises(ValueError, match="unpredictable"):
        ebz.decompress(tampered)
    v = np.sin(np.linspace(0, 6, 512)) * 3 + 0.1 * rng.standard_normal(512)
    s = ebz.compress(ebz.DataGrid((64, 8), v),
                     ebz.CompressorConfig(ebz.ErrorBoundSpec(absolute=0.01))).stream
    cut = max(8, s.code_bit_length // 4)
    tampered = ebz.CompressedStream(
        element_width=s.element_width, dims=s.dims, layers=s.layers,
        interval_exponent=s.interval_exponent, eb_effective=s.eb_effective,
        code_lengths=s.code_lengths, code_bit_length=cut, code_bits=s.code_bits[:(cut + 7) // 8],
        unpredictable_values=s.unpredictable_values)
    with pytest.raises(ValueError):
        ebz.decompress(tampered)


def test_constant_and_edge_grids(gpu):
    g = ebz.DataGrid((50, 20), np.full(1000, 4.5))
    out = ebz.compress(g, ebz.CompressorConfig(ebz.ErrorBoundSpec(absolute=1e-8)))
    assert out.stream.n_unpredictable <= 1
    assert ebz.decompress(out.stream) == g
    g = ebz.DataGrid((100,), np.full(100, 0.001))
    out = ebz.compress(g, ebz.CompressorConfig(ebz.ErrorBoundSpec(absolute=0.01)))
    assert out.stream.n_unpredictable == 0 and out.hitting_rate == 1.0
    with pytest.raises(ValueError):
        ebz.compress(ebz.DataGrid((30,), np.full(30, 2.0)),
                     ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=0.01)))
    # single point, tiny and huge magnitudes, negative zero
    for vals in ([0.0], [-0.0, 0.0, -0.0, 1e-30], [3e38, -3e38, 1.0], [1e-40, 2e-40, 0.0]):
        v = np.array(vals, np.float32)
        g = ebz.DataGrid((len(vals),), v)
        out = ebz.compress(g, ebz.CompressorConfig(ebz.ErrorBoundSpec(absolute=1e-3)))
        back = ebz.decompress(out.stream)
        assert np.all(np.abs(back.values.astype(np.float64) - v.astype(np.float64)) <= 1e-3)


def test_idempotent_recompression(gpu):
    """Criterion C09 (reference tests/test_acceptance.py:285-310)."""
    rng = np.random.default_rng(99)
    for trial in range(30):
        nd = int(rng.integers(1, 4))
        dims = tuple(int(rng.integers(4, 30)) for _ in range(nd))
        n = int(np.prod(dims))
        v = np.cumsum(rng.standard_normal(n)).astype(np.float32 if trial % 2 else np.float64)
        cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(absolute=1e-3 * float(np.ptp(v) or 1)),
                                   layers=1 + trial % 3, interval_exponent=(4, 8, 12)[trial % 3])
        first = ebz.serialize(ebz.compress(ebz.DataGrid(dims, v), cfg).stream)
        again = ebz.serialize(ebz.compress(ebz.decompress(ebz.deserialize(first)), cfg).stream)
        assert first == again


def test_fast_sweeps_multi_patch(gpu, oracle):
    """Every fast-sweep variant (2D / 3D, n = 1 / 2, u8 / u16 codes) over grids
    spanning several patches in each direction with ragged edges (axis 0 not a
    multiple of 4 / 8 / 16 included), so patch faces, pads and the unaligned
    staging paths all carry real data; values mix smooth regions, noise,
    spikes, exact and negative zeros and float32 subnormals."""
    rng = np.random.default_rng(77)
    shapes = [(45, 37, 29), (64, 24, 17), (13, 70, 9), (257, 9, 11), (3, 40, 40),
              (100, 8, 8), (33, 17, 65), (300, 70), (37, 129), (16, 200)]
    for dims in shapes:
        n = int(np.prod(dims))
        t = np.linspace(0, 1, n)
        v = np.sin(40 * t) * 10 + 0.05 * rng.standard_normal(n)
        v[rng.choice(n, n // 50, replace=False)] += rng.laplace(0, 30, n // 50)
        v[n // 3:n // 3 + n // 10] = 0.0
        v[n // 2:n // 2 + 40] = -0.0
        v[2 * n // 3:2 * n // 3 + 30] = 1e-40
        v = v.astype(np.float32)
        for layers in (1, 2):
            for m in (8, 12):
                bound = dict(absolute=None, relative=1e-4)
                ref = oracle.compress_bytes(v, dims, layers=layers, m=m, **bound)
                out = ebz.compress(ebz.DataGrid(dims, v), ebz.CompressorConfig(
                    ebz.ErrorBoundSpec(**bound), layers=layers, interval_exponent=m))
                assert ebz.serialize(out.stream) == ref["container"], (dims, layers, m)
                rec = ebz.decompress(out.stream)
                assert hashlib.sha256(rec.values.tobytes()).hexdigest() == ref["recon_digest"], \
                    (dims, layers, m)


def test_seam_scans_unaligned_verbatim(gpu, oracle):
    """The C-ABI seams ebz_compress_scan / ebz_decompress_scan
    (_kernels.py:48-105) on a 3D layer-1 grid against the oracle's scans,
    with the verbatim array at a 4-byte (not 16-byte) aligned device address:
    the reconstruct sweep's scalar refill path (the batched pipelines always
    pass 256-byte aligned arrays)."""
    import ctypes

    import torch
    from paper_1706_03791_b200 import _native as nat

    rng = np.random.default_rng(5)
    dims = (45, 37, 29)
    n = int(np.prod(dims))
    v = (np.cumsum(rng.standard_normal(n)) * 0.1).astype(np.float32)
    v[rng.choice(n, n // 4, replace=False)] += rng.laplace(0, 5, n // 4).astype(np.float32)
    for m in (8, 12):
        eb = oracle.effective_bound(v, relative=1e-4)
        codes_ref, recon_ref, k_ref = oracle.compress_scan(v, dims, 1, m, eb)
        ctx = gpu
        dev = torch.device("cuda", ctx.device)
        ct = torch.uint8 if m <= 8 else torch.int16
        d_v = torch.from_numpy(v).to(dev)
        d_codes = torch.empty(n, dtype=ct, device=dev)
        d_recon = torch.empty(n, dtype=torch.float32, device=dev)
        d_hist = torch.zeros(1 << m, dtype=torch.int64, device=dev)
        info = nat.EbzInfo()
        info.eb = eb
        d_info = torch.frombuffer(bytearray(bytes(info)), dtype=torch.uint8).to(dev)
        dims_a = nat.dims_array(dims)
        rc = ctx.lib.ebz_compress_scan(ctx.handle, d_v.data_ptr(), 32, 3, dims_a, 1, m,
                                       d_codes.data_ptr(), d_recon.data_ptr(),
                                       d_hist.data_ptr(), d_info.data_ptr(), None)
        assert rc == 0
        torch.cuda.synchronize()
        codes = d_codes.cpu().numpy().astype(np.int64) & ((1 << 16) - 1)
        assert np.array_equal(codes, codes_ref)
        unpred = v[codes_ref == 0]
        assert unpred.size == k_ref
        # verbatim values 4 bytes past a 256-byte aligned allocation
        raw = torch.zeros(unpred.size + 8, dtype=torch.float32, device=dev)
        raw[1:1 + unpred.size] = torch.from_numpy(unpred).to(dev)
        d_out = torch.empty(n, dtype=torch.float32, device=dev)
        info2 = nat.EbzInfo()
        info2.eb = eb
        d_info2 = torch.frombuffer(bytearray(bytes(info2)), dtype=torch.uint8).to(dev)
        rc = ctx.lib.ebz_decompress_scan(ctx.handle, d_codes.data_ptr(), 32, 3, dims_a, 1, m,
                                         raw.data_ptr() + 4, unpred.size, d_out.data_ptr(),
                                         d_info2.data_ptr(), None)
        assert rc == 0
        torch.cuda.synchronize()
        out = d_out.cpu().numpy()
        back, used = oracle.decompress_scan(codes_ref, unpred, dims, 1, m, eb, 32)
        assert used == unpred.size
        assert out.tobytes() == back.tobytes() == recon_ref.tobytes()
        got = nat.EbzInfo.from_buffer_copy(d_info2.cpu().numpy().tobytes())
        assert got.status == 0 and got.used == unpred.size


@pytest.mark.parametrize("dims,layers", [((40, 24, 16), 1), ((67, 45), 1), ((33, 17, 11), 2)])
def test_nonfinite_verbatim_value_raises_like_reference(gpu, dims, layers):
    # a container whose verbatim block carries Inf / NaN decompresses to a
    # non-finite grid: the reference's DataGrid check raises (core.py:92-93,
    # message checked against the installed reference); single and batched
    from dataclasses import replace
    rng = np.random.default_rng(3)
    n = int(np.prod(dims))
    v = np.cumsum(rng.standard_normal(n)).astype(np.float32)
    v[::97] += 50
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-5), layers=layers)
    st = ebz.compress(ebz.DataGrid(dims, v), cfg).stream
    assert st.n_unpredictable > 2
    for bad in (np.inf, -np.inf, np.nan):
        u = np.array(st.unpredictable_values, copy=True)
        u[len(u) // 2] = bad
        st2 = replace(st, unpredictable_values=u)
        with pytest.raises(ValueError, match="values must be finite"):
            ebz.decompress(st2)
        with pytest.raises(ValueError, match="values must be finite"):
            ebz.decompress_many([st, st2])
    # the untouched stream still decompresses (status is per field)
    assert ebz.decompress_many([st])[0].values.tobytes() == ebz.decompress(st).values.tobytes()
