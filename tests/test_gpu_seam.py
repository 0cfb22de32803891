"""The reference's kernel seam (ebzip/_kernels.py) through libebz200.

``paper_1706_03791_b200.kernels`` exposes compress_scan / decompress_scan /
original_hits / pack_bits / unpack_bits with the reference's exact
arguments on host numpy buffers (C entry points ``ebz_ref_*``).  Checked
against the CPU oracle's restatement of the same kernels (codes, recon
bytes, K; used / -1; bits / -1 / -2) on the fast 2D / 3D kernels and the
generic one (d = 1 and 4, n = 3, float64), and -- when the installed
reference (``baseline/_ref``, git-ignored, shipped with the repo) is
importable -- by running the reference's own ``codec.compress`` /
``decompress`` with its seam swapped for this one.
"""

import hashlib
import os
import sys

import numpy as np
import pytest

from paper_1706_03791_b200 import kernels as K

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _field(rng, dims, dtype, spiky=True):
    n = int(np.prod(dims))
    v = np.cumsum(rng.standard_normal(n)).reshape(tuple(reversed(dims)))
    for ax in range(v.ndim):
        v = np.cumsum(v, axis=ax) * 0.3
    v = v.reshape(-1)
    if spiky:
        idx = rng.integers(0, n, max(1, n // 50))
        v[idx] += rng.laplace(0, 5 * (v.std() + 1), idx.size)
    return v.astype(dtype)


# (dims fastest first, layers, dtype, m): fast 2D / 3D kernels (f32, n = 1, 2),
# the two-row 3D compress kernel, u16 codes, and the generic kernel
CASES = [
    ((67, 45), 1, np.float32, 8),
    ((64, 40), 2, np.float32, 8),
    ((33, 17, 11), 1, np.float32, 8),
    ((40, 24, 16), 1, np.float32, 12),
    ((21, 13, 9), 2, np.float32, 10),
    ((300,), 1, np.float32, 8),
    ((9, 7, 5, 4), 2, np.float64, 8),
    ((25, 19), 3, np.float64, 6),
    ((17, 11, 7), 1, np.float64, 16),
]


@pytest.mark.parametrize("dims,layers,dtype,m", CASES)
def test_compress_and_decompress_scan_match_oracle(gpu, oracle, dims, layers, dtype, m):
    rng = np.random.default_rng(hash((dims, layers, m)) & 0xFFFF)
    v = _field(rng, dims, dtype)
    eb = oracle.effective_bound(v, relative=10.0 ** rng.uniform(-5, -2))
    d, c, s, k = oracle.stencil_bank(layers, dims)
    center = 1 << (m - 1)
    recon = np.empty_like(v)
    codes = np.empty(v.size, np.int32)
    nk = K.compress_scan(v, recon, codes, d, c, s, k, np.asarray(dims, np.int64), layers,
                         center, eb)
    ref_codes, ref_recon, ref_k = oracle.compress_scan(v, dims, layers, m, eb)
    assert nk == ref_k
    assert np.array_equal(codes, ref_codes)
    assert recon.tobytes() == ref_recon.tobytes()
    # mirror scan from the same codes and the verbatim values in scan order
    unpred = v[codes == 0]
    out = np.empty_like(v)
    used = K.decompress_scan(codes, out, unpred, d, c, s, k, np.asarray(dims, np.int64), layers,
                             center, eb)
    assert used == nk
    assert out.tobytes() == ref_recon.tobytes()
    # underrun: one verbatim value short -> -1 (_kernels.py:97-99)
    if nk:
        assert K.decompress_scan(codes, out, unpred[:-1], d, c, s, k,
                                 np.asarray(dims, np.int64), layers, center, eb) == -1


def test_original_hits_matches_oracle(gpu, oracle):
    rng = np.random.default_rng(3)
    for dims, layers, dtype in [((50, 30), 1, np.float32), ((12, 9, 7), 2, np.float64),
                                ((200,), 3, np.float32)]:
        v = _field(rng, dims, dtype, spiky=False)
        d, c, s, k = oracle.stencil_bank(layers, dims)
        for bound in (1e-3, 1e-1, 1.0):
            assert K.original_hits(v, d, c, s, k, np.asarray(dims, np.int64), layers, bound) == \
                oracle.original_hits(v, dims, layers, bound)


def test_pack_and_unpack_bits_match_oracle(gpu, oracle):
    rng = np.random.default_rng(5)
    for nsym in (3, 200, 256, 1000, 65536):
        hist = rng.zipf(1.5, nsym).astype(np.int64)
        hist[rng.integers(0, nsym, nsym // 3)] = 0
        hist[0] = max(hist[0], 1)
        lengths = oracle.build_code(hist)
        words = oracle.code_words(lengths)
        used = np.nonzero(lengths)[0]
        sym = rng.choice(used, 5000).astype(np.int32)
        ref_bytes, nbits = oracle.encode(sym, lengths)
        out = np.zeros((nbits + 7) // 8, np.uint8)
        assert K.pack_bits(sym, words, lengths, out) == nbits
        assert out.tobytes() == ref_bytes
        # decode tables as CodeLengthTable._decode_tables builds them
        tabs = _decode_tables(lengths)
        got = np.empty(sym.size, np.int32)
        assert K.unpack_bits(out, out.size * 8, *tabs, got) == sym.size
        assert np.array_equal(got, sym)
        # exhausted (-1): one symbol more than the bits hold
        short = np.empty(sym.size + 64, np.int32)
        assert K.unpack_bits(out, out.size * 8, *tabs, short) == -1
    # invalid prefix (-2): an incomplete code, a bit pattern matching nothing
    lengths = np.array([1, 2, 0, 0], np.uint8)  # 0, 10; prefix 11 is unused
    tabs = _decode_tables(lengths)
    got = np.empty(4, np.int32)
    assert K.unpack_bits(np.array([0xFF], np.uint8), 8, *tabs, got) == -2


def _decode_tables(lengths):
    """entropy.py:67-84 restated (first_codes, level_counts, level_base,
    ordered, max_len)."""
    lengths = np.asarray(lengths, np.uint8)
    used = np.nonzero(lengths)[0]
    ordered = used[np.lexsort((used, lengths[used]))].astype(np.int32)
    level_counts = np.bincount(lengths[used].astype(np.int64), minlength=65).astype(np.int64)
    level_base = np.zeros(65, np.int64)
    level_base[1:] = np.cumsum(level_counts)[:-1]
    max_len = int(lengths[used].max())
    first_codes = np.zeros(65, np.uint64)
    word = 0
    for level in range(1, max_len + 1):
        word <<= 1
        first_codes[level] = word
        word += int(level_counts[level])
    return first_codes, level_counts, level_base, ordered, max_len


def test_seam_rejects_foreign_arguments(gpu, oracle):
    v = np.zeros(12, np.float32)
    d, c, s, k = oracle.stencil_bank(1, (4, 3))
    recon = np.empty_like(v)
    codes = np.empty(12, np.int32)
    with pytest.raises(ValueError, match="stencil bank"):
        K.compress_scan(v, recon, codes, d[:-1], c[:-1], s, k, np.array([4, 3]), 1, 128, 0.1)
    with pytest.raises(ValueError, match="center"):
        K.compress_scan(v, recon, codes, d, c, s, k, np.array([4, 3]), 1, 100, 0.1)
    with pytest.raises(TypeError):
        K.compress_scan(v, recon, codes.astype(np.int64), d, c, s, k, np.array([4, 3]), 1, 128,
                        0.1)


def _import_installed_reference():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "ebzip")):
        pytest.skip("installed reference (baseline/_ref) not present")
    try:
        import numba  # noqa: F401
    except ImportError:
        pytest.skip("numba not available")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ebz_numba_cache")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import ebzip
    return ebzip


def test_reference_codec_through_b200_seam(gpu, monkeypatch):
    """The reference's own compress / decompress (ebzip/codec.py:92-160),
    with its kernel seam rebound to this library exactly as INTEGRATION.md
    shows, produces the same containers and reconstructions as with its
    numba kernels."""
    ebzip = _import_installed_reference()
    import ebzip.codec as rc
    import ebzip.entropy as re_

    rng = np.random.default_rng(11)
    grids = [(_field(rng, (70, 50), np.float32), (70, 50), 1),
             (_field(rng, (30, 20, 12), np.float32), (30, 20, 12), 1),
             (_field(rng, (40, 30), np.float32), (40, 30), 2),
             (_field(rng, (9, 8, 7, 3), np.float64), (9, 8, 7, 3), 2)]
    expected = []
    for v, dims, layers in grids:
        cfg = ebzip.CompressorConfig(ebzip.ErrorBoundSpec(relative=1e-4), layers=layers)
        out = ebzip.compress(ebzip.DataGrid(dims, v), cfg)
        back = ebzip.decompress(out.stream)
        expected.append((ebzip.serialize(out.stream), out.recon_digest,
                         hashlib.sha256(back.values.tobytes()).hexdigest()))
    monkeypatch.setattr(rc, "compress_scan", K.compress_scan)
    monkeypatch.setattr(rc, "decompress_scan", K.decompress_scan)
    monkeypatch.setattr(re_, "pack_bits", K.pack_bits)
    monkeypatch.setattr(re_, "unpack_bits", K.unpack_bits)
    for (v, dims, layers), (blob, digest, back_digest) in zip(grids, expected):
        cfg = ebzip.CompressorConfig(ebzip.ErrorBoundSpec(relative=1e-4), layers=layers)
        out = ebzip.compress(ebzip.DataGrid(dims, v), cfg)
        assert ebzip.serialize(out.stream) == blob
        assert out.recon_digest == digest
        back = ebzip.decompress(ebzip.deserialize(blob))
        assert hashlib.sha256(back.values.tobytes()).hexdigest() == back_digest
