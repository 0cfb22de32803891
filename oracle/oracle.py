"""CPU restatement of the reference compress/decompress path (test oracle).

TEST INFRASTRUCTURE ONLY -- the checker and the CPU baseline, never the
product.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.

It drives ``libebz_oracle.so`` (``oracle/ebz_oracle.c``) through ctypes and
mirrors the orchestration of the reference codec:

* ``compress_bytes``   -- ``ebzip/codec.py:92-136`` + ``core.py:295-316``
* ``decompress_bytes`` -- ``ebzip/codec.py:139-160`` + ``core.py:319-390``
* ``build_code``       -- ``ebzip/entropy.py:87-136``
* ``auto_m``           -- ``ebzip/cli.py:146-154`` (``--auto-m`` loop)

Parity of this restatement with the reference itself is pinned by
``tests/golden`` (fixtures produced by ``tests/golden/make_golden.py``, which
imports the reference package).

``compress_bytes(..., truncate=True)`` / ``tr_pack`` / ``tr_unpack`` restate
the opt-in truncated-mantissa extension (version-2 containers), which the
reference does not have: parity unpinned for that mode (it is checked
against this restatement and the error bound only).
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
import struct
import subprocess
from concurrent.futures import ThreadPoolExecutor
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libebz_oracle.so")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double


def build() -> str:
    """Compile the oracle library (gcc, no FMA contraction)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    if not os.path.exists(_LIB_PATH):
        build()
    so = ctypes.CDLL(_LIB_PATH)
    so.ora_stencil_bank_size.restype = _I64
    so.ora_stencil_bank_size.argtypes = [_I, _I]
    so.ora_stencil_bank.restype = None
    so.ora_stencil_bank.argtypes = [_I, _P, _I, _P, _P, _P, _P]
    so.ora_compress.restype = _I64
    so.ora_compress.argtypes = [_I, _P, _P, _P, _I, _P, _I, _I64, _D, _P, _P, _P, _P]
    so.ora_compress_tr.restype = _I64
    so.ora_compress_tr.argtypes = [_I, _P, _P, _P, _I, _P, _I, _I64, _D, _I, _P, _P, _P, _P]
    so.ora_decompress.restype = _I64
    so.ora_decompress.argtypes = [_I, _P, _P, _P, _I64, _I, _P, _I, _I64, _D,
                                  _P, _P, _P, _P]
    so.ora_original_hits.restype = _I64
    so.ora_original_hits.argtypes = [_I, _P, _I, _P, _I, _D, _P, _P, _P, _P]
    so.ora_build_code.restype = _I
    so.ora_build_code.argtypes = [_P, _I64, _P]
    so.ora_code_words.restype = None
    so.ora_code_words.argtypes = [_P, _I64, _P]
    so.ora_decode_tables.restype = _I
    so.ora_decode_tables.argtypes = [_P, _I64, _P, _P, _P, _P]
    so.ora_pack_bits.restype = _I64
    so.ora_pack_bits.argtypes = [_P, _I64, _P, _P, _P]
    so.ora_unpack_bits.restype = _I64
    so.ora_unpack_bits.argtypes = [_P, _I64, _P, _P, _P, _P, _I, _P, _I64]
    so.ora_range_f32.restype = None
    so.ora_range_f32.argtypes = [_P, _I64, _P]
    so.ora_range_f64.restype = None
    so.ora_range_f64.argtypes = [_P, _I64, _P]
    return so


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@lru_cache(maxsize=64)
def stencil_bank(layers: int, dims: tuple):
    """(deltas, coeffs, starts, counts) -- ``ebzip/codec.py:54-89``."""
    nd = len(dims)
    size = lib().ora_stencil_bank_size(nd, layers)
    deltas = np.zeros(max(size, 1), np.int64)
    coeffs = np.zeros(max(size, 1), np.float64)
    nslot = ((1 << nd) - 1) * layers
    starts = np.zeros(nslot, np.int64)
    counts = np.zeros(nslot, np.int64)
    dims_a = np.asarray(dims, np.int64)
    lib().ora_stencil_bank(nd, _ptr(dims_a), layers, _ptr(deltas), _ptr(coeffs),
                           _ptr(starts), _ptr(counts))
    return deltas, coeffs, starts, counts


def value_range(values: np.ndarray) -> float:
    out = np.zeros(3, np.float64)
    fn = lib().ora_range_f32 if values.dtype == np.float32 else lib().ora_range_f64
    fn(_ptr(values), values.size, _ptr(out))
    return float(out[2])


def effective_bound(values, absolute=None, relative=None) -> float:
    cands = []
    if absolute is not None:
        cands.append(float(absolute))
    if relative is not None:
        cands.append(float(relative) * value_range(values))
    eb = min(cands)
    if eb <= 0:
        raise ValueError("effective error bound must be positive")
    return eb


def compress_scan(values: np.ndarray, dims, layers: int, m: int, eb: float):
    """Returns (codes int32, recon elem, K)."""
    values = np.ascontiguousarray(values)
    width = 8 * values.dtype.itemsize
    d, c, s, n = stencil_bank(layers, tuple(int(v) for v in dims))
    recon = np.empty_like(values)
    codes = np.empty(values.size, np.int32)
    dims_a = np.asarray(dims, np.int64)
    k = lib().ora_compress(width, _ptr(values), _ptr(recon), _ptr(codes), len(dims),
                           _ptr(dims_a), layers, 1 << (m - 1), eb,
                           _ptr(d), _ptr(c), _ptr(s), _ptr(n))
    return codes, recon, int(k)


def decompress_scan(codes, unpred, dims, layers, m, eb, width):
    dt = np.float32 if width == 32 else np.float64
    codes = np.ascontiguousarray(codes, np.int32)
    unpred = np.ascontiguousarray(unpred, dt)
    d, c, s, n = stencil_bank(layers, tuple(int(v) for v in dims))
    recon = np.empty(codes.size, dt)
    dims_a = np.asarray(dims, np.int64)
    used = lib().ora_decompress(width, _ptr(codes), _ptr(recon), _ptr(unpred),
                                unpred.size, len(dims), _ptr(dims_a), layers,
                                1 << (m - 1), eb, _ptr(d), _ptr(c), _ptr(s), _ptr(n))
    return recon, int(used)


def original_hits(values, dims, layers, eb) -> int:
    values = np.ascontiguousarray(values)
    d, c, s, n = stencil_bank(layers, tuple(int(v) for v in dims))
    dims_a = np.asarray(dims, np.int64)
    return int(lib().ora_original_hits(8 * values.dtype.itemsize, _ptr(values),
                                       len(dims), _ptr(dims_a), layers, eb,
                                       _ptr(d), _ptr(c), _ptr(s), _ptr(n)))


def build_code(hist) -> np.ndarray:
    h = np.ascontiguousarray(hist, np.int64)
    lengths = np.zeros(h.size, np.uint8)
    rc = lib().ora_build_code(_ptr(h), h.size, _ptr(lengths))
    if rc == -1:
        raise ValueError("optimal code length exceeds 64")
    if rc == -2:
        raise ValueError("histogram has no nonzero counts")
    return lengths


def code_words(lengths) -> np.ndarray:
    ln = np.ascontiguousarray(lengths, np.uint8)
    words = np.zeros(ln.size, np.uint64)
    lib().ora_code_words(_ptr(ln), ln.size, _ptr(words))
    return words


def encode(codes, lengths):
    ln = np.ascontiguousarray(lengths, np.uint8)
    codes = np.ascontiguousarray(codes, np.int32)
    nbits = int(ln[codes].sum(dtype=np.int64)) if codes.size else 0
    out = np.zeros((nbits + 7) // 8, np.uint8)
    words = code_words(ln)
    got = lib().ora_pack_bits(_ptr(codes), codes.size, _ptr(words), _ptr(ln), _ptr(out))
    assert got == nbits
    return out.tobytes(), nbits


def decode(data: bytes, lengths, count: int) -> np.ndarray:
    ln = np.ascontiguousarray(lengths, np.uint8)
    fc = np.zeros(65, np.uint64)
    lc = np.zeros(65, np.int64)
    lb = np.zeros(65, np.int64)
    ordered = np.zeros(max(int((ln > 0).sum()), 1), np.int32)
    max_len = lib().ora_decode_tables(_ptr(ln), ln.size, _ptr(fc), _ptr(lc), _ptr(lb),
                                      _ptr(ordered))
    buf = np.frombuffer(bytes(data), np.uint8).copy()
    out = np.empty(count, np.int32)
    if count == 0:
        return out
    st = lib().ora_unpack_bits(_ptr(buf), buf.size * 8, _ptr(fc), _ptr(lc), _ptr(lb),
                               _ptr(ordered), max_len, _ptr(out), count)
    if st == -1:
        raise ValueError("bit stream exhausted")
    if st == -2:
        raise ValueError("bit stream contains an invalid code prefix")
    return out


def _header(width, dims, m, layers, eb, k, nbits, block_bytes=None) -> bytes:
    return (struct.pack("<4sBBBBB3s", b"EBZ1", 1 if block_bytes is None else 2,
                        1 if width == 64 else 0, len(dims), m, layers, b"\0\0\0")
            + struct.pack(f"<{len(dims)}Q", *dims)
            + struct.pack("<dQQ", eb, k, nbits)
            + (b"" if block_bytes is None else struct.pack("<Q", block_bytes)))


# -- the opt-in truncated-mantissa extension (no reference counterpart) ------

def eb_exponent(eb: float) -> int:
    """floor(log2 eb) of a normal binary64 eb."""
    mant, e = math.frexp(eb)
    return e - 1


def _tr_fields(values: np.ndarray, eb: float):
    """(header fields, kept bits k, mantissa fields) per value."""
    if values.dtype == np.float64:
        u, M, EW, BIAS = values.view(np.uint64).astype(np.uint64), 52, 11, 1023
    else:
        u, M, EW, BIAS = values.view(np.uint32).astype(np.uint64), 23, 8, 127
    E = ((u >> np.uint64(M)) & np.uint64((1 << EW) - 1)).astype(np.int64)
    k = np.where(E == 0, M, np.clip(E - BIAS - eb_exponent(eb), 0, M)).astype(np.int64)
    h = (u >> np.uint64(M)).astype(np.uint64)
    mant = (u & np.uint64((1 << M) - 1)) >> (np.uint64(M) - k.astype(np.uint64))
    return h, k, mant, EW + 1, M


def trunc_values(values: np.ndarray, eb: float) -> np.ndarray:
    h, k, mant, hb, M = _tr_fields(values, eb)
    u = (h << np.uint64(M)) | (mant << (np.uint64(M) - k.astype(np.uint64)))
    return u.astype(np.uint64 if values.dtype == np.float64 else np.uint32).view(values.dtype)


def _put_bits(bits: np.ndarray, pos: np.ndarray, vals: np.ndarray, n: np.ndarray):
    for b in range(int(n.max()) if n.size else 0):
        sel = n > b
        bits[pos[sel] + b] = (vals[sel] >> (n[sel] - 1 - b).astype(np.uint64)) & np.uint64(1)


def tr_pack(values: np.ndarray, eb: float) -> bytes:
    """Version-2 unpredictable block (header fields, then kept mantissa bits,
    MSB first, byte padded)."""
    h, k, mant, hb, M = _tr_fields(np.ascontiguousarray(values), eb)
    K = h.size
    total = hb * K + int(k.sum())
    bits = np.zeros(total + 7, np.uint8)
    _put_bits(bits, np.arange(K, dtype=np.int64) * hb, h, np.full(K, hb, np.int64))
    mpos = hb * K + np.concatenate(([0], np.cumsum(k)[:-1])) if K else np.zeros(0, np.int64)
    _put_bits(bits, mpos.astype(np.int64), mant, k)
    return np.packbits(bits[:((total + 7) // 8) * 8]).tobytes()


def tr_unpack(block: bytes, K: int, width: int, eb: float) -> np.ndarray:
    bits = np.unpackbits(np.frombuffer(block, np.uint8)).astype(np.uint64)
    M, EW, BIAS = (52, 11, 1023) if width == 64 else (23, 8, 127)
    hb = EW + 1

    def get(pos, n):
        out = np.zeros(pos.size, np.uint64)
        for b in range(int(n.max()) if n.size else 0):
            sel = n > b
            out[sel] = (out[sel] << np.uint64(1)) | bits[pos[sel] + b]
        return out

    h = get(np.arange(K, dtype=np.int64) * hb, np.full(K, hb, np.int64))
    E = (h & np.uint64((1 << EW) - 1)).astype(np.int64)
    k = np.where(E == 0, M, np.clip(E - BIAS - eb_exponent(eb), 0, M)).astype(np.int64)
    if (hb * K + int(k.sum()) + 7) // 8 != len(block):
        raise ValueError("truncated-mantissa block size does not match its header fields")
    mpos = hb * K + np.concatenate(([0], np.cumsum(k)[:-1])) if K else np.zeros(0, np.int64)
    mant = get(mpos.astype(np.int64), k)
    u = (h << np.uint64(M)) | (mant << (np.uint64(M) - k.astype(np.uint64)))
    return u.astype(np.uint64 if width == 64 else np.uint32).view(
        np.float64 if width == 64 else np.float32)


def compress_bytes(values: np.ndarray, dims, *, layers=1, m=8, absolute=None,
                   relative=None, theta=0.9, truncate=False):
    """Full reference pipeline -> dict(container, K, hitting_rate, warning,
    recon_digest, codes, recon).  truncate: the opt-in extension."""
    values = np.ascontiguousarray(values).ravel()
    dims = tuple(int(v) for v in dims)
    width = 8 * values.dtype.itemsize
    eb = effective_bound(values, absolute, relative)
    if truncate:
        d, c, s, n = stencil_bank(layers, dims)
        recon = np.empty_like(values)
        codes = np.empty(values.size, np.int32)
        dims_a = np.asarray(dims, np.int64)
        k = int(lib().ora_compress_tr(width, _ptr(values), _ptr(recon), _ptr(codes), len(dims),
                                      _ptr(dims_a), layers, 1 << (m - 1), eb, eb_exponent(eb),
                                      _ptr(d), _ptr(c), _ptr(s), _ptr(n)))
    else:
        codes, recon, k = compress_scan(values, dims, layers, m, eb)
    hist = np.bincount(codes, minlength=1 << m)
    lengths = build_code(hist)
    bits, nbits = encode(codes, lengths)
    unpred = values[codes == 0]
    if truncate:
        block = tr_pack(recon[codes == 0], eb)  # = trunc(values[codes == 0])
        blob = _header(width, dims, m, layers, eb, unpred.size, nbits, len(block)) \
            + lengths.tobytes() + bits + block
    else:
        blob = _header(width, dims, m, layers, eb, unpred.size, nbits) + lengths.tobytes() \
            + bits + unpred.tobytes()
    rate = (values.size - k) / values.size
    warn = None
    if rate < theta:
        warn = min(m + 2, 16)
    return dict(container=blob, K=k, hitting_rate=rate, suggested=warn, eb=eb,
                recon_digest=hashlib.sha256(recon.tobytes()).hexdigest(),
                codes=codes, recon=recon)


def decompress_bytes(blob: bytes) -> np.ndarray:
    """Container bytes -> reconstruction (flat scan order)."""
    magic, ver, wf, nd, m, layers, _ = struct.unpack_from("<4sBBBBB3s", blob, 0)
    pos = 12
    dims = struct.unpack_from(f"<{nd}Q", blob, pos)
    pos += 8 * nd
    eb, k, nbits = struct.unpack_from("<dQQ", blob, pos)
    pos += 24
    block_bytes = None
    if ver == 2:
        (block_bytes,) = struct.unpack_from("<Q", blob, pos)
        pos += 8
    lengths = np.frombuffer(blob, np.uint8, 1 << m, pos)
    pos += 1 << m
    nbytes = (nbits + 7) // 8
    bits = blob[pos:pos + nbytes]
    pos += nbytes
    width = 64 if wf else 32
    if block_bytes is not None:
        unpred = tr_unpack(blob[pos:pos + block_bytes], k, width, eb)
    else:
        unpred = np.frombuffer(blob, np.float64 if wf else np.float32, k, pos)
    n = math.prod(dims)
    codes = decode(bits, lengths, n)
    if int((codes == 0).sum()) != k:
        raise ValueError("unpredictable count mismatch")
    recon, used = decompress_scan(codes, unpred, dims, layers, m, eb, width)
    if used != k:
        raise ValueError("unpredictable block not fully consumed")
    return recon


def auto_m(values, dims, *, layers=1, m=8, absolute=None, relative=None, theta=0.9):
    """CLI ``--auto-m`` loop (``ebzip/cli.py:146-154``): recompress at the
    suggested exponent while the codec warns and m < 16."""
    out = compress_bytes(values, dims, layers=layers, m=m, absolute=absolute,
                         relative=relative, theta=theta)
    trials = [m]
    while out["suggested"] is not None and m < 16:
        m = out["suggested"]
        trials.append(m)
        out = compress_bytes(values, dims, layers=layers, m=m, absolute=absolute,
                             relative=relative, theta=theta)
    out["m"] = m
    out["trials"] = trials
    return out


def compress_many(fields, dims, workers: int | None = None, **kw):
    """Reference file-level parallelism (``ebzip/cli.py:100-113``): a thread
    pool over independent fields (the C scans release the GIL via ctypes)."""
    workers = workers or os.cpu_count() or 1
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(lambda v: compress_bytes(v, dims, **kw), fields))


def decompress_many(blobs, workers: int | None = None):
    workers = workers or os.cpu_count() or 1
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(decompress_bytes, blobs))
