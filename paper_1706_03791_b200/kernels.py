"""The reference's kernel seam, bound to the B200 library.

``ebzip/_kernels.py`` holds the reference's compiled inner loops (numba):
``compress_scan``, ``decompress_scan``, ``original_hits``, ``pack_bits`` and
``unpack_bits``.  This module exports functions of the same names taking the
same arguments -- caller-allocated host numpy buffers, outputs filled in
place, the same return values and sentinels -- each a ctypes call into one
``ebz_ref_*`` entry point of ``libebz200.so`` (``include/ebz200.h``), which
stages the buffers on the device and runs the sm_100a kernels.  A
reference maintainer swaps the seam with one assignment per function
(INTEGRATION.md); nothing above it changes.

Differences a caller can observe, all outside what the reference's own
callers do (``codec.py:101-106,152-157``, ``entropy.py:153-154,168-175``,
``analysis.py:129``):

* the stencil bank must be ``codec._stencil_bank(layers, dims)`` and
  ``center`` must be ``2**(m-1)`` with 2 <= m <= 16 (``ValueError``);
* ``pack_bits`` requires canonical ``code_words`` and ``unpack_bits``
  canonical decode tables with ``n_bits == 8 * len(data)``;
* ``decompress_scan`` rejects codes outside ``[0, 2**m)``.

There is no CPU path: without the library or a B200 every call raises
``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat

__all__ = ["compress_scan", "decompress_scan", "original_hits", "pack_bits", "unpack_bits"]


def _arr(a, dtype, name, writable=False):
    if not isinstance(a, np.ndarray) or a.dtype != np.dtype(dtype) or not a.flags.c_contiguous:
        raise TypeError(f"{name} must be a C-contiguous {np.dtype(dtype)} array")
    if writable and not a.flags.writeable:
        raise TypeError(f"{name} must be writable")
    return a


def _elem(a, name, writable=False):
    if not isinstance(a, np.ndarray) or a.dtype not in (np.float32, np.float64):
        raise TypeError(f"{name} must be a float32 or float64 array")
    return _arr(a, a.dtype, name, writable), 8 * a.dtype.itemsize


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def _bank(deltas, coeffs, starts, counts):
    d = _arr(np.ascontiguousarray(deltas, np.int64), np.int64, "deltas")
    c = _arr(np.ascontiguousarray(coeffs, np.float64), np.float64, "coeffs")
    s = _arr(np.ascontiguousarray(starts, np.int64), np.int64, "starts")
    k = _arr(np.ascontiguousarray(counts, np.int64), np.int64, "counts")
    if d.size != c.size or s.size != k.size:
        raise ValueError("stencil bank arrays have inconsistent lengths")
    return d, c, s, k


def _call(fn, *args):
    ctx = nat.context()
    out = ctypes.c_longlong(0)
    with ctx.lock:
        rc = getattr(ctx.lib, fn)(ctx.handle, *args, ctypes.byref(out))
    if rc == -1:  # EBZ_E_ARG: the reference would have failed or misbehaved
        raise ValueError(f"{fn}: {nat.last_error()}")
    ctx.check(rc, fn)
    return int(out.value)


def compress_scan(values, recon, codes, deltas, coeffs, starts, counts, dims, layers, center,
                  bound):
    """Quantize every point against its prediction; fills ``recon`` and
    ``codes``, returns the number of unpredictable points
    (``_kernels.py:48-80``)."""
    values, width = _elem(values, "values")
    _arr(recon, values.dtype, "recon", writable=True)
    _arr(codes, np.int32, "codes", writable=True)
    if recon.size != values.size or codes.size != values.size:
        raise ValueError("values, recon and codes must have the same length")
    d, c, s, k = _bank(deltas, coeffs, starts, counts)
    dm = np.ascontiguousarray(dims, np.int64)
    if int(np.prod(dm)) != values.size:
        raise ValueError("dims do not match the value count")
    return _call("ebz_ref_compress_scan", _p(values), width, _p(recon), _p(codes), _p(d), _p(c),
                 d.size, _p(s), _p(k), s.size, _p(dm), dm.size, int(layers), int(center),
                 float(bound))


def decompress_scan(codes, recon, unpredictable, deltas, coeffs, starts, counts, dims, layers,
                    center, bound):
    """Rebuild ``recon`` from codes; returns the verbatim values consumed, or
    -1 when the unpredictable block runs out (``_kernels.py:83-105``)."""
    codes = _arr(np.ascontiguousarray(codes, np.int32), np.int32, "codes")
    recon, width = _elem(recon, "recon", writable=True)
    unp = _arr(np.ascontiguousarray(unpredictable, recon.dtype), recon.dtype, "unpredictable")
    if recon.size != codes.size:
        raise ValueError("codes and recon must have the same length")
    d, c, s, k = _bank(deltas, coeffs, starts, counts)
    dm = np.ascontiguousarray(dims, np.int64)
    if int(np.prod(dm)) != codes.size:
        raise ValueError("dims do not match the code count")
    return _call("ebz_ref_decompress_scan", _p(codes), _p(recon), width, _p(unp), unp.size,
                 _p(d), _p(c), d.size, _p(s), _p(k), s.size, _p(dm), dm.size, int(layers),
                 int(center), float(bound))


def original_hits(values, deltas, coeffs, starts, counts, dims, layers, bound):
    """Points predicted within ``bound`` from the original values
    (``_kernels.py:108-121``)."""
    values, width = _elem(values, "values")
    d, c, s, k = _bank(deltas, coeffs, starts, counts)
    dm = np.ascontiguousarray(dims, np.int64)
    return _call("ebz_ref_original_hits", _p(values), width, _p(d), _p(c), d.size, _p(s), _p(k),
                 s.size, _p(dm), dm.size, int(layers), float(bound))


def pack_bits(symbols, code_words, code_lens, out):
    """Concatenate each symbol's codeword MSB-first into ``out`` (zeroed
    uint8); returns the total bit count (``_kernels.py:124-148``)."""
    sym = _arr(np.ascontiguousarray(symbols, np.int32), np.int32, "symbols")
    words = _arr(np.ascontiguousarray(code_words, np.uint64), np.uint64, "code_words")
    lens = _arr(np.ascontiguousarray(code_lens, np.uint8), np.uint8, "code_lens")
    _arr(out, np.uint8, "out", writable=True)
    if words.size != lens.size:
        raise ValueError("code_words and code_lens must have the same length")
    return _call("ebz_ref_pack_bits", _p(sym), sym.size, _p(words), _p(lens), lens.size, _p(out),
                 out.size)


def unpack_bits(data, n_bits, first_codes, level_counts, level_base, ordered_symbols, max_len,
                out):
    """Canonical decode until ``out`` is full: the symbol count, -1 when the
    bits run out, -2 on an invalid prefix (``_kernels.py:151-183``)."""
    buf = _arr(np.ascontiguousarray(data, np.uint8), np.uint8, "data")
    fc = _arr(np.ascontiguousarray(first_codes, np.uint64), np.uint64, "first_codes")
    lc = _arr(np.ascontiguousarray(level_counts, np.int64), np.int64, "level_counts")
    lb = _arr(np.ascontiguousarray(level_base, np.int64), np.int64, "level_base")
    od = _arr(np.ascontiguousarray(ordered_symbols, np.int32), np.int32, "ordered_symbols")
    _arr(out, np.int32, "out", writable=True)
    if min(fc.size, lc.size, lb.size) <= int(max_len):
        raise ValueError("decode tables shorter than max_len + 1")
    return _call("ebz_ref_unpack_bits", _p(buf), buf.size, int(n_bits), _p(fc), _p(lc), _p(lb),
                 _p(od), od.size, int(max_len), _p(out), out.size)
