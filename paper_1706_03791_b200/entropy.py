"""Canonical prefix coding -- mirror of ``ebzip/entropy.py`` on the device.

``CodeLengthTable`` validation and table derivation are O(2^m) host
metadata; ``build_code`` / ``encode`` / ``decode`` run the same device
kernels the codec pipeline uses (huffman.cu, encode.cu, decode.cu), with
torch tensors as device buffers.
"""

from __future__ import annotations

import ctypes
from collections.abc import Mapping
from dataclasses import dataclass
from functools import cached_property

import numpy as np

from . import _native as nat

MAX_CODE_LENGTH = 64
MAX_ALPHABET = 1 << 16


@dataclass(frozen=True, eq=False)
class CodeLengthTable:
    """Per-symbol code lengths (0 = unused) + derived canonical tables."""

    lengths: np.ndarray

    def __post_init__(self):
        ln = np.ascontiguousarray(self.lengths, dtype=np.uint8)
        if ln.ndim != 1 or ln.size == 0:
            raise ValueError("lengths must be a non-empty one-dimensional array")
        if int(ln.max()) > MAX_CODE_LENGTH:
            raise ValueError(f"code length exceeds {MAX_CODE_LENGTH}")
        used = ln[ln > 0].astype(np.int64)
        if used.size == 0:
            raise ValueError("table has no coded symbols")
        # Kraft: sum 2^-l <= 1, evaluated exactly in integers
        if sum(1 << (MAX_CODE_LENGTH - int(v)) for v in used) > (1 << MAX_CODE_LENGTH):
            raise ValueError("lengths violate the Kraft inequality")
        view = ln.view()
        view.flags.writeable = False
        object.__setattr__(self, "lengths", view)

    @property
    def n_symbols(self) -> int:
        return int(self.lengths.size)

    @cached_property
    def code_words(self) -> np.ndarray:
        """Canonical words by (length, symbol), right-aligned u64."""
        ln = self.lengths
        words = np.zeros(ln.size, np.uint64)
        word = 0
        prev = 0
        for length in range(1, MAX_CODE_LENGTH + 1):
            for s in np.flatnonzero(ln == length):
                word <<= length - prev
                words[s] = word
                word += 1
                prev = length
        words.flags.writeable = False
        return words


def _alphabet_bits(n: int) -> int:
    m = 1
    while (1 << m) < n:
        m += 1
    return m


def _torch():
    import torch
    return torch


def _dev():
    return _torch().device("cuda", nat.context().device)


def build_code(histogram) -> CodeLengthTable:
    """Optimal lengths from counts (entropy.py:87-136), built on the GPU."""
    if isinstance(histogram, Mapping):
        counts = np.zeros(max(histogram) + 1, np.int64)
        for sym, c in histogram.items():
            counts[sym] = c
    else:
        counts = np.ascontiguousarray(histogram, dtype=np.int64)
    if counts.ndim != 1 or counts.size == 0:
        raise ValueError("histogram must be non-empty and one-dimensional")
    if counts.min() < 0:
        raise ValueError("histogram counts must be >= 0")
    if not counts.any():
        raise ValueError("histogram has no nonzero counts")
    if counts.size > MAX_ALPHABET:
        raise ValueError(f"alphabet larger than {MAX_ALPHABET} symbols")
    torch = _torch()
    ctx = nat.context()
    m = _alphabet_bits(counts.size)
    hist = torch.zeros(1 << m, dtype=torch.int64, device=_dev())
    hist[: counts.size] = torch.from_numpy(counts).to(hist.device)
    lengths = torch.zeros(1 << m, dtype=torch.uint8, device=hist.device)
    words = torch.zeros(1 << m, dtype=torch.int64, device=hist.device)
    info = torch.zeros(128, dtype=torch.uint8, device=hist.device)
    stream = torch.cuda.current_stream(hist.device).cuda_stream
    with ctx.lock:
        ctx.check(ctx.lib.ebz_build_code(ctx.handle, hist.data_ptr(), m, lengths.data_ptr(),
                                         words.data_ptr(), info.data_ptr(), stream),
                  "ebz_build_code")
        h = nat.EbzInfo.from_buffer_copy(info.cpu().numpy().tobytes()[:ctypes.sizeof(nat.EbzInfo)])
    if h.status & nat.ST_DEPTH_GT_64:
        raise ValueError(f"optimal code length exceeds {MAX_CODE_LENGTH}")
    return CodeLengthTable(lengths.cpu().numpy()[: counts.size].copy())


def encode(symbols, table: CodeLengthTable) -> tuple[bytes, int]:
    """Pack symbols MSB-first; returns (bytes, exact bit length)."""
    sym = np.ascontiguousarray(symbols, dtype=np.int32)
    if sym.ndim != 1:
        raise ValueError("symbols must be one-dimensional")
    if sym.size == 0:
        return b"", 0
    if int(sym.min()) < 0 or int(sym.max()) >= table.n_symbols:
        raise ValueError("symbol outside the table's alphabet")
    lens = table.lengths[sym]
    if not lens.all():
        raise ValueError(f"symbol {int(sym[np.argmin(lens)])} has no assigned code")
    torch = _torch()
    ctx = nat.context()
    dev = _dev()
    m = _alphabet_bits(table.n_symbols)
    m = max(m, 2)
    ln = np.zeros(1 << m, np.uint8)
    ln[: table.n_symbols] = table.lengths
    wd = np.zeros(1 << m, np.uint64)
    wd[: table.n_symbols] = table.code_words
    codes_np = sym.astype(np.uint8 if m <= 8 else np.uint16)
    codes = torch.from_numpy(codes_np).to(dev)
    d_len = torch.from_numpy(ln).to(dev)
    d_words = torch.from_numpy(wd.view(np.int64)).to(dev)
    nbits_max = int(lens.sum(dtype=np.int64))
    bits = torch.zeros(nbits_max // 8 + 64, dtype=torch.uint8, device=dev)
    info = torch.zeros(128, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    with ctx.lock:
        ctx.check(ctx.lib.ebz_pack_bits(ctx.handle, codes.data_ptr(), m, sym.size, None, 32,
                                        d_len.data_ptr(), d_words.data_ptr(), bits.data_ptr(),
                                        bits.numel(), None, info.data_ptr(), stream),
                  "ebz_pack_bits")
        h = nat.EbzInfo.from_buffer_copy(info.cpu().numpy().tobytes()[:ctypes.sizeof(nat.EbzInfo)])
    nbits = int(h.bit_length)
    if nbits != nbits_max:
        raise AssertionError("bit accounting mismatch")
    return bits[: (nbits + 7) // 8].cpu().numpy().tobytes(), nbits


def decode(data: bytes, table: CodeLengthTable, count: int) -> np.ndarray:
    """Decode exactly ``count`` symbols (entropy.py:160-183)."""
    if count < 0:
        raise ValueError(f"count must be >= 0, got {count}")
    if count == 0:
        return np.empty(0, np.int32)
    torch = _torch()
    ctx = nat.context()
    dev = _dev()
    m = max(_alphabet_bits(table.n_symbols), 2)
    ln = np.zeros(1 << m, np.uint8)
    ln[: table.n_symbols] = table.lengths
    raw = np.frombuffer(bytes(data), np.uint8)
    buf = np.zeros(raw.size + 64, np.uint8)
    buf[: raw.size] = raw
    d_bits = torch.from_numpy(buf).to(dev)
    d_len = torch.from_numpy(ln).to(dev)
    out = torch.zeros(count, dtype=torch.uint8 if m <= 8 else torch.int16, device=dev)
    info = torch.zeros(128, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    with ctx.lock:
        ctx.check(ctx.lib.ebz_unpack_bits(ctx.handle, d_bits.data_ptr(), raw.size,
                                          d_len.data_ptr(), m, count, out.data_ptr(),
                                          info.data_ptr(), stream), "ebz_unpack_bits")
        h = nat.EbzInfo.from_buffer_copy(info.cpu().numpy().tobytes()[:ctypes.sizeof(nat.EbzInfo)])
    if h.status & nat.ST_DEC_INVALID:
        raise ValueError("bit stream contains an invalid code prefix")
    if h.status & nat.ST_DEC_EXHAUSTED:
        raise ValueError(f"bit stream exhausted after {raw.size * 8} bits; "
                         f"expected {count} symbols")
    res = out.cpu().numpy()
    if m > 8:
        res = res.view(np.uint16)
    return res.astype(np.int32)
