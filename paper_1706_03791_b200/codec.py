"""compress / decompress -- the drop-in entry points (ebzip/codec.py:92-160).

Same signatures, return types, warnings and exceptions as the reference;
the work runs on the B200 through ``libebz200.so``:

    compress(grid, config)   -> CompressionOutcome      (codec.py:92-136)
    decompress(stream)       -> DataGrid                (codec.py:139-160)
    compress_auto_m(...)     -> the CLI ``--auto-m`` loop (cli.py:146-154)

Host <-> device copies happen only at this API edge.  ``recon_digest`` (a
SHA-256 of the compressor's reconstruction, codec.py:135) is computed on
first access from a device decompression of the stream, which reproduces the
compressor's reconstruction bit for bit; the hash itself is a host-side,
inherently sequential computation and is kept off the compress path.
"""

from __future__ import annotations

import ctypes
import hashlib
from dataclasses import dataclass, replace

import numpy as np

from . import _native as nat
from .core import (
    CompressedStream,
    CompressorConfig,
    DataGrid,
    element_dtype,
    header_size,
)

MAX_INTERVAL_EXPONENT = 16
# context slots of the drop-in API (device batches use 0 .. 2*nfields)
API_SLOT = 1 << 20


@dataclass(frozen=True)
class IntervalSuggestion:
    """Raised-exponent advice when the hitting rate misses theta."""

    hitting_rate: float
    threshold: float
    suggested_exponent: int


class CompressionOutcome:
    """Result of one compression (fields as ebzip.codec.CompressionOutcome)."""

    __slots__ = ("stream", "hitting_rate", "warning", "_digest")

    def __init__(self, stream, hitting_rate, warning, recon_digest=None):
        self.stream = stream
        self.hitting_rate = hitting_rate
        self.warning = warning
        self._digest = recon_digest

    @property
    def recon_digest(self) -> str:
        if self._digest is None:
            self._digest = grid_digest(decompress(self.stream))
        return self._digest

    def __eq__(self, other):
        if not isinstance(other, CompressionOutcome):
            return NotImplemented
        return (self.stream == other.stream and self.hitting_rate == other.hitting_rate
                and self.warning == other.warning and self.recon_digest == other.recon_digest)

    def __repr__(self):
        return (f"CompressionOutcome(hitting_rate={self.hitting_rate!r}, "
                f"warning={self.warning!r}, K={self.stream.n_unpredictable})")


def grid_digest(grid: DataGrid) -> str:
    """SHA-256 of the grid's element bytes in scan order (codec.py:49-51)."""
    return hashlib.sha256(grid.values.tobytes()).hexdigest()


def _bound_args(config: CompressorConfig):
    b = config.bound
    return (1 if b.absolute is not None else 0, float(b.absolute or 0.0),
            1 if b.relative is not None else 0, float(b.relative or 0.0))


def _raise_compress_status(info: nat.EbzInfo):
    st = info.status
    if st & nat.ST_NONFINITE_IN:
        raise ValueError("values must be finite (no NaN/Inf)")
    if st & nat.ST_EB_NONPOSITIVE:
        raise ValueError(
            f"effective error bound must be positive, got {info.eb} "
            "(relative bound on a constant-range grid?)")
    if st & nat.ST_EMPTY_HIST:
        raise ValueError("histogram has no nonzero counts")
    if st & nat.ST_DEPTH_GT_64:
        raise ValueError("optimal code length exceeds 64")


def _outcome(grid_dims, n, width, config, info, head, bits, unpred) -> CompressionOutcome:
    m = config.interval_exponent
    hsz = header_size(len(grid_dims))
    stream = CompressedStream(
        element_width=width,
        dims=tuple(grid_dims),
        layers=config.layers,
        interval_exponent=m,
        eb_effective=float(info.eb),
        code_lengths=head[hsz:hsz + (1 << m)],
        code_bit_length=int(info.bit_length),
        code_bits=bits.tobytes(),
        unpredictable_values=unpred,
        unpredictable_coding=1 if getattr(config, "truncate_unpredictable", False) else 0,
    )
    return _outcome_of(stream, n, config, info)


def _outcome_of(stream, n, config, info) -> CompressionOutcome:
    """Hitting rate and interval advice (codec.py:121-130) around a stream."""
    m = config.interval_exponent
    rate = (n - int(info.n_unpred)) / n
    warning = None
    if rate < config.hitting_rate_threshold:
        warning = IntervalSuggestion(
            hitting_rate=rate,
            threshold=config.hitting_rate_threshold,
            suggested_exponent=min(m + 2, MAX_INTERVAL_EXPONENT),
        )
    return CompressionOutcome(stream, rate, warning)


def compress(grid: DataGrid, config: CompressorConfig, *, device: int | None = None
             ) -> CompressionOutcome:
    """Compress a grid under the configured bound (codec.py:92-136)."""
    ctx = nat.context(device)
    values = np.ascontiguousarray(grid.values)
    width = grid.element_width
    dims = nat.dims_array(grid.dims)
    info = nat.EbzInfo()
    ha, av, hr, rv = _bound_args(config)
    flags = 1 if config.truncate_unpredictable else 0  # EBZ_FLAG_TRUNCATE (opt-in)
    with ctx.lock:
        ctx.check(ctx.lib.ebz_compress_flags(
            ctx.handle, API_SLOT, nat.ptr(values), 1, width, grid.ndim, dims, config.layers,
            config.interval_exponent, flags, ha, av, hr, rv, None, ctypes.byref(info)),
            "ebz_compress_flags")
        _raise_compress_status(info)
        m = config.interval_exponent
        head = np.empty(header_size(grid.ndim) + (1 << m), np.uint8)
        bits = np.empty((int(info.bit_length) + 7) // 8, np.uint8)
        unpred = np.empty(int(info.n_unpred), element_dtype(width))
        ctx.check(ctx.lib.ebz_compress_fetch(
            ctx.handle, API_SLOT, nat.ptr(head), nat.ptr(bits), nat.ptr(unpred), None),
            "ebz_compress_fetch")
    return _outcome(grid.dims, grid.n_values, width, config, info, head, bits, unpred)


def _validate_table(lengths: np.ndarray):
    """CodeLengthTable checks (entropy.py:29-44), host-side metadata only."""
    from .entropy import CodeLengthTable
    CodeLengthTable(lengths)


def decompress(stream: CompressedStream, *, device: int | None = None) -> DataGrid:
    """Rebuild the reconstructed grid from a stream (codec.py:139-160)."""
    _validate_table(stream.code_lengths)
    ctx = nat.context(device)
    n = stream.n_points
    dtype = stream.element_dtype
    lengths = np.ascontiguousarray(stream.code_lengths, np.uint8)
    bits = np.frombuffer(stream.code_bits, np.uint8) if stream.code_bits else np.zeros(1, np.uint8)
    nbytes = len(stream.code_bits)
    unpred = np.ascontiguousarray(stream.unpredictable_values, dtype)
    if unpred.size == 0:
        unpred = np.zeros(1, dtype)
    recon = np.empty(n, dtype)
    info = nat.EbzInfo()
    with ctx.lock:
        ctx.check(ctx.lib.ebz_decompress(
            ctx.handle, API_SLOT + 1, 1, stream.element_width, len(stream.dims),
            nat.dims_array(stream.dims), stream.layers, stream.interval_exponent,
            float(stream.eb_effective), nat.ptr(lengths), nat.ptr(bits), nbytes,
            nat.ptr(unpred), stream.n_unpredictable, nat.ptr(recon), None,
            ctypes.byref(info)), "ebz_decompress")
    _raise_decompress_status(info, stream, nbytes)
    return _trusted_grid(stream.dims, recon)


def _raise_decompress_status(info: nat.EbzInfo, stream: CompressedStream, nbytes: int):
    """Device status -> the reference's errors, in the reference's order."""
    st = info.status
    if st & nat.ST_DEC_INVALID:
        raise ValueError("bit stream contains an invalid code prefix")
    if st & nat.ST_DEC_EXHAUSTED:
        raise ValueError(f"bit stream exhausted after {nbytes * 8} bits; "
                         f"expected {stream.n_points} symbols")
    if st & nat.ST_UNPRED_MISMATCH:
        raise ValueError(
            f"stream carries {stream.n_unpredictable} unpredictable values "
            f"but codes mark {int(info.zeros_decoded)}")
    if st & nat.ST_UNDERRUN or int(info.used) != stream.n_unpredictable:
        raise ValueError("unpredictable block not fully consumed")
    if st & nat.ST_NONFINITE_OUT:
        raise ValueError("values must be finite (no NaN/Inf)")


def _trusted_grid(dims, values: np.ndarray) -> DataGrid:
    """DataGrid around device-validated output (finiteness was checked on the
    device, ST_NONFINITE_OUT), skipping the redundant host pass."""
    grid = object.__new__(DataGrid)
    view = values.view()
    view.flags.writeable = False
    object.__setattr__(grid, "dims", tuple(int(v) for v in dims))
    object.__setattr__(grid, "values", view)
    return grid


# --auto-m: candidate exponents are swept speculatively in one batched launch
# while the batch stays below this many points (a lone field's wavefront
# leaves most of the GPU idle, so extra trials run in its shadow); larger
# fields sweep m0 first and batch the rest only if m0 misses theta
AUTO_M_SPECULATE_POINTS = 1 << 26
TRIAL_SLOT = API_SLOT + 64


def _trial_ks(ctx, values, grid, config, ms, slot0):
    """One batched predict/quantize sweep over the exponents ms
    (ebz_compress_trials); returns each trial's record (eb, status, K)."""
    ha, av, hr, rv = _bound_args(config)
    arr = (ctypes.c_int * len(ms))(*ms)
    ctx.check(ctx.lib.ebz_compress_trials(
        ctx.handle, slot0, nat.ptr(values), 1, grid.element_width, grid.ndim,
        nat.dims_array(grid.dims), config.layers, len(ms), arr, ha, av, hr, rv, None),
        "ebz_compress_trials")
    infos = []
    for i in range(len(ms)):
        inf = nat.EbzInfo()
        ctx.check(ctx.lib.ebz_slot_info(ctx.handle, slot0 + i, ctypes.byref(inf), None),
                  "ebz_slot_info")
        infos.append(inf)
    return infos


def compress_auto_m(grid: DataGrid, config: CompressorConfig, *, device: int | None = None):
    """CLI ``--auto-m`` semantics (cli.py:146-154): while the codec warns and
    m < 16, recompress at the suggested exponent m + 2.  Returns
    (outcome, final_config, trials).

    The trial sequence m0, m0 + 2, ... is fixed in advance and only each
    trial's K decides whether the loop goes on, so the candidates' sweeps run
    as one batched launch (ebz_compress_trials: per-field m over the same
    input) and only the chosen trial goes through the histogram, codebook
    and encoder (ebz_compress_trial_finish): the outcome is the one the loop
    ends with, element for element."""
    if config.truncate_unpredictable:  # the trials sweep the reference's coding only
        return _compress_auto_m_loop(grid, config, device=device)
    m0 = config.interval_exponent
    cand = [m0]
    while cand[-1] < MAX_INTERVAL_EXPONENT:
        cand.append(min(cand[-1] + 2, MAX_INTERVAL_EXPONENT))
    n = grid.n_values
    ctx = nat.context(device)
    values = np.ascontiguousarray(grid.values)
    theta = config.hitting_rate_threshold

    def stops(i, inf):  # the loop ends at trial i: no warning, or m = 16
        return (n - int(inf.n_unpred)) / n >= theta or cand[i] >= MAX_INTERVAL_EXPONENT

    with ctx.lock:
        spec = n * len(cand) <= AUTO_M_SPECULATE_POINTS
        batches = [cand] if spec else [cand[:1], cand[1:]]
        pick, slot, base = None, None, 0
        for b, ms in enumerate(batches):
            if not ms:
                continue
            slot0 = TRIAL_SLOT + base
            infos = _trial_ks(ctx, values, grid, config, ms, slot0)
            if any(inf.status for inf in infos):
                break  # an input / bound error: the plain path raises it in order
            for k, inf in enumerate(infos):
                if stops(base + k, inf):
                    pick, slot = base + k, slot0 + k
                    break
            if pick is not None:
                break
            base += len(ms)
        if pick is not None:
            info = nat.EbzInfo()
            ctx.check(ctx.lib.ebz_compress_trial_finish(ctx.handle, slot, None,
                                                        ctypes.byref(info)),
                      "ebz_compress_trial_finish")
            _raise_compress_status(info)
            final = replace(config, interval_exponent=cand[pick])
            m = cand[pick]
            head = np.empty(header_size(grid.ndim) + (1 << m), np.uint8)
            bits = np.empty((int(info.bit_length) + 7) // 8, np.uint8)
            unpred = np.empty(int(info.n_unpred), element_dtype(grid.element_width))
            ctx.check(ctx.lib.ebz_compress_fetch(
                ctx.handle, slot, nat.ptr(head), nat.ptr(bits), nat.ptr(unpred), None),
                "ebz_compress_fetch")
            outcome = _outcome(grid.dims, n, grid.element_width, final, info, head, bits,
                               unpred)
            return outcome, final, cand[:pick + 1]
    # error statuses: the reference loop's first compress raises
    return _compress_auto_m_loop(grid, config, device=device)


def _compress_auto_m_loop(grid: DataGrid, config: CompressorConfig, *,
                          device: int | None = None):
    """The loop itself, one full compression per trial (cli.py:146-154)."""
    outcome = compress(grid, config, device=device)
    current = config
    trials = [config.interval_exponent]
    while outcome.warning and current.interval_exponent < MAX_INTERVAL_EXPONENT:
        current = replace(current, interval_exponent=outcome.warning.suggested_exponent)
        trials.append(current.interval_exponent)
        outcome = compress(grid, current, device=device)
    return outcome, current, trials
