"""Host-side boundary: container bytes, typed errors, DataGrid/config
semantics -- mirrors the reference's tests/test_core.py pins (CPU only)."""

import numpy as np
import pytest

from paper_1706_03791_b200 import (
    CompressedStream, CompressorConfig, ContainerError, DataGrid, ErrorBoundSpec,
    MagicError, PayloadMismatchError, TruncatedError, VersionError, deserialize,
    grid_range, serialize,
)


def small_stream(**over):
    f = dict(element_width=64, dims=(4,), layers=1, interval_exponent=2, eb_effective=0.5,
             code_lengths=np.array([1, 1, 0, 0], np.uint8), code_bit_length=4,
             code_bits=b"\x50", unpredictable_values=np.array([7.0, 8.0]))
    f.update(over)
    return CompressedStream(**f)


# hand-assembled container (the reference's tests/test_core.py:38-55 layout)
GOLDEN = (b"EBZ1" + b"\x01" + b"\x01" + b"\x01" + b"\x02" + b"\x01" + b"\x00" * 3
          + b"\x04" + b"\x00" * 7 + b"\x00" * 6 + b"\xe0\x3f" + b"\x02" + b"\x00" * 7
          + b"\x04" + b"\x00" * 7 + b"\x01\x01\x00\x00" + b"\x50"
          + b"\x00" * 6 + b"\x1c\x40" + b"\x00" * 6 + b"\x20\x40")


def test_golden_bytes_and_roundtrip():
    assert serialize(small_stream()) == GOLDEN
    assert deserialize(GOLDEN) == small_stream()


def test_size_accounting():
    s = small_stream()
    assert len(serialize(s)) == 12 + 8 + 24 + 4 + 1 + 16


def test_typed_errors():
    with pytest.raises(MagicError):
        deserialize(b"XXXX" + GOLDEN[4:])
    with pytest.raises(VersionError):
        deserialize(GOLDEN[:4] + b"\x09" + GOLDEN[5:])
    for cut in (0, 5, 11, 20, len(GOLDEN) - 1):
        with pytest.raises(TruncatedError):
            deserialize(GOLDEN[:cut])
    with pytest.raises(PayloadMismatchError):
        deserialize(GOLDEN + b"\x00")
    bad = bytearray(GOLDEN); bad[9] = 1
    with pytest.raises(ContainerError):
        deserialize(bytes(bad))
    bad = bytearray(GOLDEN); bad[5] = 7
    with pytest.raises(ContainerError):
        deserialize(bytes(bad))
    bad = bytearray(GOLDEN); bad[28] = 200
    with pytest.raises(PayloadMismatchError):
        deserialize(bytes(bad))


def test_stream_validation():
    for over in (dict(eb_effective=0.0), dict(code_lengths=np.array([1, 1], np.uint8)),
                 dict(code_bits=b"\x50\x00"), dict(code_bit_length=100),
                 dict(unpredictable_values=np.zeros(9)), dict(element_width=16)):
        with pytest.raises(ValueError):
            small_stream(**over)


def test_float32_and_multidim_roundtrip():
    s = small_stream(element_width=32, unpredictable_values=np.array([7.0, 8.5], np.float32))
    again = deserialize(serialize(s))
    assert again == s and again.unpredictable_values.dtype == np.dtype("<f4")
    s = small_stream(dims=(2, 1, 2), layers=3)
    assert deserialize(serialize(s)) == s


def test_datagrid_semantics():
    a = np.arange(6, dtype=np.float64).reshape(2, 3)
    g = DataGrid.from_array(a)
    assert g.dims == (3, 2)
    assert np.array_equal(g.to_array(), a)
    assert g.values[1 + 3 * 1] == a[1, 1]
    with pytest.raises(ValueError):
        g.values[0] = 1.0
    for bad in (np.array([1, 2], np.int32), np.array([np.nan, 1.0]), np.array([np.inf, 1.0])):
        with pytest.raises(ValueError):
            DataGrid((2,), bad)
    with pytest.raises(ValueError):
        DataGrid((3,), np.zeros(4))
    with pytest.raises(ValueError):
        DataGrid((1, 1, 1, 1, 1), np.zeros(1))


def test_range_is_element_precision():
    v = np.array([1e8, 1e8 + 8, -3.0], np.float32)
    g = DataGrid((3,), v)
    assert grid_range(g) == float(np.float32(v.max()) - np.float32(v.min()))


def test_config_validation():
    b = ErrorBoundSpec(absolute=1.0)
    for kw in (dict(layers=0), dict(interval_exponent=1), dict(interval_exponent=17),
               dict(hitting_rate_threshold=0.0), dict(hitting_rate_threshold=1.5)):
        with pytest.raises(ValueError):
            CompressorConfig(bound=b, **kw)
    with pytest.raises(ValueError):
        ErrorBoundSpec()
    with pytest.raises(ValueError):
        ErrorBoundSpec(absolute=-1.0)
    with pytest.raises(ValueError):
        ErrorBoundSpec(relative=float("nan"))
    g = DataGrid((30,), np.linspace(0, 2, 30))
    assert ErrorBoundSpec(absolute=0.005, relative=0.01).effective_bound(g) == 0.005
    with pytest.raises(ValueError):
        ErrorBoundSpec(relative=0.01).effective_bound(DataGrid((3,), np.full(3, 2.0)))


def test_version2_header_of_the_truncated_extension():
    # the opt-in truncated-mantissa coding (not the reference's format) uses
    # container version 2 with the block size after the tail; version 3 is
    # rejected like any unknown version
    from paper_1706_03791_b200 import core as C
    head = C.pack_header(32, (4, 3), 8, 1, 0.5, 5, 17, block_bytes=9)
    blob = head + bytes(256) + bytes(3) + bytes(9)
    h = C.parse_header(blob)
    assert h["coding"] == 1 and h["end"] == len(blob) and h["n_unpred"] == 5
    with pytest.raises(C.TruncatedError):
        C.parse_header(blob[:-1])
    with pytest.raises(C.PayloadMismatchError):
        C.parse_header(blob + b"\0")
    bad = bytearray(blob)
    bad[4] = 3
    with pytest.raises(C.VersionError):
        C.parse_header(bytes(bad))
    plain = C.pack_header(32, (4, 3), 8, 1, 0.5, 5, 17)
    assert C.parse_header(plain + bytes(256) + bytes(3) + bytes(20))["coding"] == 0
    with pytest.raises(ValueError, match="unknown unpredictable coding"):
        C.CompressedStream(32, (4, 3), 1, 8, 0.5, np.zeros(256, np.uint8), 0, b"",
                           np.zeros(0, np.float32), unpredictable_coding=2)


def test_truncation_oracle_respects_the_bound(oracle):
    rng = np.random.default_rng(1)
    for dt in (np.float32, np.float64):
        v = (rng.standard_normal(5000) * 10.0 ** rng.uniform(-20, 20, 5000)).astype(dt)
        for eb in (1e-6, 0.25, 3.0e4):
            t = oracle.trunc_values(v, eb)
            assert np.all(np.abs(v.astype(np.float64) - t.astype(np.float64)) < eb)
            w = 64 if dt == np.float64 else 32
            assert oracle.tr_unpack(oracle.tr_pack(v, eb), v.size, w, eb).tobytes() == t.tobytes()
