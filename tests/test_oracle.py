"""The CPU oracle is pinned against the reference's own outputs and known
answers before it is trusted as a checker (CPU only)."""

import hashlib

import numpy as np
import pytest


def test_oracle_matches_reference_golden(golden, oracle):
    meta, z = golden
    for c in meta:
        v = z[c["name"] + "__values"]
        kw = dict(layers=c["layers"], m=c["m"], absolute=c["absolute"],
                  relative=c["relative"], theta=c["theta"])
        if "error" in c:
            with pytest.raises(ValueError):
                oracle.compress_bytes(v, c["dims"], **kw)
            continue
        if c.get("auto_m"):
            out = oracle.auto_m(v, c["dims"], **kw)
            assert out["trials"] == c["trials"], c["name"]
        else:
            out = oracle.compress_bytes(v, c["dims"], **kw)
        ref = z[c["name"] + "__container"].tobytes()
        assert out["container"] == ref, c["name"]
        assert out["recon_digest"] == c["recon_digest"], c["name"]
        assert out["hitting_rate"] == c["hitting_rate"], c["name"]
        rec = oracle.decompress_bytes(ref)
        assert hashlib.sha256(rec.tobytes()).hexdigest() == c["recon_digest"], c["name"]


# known answers from the reference's own tests (tests/test_entropy.py)
def test_huffman_known_answers(oracle):
    assert oracle.build_code([2, 1, 1]).tolist() == [1, 2, 2]
    assert oracle.code_words([1, 2, 2]).tolist() == [0, 0b10, 0b11]
    assert oracle.build_code([1, 1, 1, 1]).tolist() == [2, 2, 2, 2]
    assert oracle.build_code([2, 2, 2, 2, 2]).tolist() == [3, 3, 2, 2, 2]  # tie-break pin
    assert oracle.build_code([0, 5, 0]).tolist() == [0, 1, 0]
    data, nbits = oracle.encode([0, 0, 1], oracle.build_code([2, 1, 1]))
    assert (data, nbits) == (b"\x20", 4)
    data, nbits = oracle.encode([1] * 7, oracle.build_code([0, 7]))
    assert (data, nbits) == (b"\x00", 7)
    with pytest.raises(ValueError, match="exhausted"):
        d, _ = oracle.encode([0, 1, 2], oracle.build_code([2, 1, 1]))
        oracle.decode(d, oracle.build_code([2, 1, 1]), 50)
    with pytest.raises(ValueError, match="invalid"):
        oracle.decode(b"\xff", oracle.build_code([0, 9]), 2)


def test_quantizer_known_answers(oracle):
    # tests/test_quantizer.py:13-15 and :38-44 restated through the scan:
    # [10.0, 10.025] -> point 0 is verbatim (|s| = 500 > center + 1), so
    # point 1 is quantized against exactly 10.0 -> (129, 10.02).
    codes, recon, k = oracle.compress_scan(np.array([10.0, 10.025]), (2,), 1, 8, 0.01)
    assert codes.tolist() == [0, 129] and k == 1
    assert recon[1] == 10.0 + 1 * (2.0 * 0.01)
    # inexact tie demoted to unpredictable (quantize(0.03, 0, 0.01, 8) -> 0)
    codes, recon, k = oracle.compress_scan(np.array([0.03]), (1,), 1, 8, 0.01)
    assert codes.tolist() == [0] and recon[0] == 0.03
    # exhaustive interval scan (tests/test_quantizer.py:46-57): every
    # representable multiple reconstructs within the bound
    for m in (4, 8, 12):
        center = 1 << (m - 1)
        ks = np.arange(-(center - 1), center, max(1, center // 64))
        vals = np.concatenate([[0.0], ks * 0.02])
        codes, recon, _ = oracle.compress_scan(vals, (vals.size,), 1, m, 0.01)
        assert np.all(np.abs(recon - vals) <= 0.01)


def test_stencil_bank_table_one(oracle):
    # Table I coefficients for 2D n = 1, 2 (tests/_reference.py:17-39)
    d, c, s, n = oracle.stencil_bank(2, (10, 10))
    full = 2 * (3 - 1) + 1   # slot of mask {x,y}, eff = 2 -> (3-1)*2 + 1
    terms = c[s[full]:s[full] + n[full]].tolist()
    assert terms == [2, -1, 2, -4, 2, -1, 2, -1]
    d, c, s, n = oracle.stencil_bank(1, (10, 10))
    assert c[s[2]:s[2] + n[2]].tolist() == [1, 1, -1]
    assert d[s[2]:s[2] + n[2]].tolist() == [10, 1, 11]


def test_oracle_has_no_fma():
    """The restatement must not contract a + b*c (numba emits no FMA)."""
    import subprocess, os
    so = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle",
                      "libebz_oracle.so")
    out = subprocess.run(["objdump", "-d", so], capture_output=True, text=True).stdout
    assert "vfmadd" not in out and "vfnmadd" not in out
