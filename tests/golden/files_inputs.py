"""Deterministic raw inputs of the multi-file driver fixtures (shared by
tests/golden/make_golden_files.py, which runs the reference CLI on them, and
tests/test_files.py, which runs the B200 driver on the same bytes)."""

from __future__ import annotations

from pathlib import Path

import numpy as np

DIMS = (40, 30, 20)   # reference order, axis 0 fastest
REL = 1e-4


def _smooth(seed: int, n: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    t = np.linspace(0.0, 1.0, n)
    return np.sin(25 * t) * 5 + np.cumsum(rng.standard_normal(n)) * 0.02


def make_inputs(d) -> dict[str, Path]:
    """Writes the raw files into directory `d`; returns name -> path."""
    d = Path(d)
    d.mkdir(parents=True, exist_ok=True)
    n = int(np.prod(DIMS))
    files = {
        "a.raw": _smooth(1, n).astype("<f4"),
        "b.raw": _smooth(2, n).astype("<f4"),
        "short.raw": _smooth(3, n - 7).astype("<f4"),          # wrong value count
        "nan.raw": np.where(np.arange(n) == 123, np.nan, _smooth(4, n)).astype("<f4"),
        # noise: m = 8 misses the 0.9 hitting rate, so --auto-m raises m
        "noisy.raw": np.random.default_rng(5).standard_normal(n).astype("<f4"),
        "wide.raw": _smooth(6, n).astype("<f8"),                # 64-bit elements
    }
    out = {}
    for name, arr in files.items():
        p = d / name
        arr.tofile(p)
        out[name] = p
    return out
