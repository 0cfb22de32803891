"""Analysis / metrics callers of the path against
fixtures produced by the reference itself (tests/golden/analysis.json,
tests/golden/make_golden_analysis.py).

CPU tests: the synthetic generators (host numpy, bit-identical) and the
oracle's original_hits.  GPU tests: original_hits on the device (exact
counts, also against the oracle on random configurations), the layer scan,
interval sweep and rate-distortion sweep (exact hitting rates, sizes and
selections; PSNR to 1e-12 relative), and compute_metrics (max error exact,
reductions to 1e-12 relative: the device sums in a different order than
numpy's pairwise dot)."""

import hashlib
import json
import math
import os

import numpy as np
import pytest

import paper_1706_03791_b200 as ebz
from paper_1706_03791_b200 import analysis as A
from paper_1706_03791_b200 import metrics as M

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "analysis.json")
RTOL = 1e-12


@pytest.fixture(scope="module")
def gold():
    with open(GOLDEN) as fh:
        return json.load(fh)


def _close(a, b, rtol=RTOL):
    if isinstance(b, float) and math.isnan(b):
        return isinstance(a, float) and math.isnan(a)
    if isinstance(b, float) and math.isinf(b):
        return a == b
    return abs(a - b) <= rtol * max(1.0, abs(b))


def _cfg(rel=1e-3, layers=1, m=8, theta=0.9):
    return ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=rel), layers=layers,
                                interval_exponent=m, hitting_rate_threshold=theta)


def test_generators_bit_identical(gold):
    for c in gold["generators"]:
        g = A.generate(c["name"], c["dims"], seed=c["seed"], width=c["width"])
        assert hashlib.sha256(g.values.tobytes()).hexdigest() == c["sha256"], c
    with pytest.raises(ValueError):
        A.generate("bogus", (4,))
    with pytest.raises(ValueError):
        A.generate("sines", (4,), width=16)


def test_oracle_original_hits_pinned(gold, oracle):
    for c in gold["original_hits"]:
        g = A.generate(c["name"], c["dims"], seed=5, width=c["width"])
        bound = ebz.ErrorBoundSpec(relative=c["rel"]).effective_bound(g)
        assert oracle.original_hits(g.values, g.dims, c["layers"], bound) == c["hits"], c


def test_report_csv_matches_reference(gold):
    """CSV writers (ebzip/analysis.py:251-307) on reports rebuilt from the
    reference's own rows render the reference's CSV text byte for byte."""
    for c in gold["layer_scans"]:
        rep = A.LayerScanReport(rows=tuple(A.LayerScanRow(*r) for r in c["rows"]),
                                recommended_layers=c["recommended"])
        assert A.layer_scan_csv(rep) == c["csv"]
    for c in gold["interval_sweeps"]:
        rep = A.IntervalSweepReport(threshold=c["threshold"],
                                    cells=tuple(A.SweepCell(*x) for x in c["cells"]),
                                    selections=tuple(tuple(x) for x in c["selections"]))
        assert A.interval_sweep_csv(rep) == c["csv"]
    for c in gold["rd_sweeps"]:
        rep = A.RateDistortionReport(points=tuple(A.RatePoint(*p) for p in c["points"]))
        assert A.rate_distortion_csv(rep) == c["csv"]


@pytest.mark.gpu
def test_gpu_original_hits(gold, gpu, oracle):
    for c in gold["original_hits"]:
        g = A.generate(c["name"], c["dims"], seed=5, width=c["width"])
        bound = ebz.ErrorBoundSpec(relative=c["rel"]).effective_bound(g)
        assert A.original_hits(g, c["layers"], bound) == c["hits"], c
    rng = np.random.default_rng(21)
    for _ in range(40):
        nd = int(rng.integers(1, 5))
        dims = tuple(int(rng.integers(1, {1: 500, 2: 40, 3: 14, 4: 7}[nd])) for _ in range(nd))
        width = 32 if rng.random() < 0.5 else 64
        v = (np.cumsum(rng.standard_normal(int(np.prod(dims)))) * 0.1).astype(
            np.float32 if width == 32 else np.float64)
        g = ebz.DataGrid(dims, v)
        layers = int(rng.integers(1, 4))
        bound = float(10 ** rng.uniform(-3, 0))
        assert A.original_hits(g, layers, bound) == oracle.original_hits(v, dims, layers, bound)


@pytest.mark.gpu
def test_gpu_layer_scan_and_sweeps(gold, gpu):
    for c in gold["layer_scans"]:
        g = A.generate(c["name"], c["dims"], seed=5, width=c["width"])
        rep = A.best_layer_scan(g, _cfg(c["rel"]), candidates=c["candidates"])
        assert [[r.layers, r.hit_rate_original, r.hit_rate_decompressed] for r in rep.rows] \
            == c["rows"]
        assert rep.recommended_layers == c["recommended"]
        assert A.layer_scan_csv(rep) == c["csv"]
    for c in gold["interval_sweeps"]:
        g = A.generate(c["name"], c["dims"], seed=5, width=c["width"])
        rep = A.interval_sweep(g, _cfg(), c["bounds"], c["exponents"])
        assert rep.threshold == c["threshold"]
        assert [[x.relative_bound, x.interval_exponent, x.hitting_rate, x.meets_threshold]
                for x in rep.cells] == c["cells"]
        assert [list(s) for s in rep.selections] == c["selections"]
        assert A.interval_sweep_csv(rep) == c["csv"]
    for c in gold["rd_sweeps"]:
        g = A.generate(c["name"], c["dims"], seed=5, width=c["width"])
        rep = A.rate_distortion_sweep(g, _cfg(), c["bounds"])
        assert len(rep.points) == len(c["points"])
        for p, q in zip(rep.points, c["points"]):
            assert [p.relative_bound, p.bit_rate, p.compression_factor, p.hitting_rate] == \
                [q[0], q[1], q[3], q[4]]
            assert _close(p.psnr, q[2])
    with pytest.raises(ValueError):
        A.best_layer_scan(A.generate("sines", (8, 8)), _cfg(), candidates=())
    with pytest.raises(ValueError):
        A.interval_sweep(A.generate("sines", (8, 8)), _cfg(), [], [8])


@pytest.mark.gpu
def test_gpu_compute_metrics(gold, gpu):
    for c in gold["metrics"]:
        g = A.generate(c["name"], c["dims"], seed=5 if c["name"] != "constant" else 0,
                       width=c["width"])
        if c.get("self_pair"):
            rec = g
        else:
            out = ebz.compress(g, _cfg(c["rel"]))
            assert len(ebz.serialize(out.stream)) == c["compressed_bytes"]
            rec = ebz.decompress(out.stream)
            assert hashlib.sha256(rec.values.tobytes()).hexdigest() == c["recon_sha256"]
        r = M.compute_metrics(g, rec, compressed_bytes=c["compressed_bytes"], lags=c["lags"])
        got = [r.max_abs_error, r.max_rel_error, r.rmse, r.nrmse, r.psnr, r.pearson_rho,
               r.compression_factor, r.bit_rate]
        assert got[0] == c["fields"][0] or (math.isnan(got[0]) and math.isnan(c["fields"][0]))
        for a, b in zip(got, c["fields"]):
            assert _close(a, b), (c["name"], got, c["fields"])
        assert len(r.autocorr) == len(c["autocorr"])
        for a, b in zip(r.autocorr, c["autocorr"]):
            assert _close(float(a), b, 1e-10), (c["name"], list(r.autocorr), c["autocorr"])
        assert M.metrics_csv_row(r).count(",") == 7
    with pytest.raises(ValueError):
        M.compute_metrics(A.generate("sines", (4, 5)), A.generate("sines", (5, 4)))
    ac = M.autocorrelation(np.arange(10.0), lags=12)
    assert ac[0] == 1.0 and math.isnan(ac[11]) and math.isnan(ac[12])
    assert all(math.isnan(v) for v in M.autocorrelation(np.ones(5), lags=2))
