"""Golden fixtures for the analysis / metrics callers,
produced by running the REFERENCE itself (build container only):

    python tests/golden/make_golden_analysis.py

Records: generator outputs (SHA-256 of the bytes), best_layer_scan,
interval_sweep and rate_distortion_sweep reports (and their CSV renderings), compute_metrics reports and
original-hit counts, for small seeded grids.  Output: analysis.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

import ebzip  # noqa: E402  (the reference)
from ebzip import analysis as A  # noqa: E402
from ebzip import metrics as M  # noqa: E402
from ebzip._kernels import original_hits  # noqa: E402
from ebzip.codec import _stencil_bank, compress, decompress  # noqa: E402
from ebzip.core import CompressorConfig, ErrorBoundSpec, serialize  # noqa: E402


def digest(grid):
    return hashlib.sha256(grid.values.tobytes()).hexdigest()


def cfg(rel=1e-3, layers=1, m=8, theta=0.9):
    return CompressorConfig(bound=ErrorBoundSpec(relative=rel), layers=layers,
                            interval_exponent=m, hitting_rate_threshold=theta)


def main():
    out = {"generators": [], "layer_scans": [], "interval_sweeps": [], "rd_sweeps": [],
           "metrics": [], "original_hits": []}
    for name in A.GENERATOR_NAMES:
        for dims in ((40,), (17, 11), (9, 7, 5), (5, 4, 3, 3)):
            for width in (32, 64):
                g = A.generate(name, dims, seed=3, width=width)
                out["generators"].append(dict(name=name, dims=list(dims), seed=3, width=width,
                                              sha256=digest(g)))
    grids = [("sines", (33, 21), 64), ("spiky", (13, 12, 9), 32), ("poly", (300,), 64),
             ("noise", (24, 20), 32)]
    for name, dims, width in grids:
        g = A.generate(name, dims, seed=5, width=width)
        rep = A.best_layer_scan(g, cfg(1e-3), candidates=(1, 2, 3))
        out["layer_scans"].append(dict(
            name=name, dims=list(dims), width=width, rel=1e-3, candidates=[1, 2, 3],
            rows=[[r.layers, r.hit_rate_original, r.hit_rate_decompressed] for r in rep.rows],
            recommended=rep.recommended_layers, csv=A.layer_scan_csv(rep)))
        sw = A.interval_sweep(g, cfg(1e-3), bounds=(1e-2, 1e-3, 1e-4), exponents=(4, 6, 8, 10))
        out["interval_sweeps"].append(dict(
            name=name, dims=list(dims), width=width, bounds=[1e-2, 1e-3, 1e-4],
            exponents=[4, 6, 8, 10], threshold=sw.threshold,
            cells=[[c.relative_bound, c.interval_exponent, c.hitting_rate, c.meets_threshold]
                   for c in sw.cells],
            selections=[[b, e] for b, e in sw.selections], csv=A.interval_sweep_csv(sw)))
        rd = A.rate_distortion_sweep(g, cfg(), bounds=(1e-2, 1e-3, 1e-4))
        out["rd_sweeps"].append(dict(
            name=name, dims=list(dims), width=width, bounds=[1e-2, 1e-3, 1e-4],
            points=[[p.relative_bound, p.bit_rate, p.psnr, p.compression_factor,
                     p.hitting_rate] for p in rd.points], csv=A.rate_distortion_csv(rd)))
        for layers in (1, 2, 3):
            for rel in (1e-2, 1e-4):
                bound = ErrorBoundSpec(relative=rel).effective_bound(g)
                d, c, s, k = _stencil_bank(layers, g.dims)
                hits = original_hits(g.values, d, c, s, k, np.asarray(g.dims, np.int64), layers,
                                     bound)
                out["original_hits"].append(dict(name=name, dims=list(dims), width=width,
                                                 layers=layers, rel=rel, hits=int(hits)))
        o = compress(g, cfg(1e-3))
        blob = serialize(o.stream)
        rec = decompress(o.stream)
        for lags in (0, 5, 100):
            r = M.compute_metrics(g, rec, compressed_bytes=len(blob), lags=lags)
            out["metrics"].append(dict(
                name=name, dims=list(dims), width=width, rel=1e-3, lags=lags,
                compressed_bytes=len(blob), recon_sha256=digest(rec),
                fields=[r.max_abs_error, r.max_rel_error, r.rmse, r.nrmse, r.psnr,
                        r.pearson_rho, r.compression_factor, r.bit_rate],
                autocorr=[float(v) for v in r.autocorr]))
    # degenerate: constant grid against itself (nan / inf sentinels)
    cg = A.generate("constant", (6, 5), width=64)
    r = M.compute_metrics(cg, cg, compressed_bytes=10, lags=3)
    out["metrics"].append(dict(name="constant", dims=[6, 5], width=64, rel=None, lags=3,
                               compressed_bytes=10, recon_sha256=digest(cg), self_pair=True,
                               fields=[r.max_abs_error, r.max_rel_error, r.rmse, r.nrmse,
                                       r.psnr, r.pearson_rho, r.compression_factor,
                                       r.bit_rate],
                               autocorr=[float(v) for v in r.autocorr]))
    out["reference_version"] = getattr(ebzip, "__version__", None)
    with open(os.path.join(HERE, "analysis.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print("wrote", os.path.join(HERE, "analysis.json"))


if __name__ == "__main__":
    main()
