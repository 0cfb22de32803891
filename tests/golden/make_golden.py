"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``ebzip`` from ``/root/reference/pkg/src`` (numba JIT, cache in
/tmp) and records, for a spread of seeded small grids plus the full cfg1
field, the reference's container bytes, hitting rate, warning suggestion and
recon digest.  The output ``cases.npz`` is committed; tests and the GPU box
read only that file (the reference does not travel).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

import ebzip  # noqa: E402  (the reference)
from ebzip.codec import compress, decompress  # noqa: E402

from tools.synth import make_numpy, mixed_field  # noqa: E402


def field(rng, kind, n):
    if kind == "mixed":
        return mixed_field(rng, n, float(rng.uniform(0.0, 1.5)))
    if kind == "noise":
        return rng.standard_normal(n) * 10.0
    if kind == "spiky":
        v = mixed_field(rng, n, 0.05)
        idx = rng.choice(n, max(1, n // 50), replace=False)
        v[idx] += rng.laplace(0, 20.0, idx.size)
        return v
    if kind == "lognormal":
        return np.exp(rng.standard_normal(n) * 4.0 + np.linspace(-10, 10, n))
    if kind == "tiny":
        return (mixed_field(rng, n, 0.3) * 1e-30)
    if kind == "constant":
        return np.full(n, float(rng.uniform(-3, 3)))
    if kind == "ramp":
        return np.linspace(-1.0, 1.0, n) + 1e-3 * rng.standard_normal(n)
    raise KeyError(kind)


def cases():
    rng = np.random.default_rng(20260101)
    kinds = ["mixed", "noise", "spiky", "lognormal", "tiny", "constant", "ramp"]
    # shapes chosen to cover d = 1..4 and the specialised 2D / 3D kernels'
    # ragged edges (dims not multiples of the 32-row / 8x4 patch)
    shapes = [
        (97,), (1,), (5000,),
        (33, 65), (70, 45), (64, 32), (1, 17), (17, 1), (129, 3), (40, 40),
        (9, 13, 11), (17, 8, 5), (33, 9, 10), (8, 4, 7), (1, 1, 9), (20, 20, 20),
        (3, 4, 5, 6), (7, 6, 5, 4),
    ]
    out = []
    i = 0
    for shape in shapes:
        for rep in range(3):
            kind = kinds[(i + rep) % len(kinds)]
            n = int(np.prod(shape))
            v = field(rng, kind, n)
            width = 32 if (i + rep) % 2 == 0 else 64
            v = v.astype(np.float32 if width == 32 else np.float64)
            nd = len(shape)
            max_layers = {1: 4, 2: 4, 3: 2, 4: 1}[nd]
            layers = 1 + (i + rep) % max_layers
            m = [2, 4, 8, 8, 12, 16][(i * 3 + rep) % 6]
            if kind == "constant":
                bound = dict(absolute=1e-6)
            elif rep == 0:
                bound = dict(relative=float(10.0 ** -rng.integers(2, 6)))
            elif rep == 1:
                bound = dict(absolute=float(rng.uniform(1e-4, 0.2)) *
                             (1e-30 if kind == "tiny" else 1.0))
            else:
                bound = dict(relative=1e-3, absolute=0.05)
            out.append(dict(name=f"c{i:03d}_{rep}_{kind}", dims=shape, values=v,
                            layers=layers, m=m, theta=0.9, **bound))
        i += 1
    # explicit n = 2 / n = 3 in 2D and n = 2 in 3D on larger fields
    for j, (shape, layers) in enumerate([((80, 70), 2), ((64, 96), 3), ((40, 33, 17), 2),
                                         ((48, 40, 9), 1), ((300, 37), 2)]):
        n = int(np.prod(shape))
        v = mixed_field(np.random.default_rng(500 + j), n, 0.2).astype(np.float32)
        out.append(dict(name=f"n{layers}_{j}", dims=shape, values=v, layers=layers,
                        m=8, theta=0.9, relative=1e-4))
    # full cfg1 (BASELINE configs[0]): numpy-shape (256,256) -> dims (256,256)
    cfg1 = make_numpy("cfg1")
    out.append(dict(name="cfg1", dims=cfg1.shape[::-1], values=cfg1.reshape(-1),
                    layers=1, m=8, theta=0.9, relative=1e-4))
    # a small auto-m case (exercises m -> m+2 loop semantics)
    v = np.random.default_rng(7).standard_normal(60 * 50).astype(np.float32)
    out.append(dict(name="automx", dims=(60, 50), values=v, layers=1, m=4, theta=0.9,
                    relative=1e-3, auto_m=True))
    return out


def main():
    meta = []
    arrays = {}
    for c in cases():
        bound = ebzip.ErrorBoundSpec(absolute=c.get("absolute"), relative=c.get("relative"))
        m = c["m"]
        grid = ebzip.DataGrid(tuple(c["dims"]), c["values"])
        cfg = ebzip.CompressorConfig(bound=bound, layers=c["layers"],
                                     interval_exponent=m,
                                     hitting_rate_threshold=c["theta"])
        trials = [m]
        try:
            outcome = compress(grid, cfg)
        except ValueError as exc:
            meta.append(dict(name=c["name"], dims=list(c["dims"]), layers=c["layers"],
                             m=m, theta=c["theta"], absolute=c.get("absolute"),
                             relative=c.get("relative"), error=str(exc)))
            arrays[c["name"] + "__values"] = c["values"]
            continue
        if c.get("auto_m"):
            from dataclasses import replace
            while outcome.warning and cfg.interval_exponent < 16:
                cfg = replace(cfg, interval_exponent=outcome.warning.suggested_exponent)
                trials.append(cfg.interval_exponent)
                outcome = compress(grid, cfg)
        blob = ebzip.serialize(outcome.stream)
        recon = decompress(outcome.stream)
        assert recon.values.tobytes() is not None
        meta.append(dict(
            name=c["name"], dims=list(c["dims"]), layers=c["layers"], m=m,
            theta=c["theta"], absolute=c.get("absolute"), relative=c.get("relative"),
            auto_m=bool(c.get("auto_m")), trials=trials,
            final_m=cfg.interval_exponent,
            hitting_rate=outcome.hitting_rate,
            suggested=(outcome.warning.suggested_exponent if outcome.warning else None),
            recon_digest=outcome.recon_digest,
            eb=outcome.stream.eb_effective, K=outcome.stream.n_unpredictable,
            bit_length=outcome.stream.code_bit_length,
        ))
        arrays[c["name"] + "__values"] = c["values"]
        arrays[c["name"] + "__container"] = np.frombuffer(blob, np.uint8)
    arrays["__meta__"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    path = os.path.join(HERE, "cases.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {len(meta)} cases -> {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
