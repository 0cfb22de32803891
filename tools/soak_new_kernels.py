"""Soak of the sweep kernels (sweep2 f32 / f64, sweep3b f64 and forced f32, and --
by EBZ_SWEEP3 = always / never -- the z-rows, two-row and one-row float32 3D
kernels): random shapes, bounds, interval exponents and field contents
against the CPU oracle, byte for byte.  python tools/soak_new_kernels.py [N [SCALE]]
(SCALE multiplies the shape ranges: many patches in every direction)."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1706_03791_b200 as ebz  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker)


def field(rng, n, dt):
    kind = rng.integers(0, 4)
    t = np.linspace(0, rng.uniform(1, 60), n)
    if kind == 0:
        v = np.sin(t) * 10 ** rng.uniform(-3, 3) + 10 ** rng.uniform(-4, 0) * rng.standard_normal(n)
    elif kind == 1:
        v = np.cumsum(rng.standard_normal(n)) * 10 ** rng.uniform(-3, 1)
    elif kind == 2:
        v = rng.integers(-50, 50, n).astype(np.float64) * rng.choice([0.5, 1.0, 0.25])
    else:
        v = rng.standard_normal(n) * 10 ** rng.uniform(-5, 5)
    if rng.random() < 0.5:
        v[rng.integers(0, n, max(1, n // 30))] += 10 ** rng.uniform(0, 4)
    return v.astype(dt)


def main():
    ncase = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    sc = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(2024)
    bad = 0
    done = 0
    for i in range(ncase):
        nd = int(rng.choice([2, 3]))
        dt = np.float32 if rng.random() < 0.5 else np.float64
        if nd == 2:
            dims = (int(rng.integers(1, 300 * sc)), int(rng.integers(1, 130 * sc)))
            layers = int(rng.choice([1, 2]))
        else:
            dims = (int(rng.integers(1, 90 * sc)), int(rng.integers(1, 40 * sc)), int(rng.integers(1, 24 * sc)))
            layers = 1
        os.environ.pop("EBZ_SWEEP3B32", None)
        os.environ.pop("EBZ_SWEEP3", None)
        if nd == 3 and dt == np.float32:
            pick = rng.integers(0, 4)            # which float32 3D kernels take the case
            if pick == 0:
                os.environ["EBZ_SWEEP3B32"] = "cd"
            elif pick == 1:
                os.environ["EBZ_SWEEP3"] = "always"   # z-rows compress, one-row decompress
            elif pick == 2:
                os.environ["EBZ_SWEEP3"] = "never"    # two-row compress
                layers = int(rng.choice([1, 2]))       # (n = 2: the one-row kernel both ways)
        n = int(np.prod(dims))
        v = field(rng, n, dt)
        m = int(rng.choice([2, 4, 8, 8, 8, 10, 12, 16]))
        if rng.random() < 0.5:
            bound = dict(relative=float(10 ** rng.uniform(-7, -1)))
        else:
            bound = dict(absolute=float(10 ** rng.uniform(-6, 1)))
        try:
            ref = O.compress_bytes(v, dims, layers=layers, m=m, **bound)
        except ValueError:
            continue
        cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(**bound), layers=layers, interval_exponent=m)
        out = ebz.compress(ebz.DataGrid(dims, v), cfg)
        blob = ebz.serialize(out.stream)
        back = ebz.decompress(ebz.deserialize(blob))
        ok = blob == ref["container"] and \
            hashlib.sha256(back.values.tobytes()).hexdigest() == ref["recon_digest"]
        done += 1
        if not ok:
            bad += 1
            print("MISMATCH", i, dims, dt.__name__, layers, m, bound, flush=True)
    from paper_1706_03791_b200 import _native as nat
    print(f"soak: {ncase} cases, {done} compared, {bad} mismatches, "
          f"{nat.context().launches()} sweep launches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
