import sys, os, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1706_03791_b200 as ebz
from oracle import oracle as O
rng = np.random.default_rng(99)
for trial in range(30):
    nd = int(rng.integers(1, 4))
    dims = tuple(int(rng.integers(4, 30)) for _ in range(nd))
    n = int(np.prod(dims))
    v = np.cumsum(rng.standard_normal(n)).astype(np.float32 if trial % 2 else np.float64)
    L = 1 + trial % 3; m = (4, 8, 12)[trial % 3]; ab = 1e-3 * float(np.ptp(v) or 1)
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(absolute=ab), layers=L, interval_exponent=m)
    first = ebz.serialize(ebz.compress(ebz.DataGrid(dims, v), cfg).stream)
    ref = O.compress_bytes(v, dims, layers=L, m=m, absolute=ab)
    ok1 = first == ref["container"]
    rec_gpu = ebz.decompress(ebz.deserialize(first)).values
    rec_ora = O.decompress_bytes(ref["container"])
    ok2 = rec_gpu.tobytes() == rec_ora.tobytes()
    again = ebz.serialize(ebz.compress(ebz.DataGrid(dims, rec_gpu), cfg).stream)
    ref2 = O.compress_bytes(rec_ora, dims, layers=L, m=m, absolute=ab)
    ok3 = again == ref2["container"]
    if not (ok1 and ok2 and ok3 and first == again):
        print("trial", trial, dims, v.dtype, "L", L, "m", m, "first==oracle", ok1, "recon==oracle", ok2, "again==oracle", ok3)
        if not ok2:
            d = np.flatnonzero(rec_gpu != rec_ora)
            print("  recon diffs", d.size, "first at", d[:5], rec_gpu[d[:3]], rec_ora[d[:3]])
        if not ok3:
            a = np.frombuffer(again, np.uint8); b = np.frombuffer(ref2["container"], np.uint8)
            print("  lens", a.size, b.size)
            dd = np.flatnonzero(a[:min(a.size,b.size)] != b[:min(a.size,b.size)])
            print("  first byte diff", dd[:5])
            codes_o, recon_o, k = O.compress_scan(rec_ora, dims, L, m, ab)
            print("  oracle K", k)
print("done")
