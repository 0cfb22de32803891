"""Debug: sweep3 REC recon vs the oracle on the failing seam case."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
from paper_1706_03791_b200 import kernels as K
from oracle import oracle
from test_gpu_seam import _field
for dims, layers, dtype, m in [((40, 24, 16), 1, np.float32, 12), ((40, 24, 16), 1, np.float32, 8),
                               ((64, 40, 20), 1, np.float32, 8)]:
    rng = np.random.default_rng(hash((dims, layers, m)) & 0xFFFF)
    v = _field(rng, dims, dtype)
    eb = oracle.effective_bound(v, relative=10.0 ** rng.uniform(-5, -2))
    d, c, s, k = oracle.stencil_bank(layers, dims)
    center = 1 << (m - 1)
    for fill in (0.0, -0.0, 7.0):
        recon = np.full_like(v, fill)
        codes = np.empty(v.size, np.int32)
        nk = K.compress_scan(v, recon, codes, d, c, s, k, np.asarray(dims, np.int64), layers, center, eb)
        rc, rr, rk = oracle.compress_scan(v, dims, layers, m, eb)
        bad = np.nonzero(recon.view(np.uint32) != rr.view(np.uint32))[0]
        print(dims, m, "fill", fill, "K", nk, rk, "codes eq", np.array_equal(codes, rc), "nbad", bad.size,
              "first", [(int(i), float(recon[i]), float(rr[i]), int(codes[i])) for i in bad[:6]])
