import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_1706_03791_b200 as ebz
from paper_1706_03791_b200 import codec
dims, layers, dtype, m0, rel, theta, rough = ((300, 180), 1, np.float32, 8, 1e-5, 0.9, 0.3)
rng = np.random.default_rng(abs(hash((dims, layers, m0))) % 2**32)
n = int(np.prod(dims))
v = (np.cumsum(rng.standard_normal(n)) * 0.05 + rough * rng.standard_normal(n)).astype(dtype)
grid = ebz.DataGrid(dims, v)
cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=rel), layers=layers, interval_exponent=m0, hitting_rate_threshold=theta)
ref, used, tr = codec._compress_auto_m_loop(grid, cfg)
print("loop", tr, ref.stream.code_bit_length, ref.stream.n_unpredictable)
for order in ["spec", "split", "spec", "split", "split"]:
    codec.AUTO_M_SPECULATE_POINTS = (1 << 26) if order == "spec" else 0
    out, u, t = ebz.compress_auto_m(grid, cfg)
    a, b = out.stream.code_lengths, ref.stream.code_lengths
    d = np.nonzero(a != b)[0]
    print(order, t, out.stream.code_bit_length, out.stream.n_unpredictable, "len diffs", d[:10], a[d[:5]], b[d[:5]])
