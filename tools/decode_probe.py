"""Decoder throughput probe on synthetic symbol streams (seam entry points)."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_03791_b200 import entropy  # noqa: E402
from paper_1706_03791_b200 import _native as nat  # noqa: E402


def probe(name, sym):
    t = entropy.build_code(np.bincount(sym, minlength=256))
    data, nbits = entropy.encode(sym, t)
    ctx = nat.context()
    dev = torch.device("cuda", 0)
    raw = np.frombuffer(data, np.uint8)
    buf = np.zeros(raw.size + 64, np.uint8)
    buf[: raw.size] = raw
    d_bits = torch.from_numpy(buf).to(dev)
    d_len = torch.from_numpy(np.ascontiguousarray(t.lengths)).to(dev)
    out = torch.zeros(sym.size, dtype=torch.uint8, device=dev)
    info = torch.zeros(128, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        ctx.lib.ebz_unpack_bits(ctx.handle, d_bits.data_ptr(), raw.size, d_len.data_ptr(), 8,
                                sym.size, out.data_ptr(), info.data_ptr(), st)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ctx.lib.ebz_unpack_bits(ctx.handle, d_bits.data_ptr(), raw.size, d_len.data_ptr(), 8,
                                sym.size, out.data_ptr(), info.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    ok = bool((out.cpu().numpy() == sym).all())
    print(f"{name:28s} n={sym.size} bits/sym={nbits/sym.size:5.2f} maxlen={int(t.lengths.max())} "
          f"decode {ms:.3f} ms  ({sym.size/ms/1e6:.1f} Msym/ms) ok={ok}", flush=True)


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    n = 16_777_216
    if len(sys.argv) > 1 and sys.argv[1] == "mix":
        mix = np.where(rng.random(n) < 0.74, 0, rng.integers(1, 256, n)).astype(np.uint8)
        probe("74% zero + uniform", mix)
        sys.exit(0)
    probe("uniform256", rng.integers(0, 256, n).astype(np.uint8))
    probe("laplace(b=3)", np.clip(128 + np.round(rng.laplace(0, 3, n)), 0, 255).astype(np.uint8))
    mix = np.where(rng.random(n) < 0.74, 0, rng.integers(1, 256, n)).astype(np.uint8)
    probe("74% zero + uniform", mix)
    # blocky: long runs of zeros alternating with uniform regions
    blk = np.zeros(n, np.uint8)
    reg = rng.random(n // 4096) < 0.3
    for i in np.flatnonzero(reg):
        blk[i * 4096:(i + 1) * 4096] = rng.integers(1, 256, 4096)
    probe("blocky zeros/uniform", blk)
