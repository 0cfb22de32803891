"""Sweep latency vs. patch-grid shape (critical-path diagnosis).

Times the compress / decompress sweeps alone (in-stream events) on smooth
random fields whose patch grids are 1x1, a Y chain, a Z chain and full.
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1706_03791_b200 as ebz  # noqa: E402
from paper_1706_03791_b200.device import DeviceBatch  # noqa: E402


def one(shape, reps=5):
    n = 1
    for s in shape:
        n *= s
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    f = torch.randn(shape, device="cuda", generator=g, dtype=torch.float64)
    for ax in range(len(shape)):
        f = f.cumsum(ax)
    f = (f / f.abs().max()).float().reshape(-1).contiguous()
    out = torch.empty_like(f)
    dims = tuple(reversed(shape))
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-4))
    b = DeviceBatch(nstreams=1)
    ctx = b.ctx
    for _ in range(2):
        b.roundtrip([f], dims, cfg, [out])
    torch.cuda.synchronize()
    ms = (ctypes.c_double * 8)()
    cnt = (ctypes.c_ulonglong * 8)()
    ctx.lib.ebz_stage_times(ctx.handle, ms, cnt, 8)
    ctx.lib.ebz_profile(ctx.handle, 1)
    for _ in range(reps):
        b.roundtrip([f], dims, cfg, [out])
    torch.cuda.synchronize()
    ctx.lib.ebz_profile(ctx.handle, 0)
    ctx.lib.ebz_stage_times(ctx.handle, ms, cnt, 8)
    ok = (out - f).abs().max().item() <= b.info(0).eb * 1.0000001
    print(json.dumps({"shape": shape, "sweep_c_ms": ms[1] / cnt[1], "sweep_d_ms": ms[6] / cnt[6],
                      "ok": ok}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        one(tuple(int(v) for v in sys.argv[1].split("x")), reps=1)
        sys.exit(0)
    for shp in [(4, 8, 256), (4, 8, 1024), (4, 256, 256), (64, 8, 256), (128, 8, 256),
                (64, 64, 256), (256, 256, 256), (32, 256), (1024, 256), (256, 4096)]:
        one(shp)
