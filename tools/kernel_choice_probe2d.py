"""Sweep times of 2D fields over shapes, layers and field counts, for the
sweep2 / one-row kernel choice (run once as is and once with
EBZ_NO_SWEEP2=1; in-stream stage events)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1706_03791_b200 as ebz  # noqa: E402
from paper_1706_03791_b200.device import DeviceBatch  # noqa: E402


def one(shape, nf, layers, reps=3):
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    fs, outs = [], []
    for i in range(nf):
        f = torch.randn(shape, device="cuda", generator=g, dtype=torch.float32)
        for ax in range(len(shape)):
            f = f.cumsum(ax)
        f = (f / f.abs().max()).reshape(-1).contiguous()
        fs.append(f)
        outs.append(torch.empty_like(f))
    dims = tuple(reversed(shape))
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-4), layers=layers)
    b = DeviceBatch(nstreams=1)
    ctx = b.ctx
    for _ in range(2):
        b.roundtrip(fs, dims, cfg, outs)
    torch.cuda.synchronize()
    ms = (ctypes.c_double * 8)()
    cnt = (ctypes.c_ulonglong * 8)()
    ctx.lib.ebz_stage_times(ctx.handle, ms, cnt, 8)
    ctx.lib.ebz_profile(ctx.handle, 1)
    for _ in range(reps):
        b.roundtrip(fs, dims, cfg, outs)
    torch.cuda.synchronize()
    ctx.lib.ebz_profile(ctx.handle, 0)
    ctx.lib.ebz_stage_times(ctx.handle, ms, cnt, 8)
    print(json.dumps({"shape": shape, "nf": nf, "layers": layers,
                      "mode": "one-row" if os.environ.get("EBZ_NO_SWEEP2") else "sweep2",
                      "sweep_c_ms": round(ms[1] / cnt[1], 4),
                      "sweep_d_ms": round(ms[6] / cnt[6], 4)}), flush=True)
    del b


if __name__ == "__main__":
    for layers in (1, 2):
        for shp in [(256, 256), (1024, 1024), (1800, 3600), (4096, 512), (512, 4096)]:
            n = shp[0] * shp[1]
            for nf in (1, 4, 16, 64):
                if n * nf * 4 > (1 << 30):
                    continue
                one(shp, nf, layers)
