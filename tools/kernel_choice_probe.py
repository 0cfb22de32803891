"""Compress-sweep time of 3D n = 1 float32 fields over shapes and field counts,
for the three-kernel choice (sweep3.cu sweep3_model_choice).  Run three times:
EBZ_SWEEP3=always (sweep3c), EBZ_SWEEP3=never (two-row), EBZ_SWEEP3B32=c
(one-row sweep3b); in-stream stage events."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1706_03791_b200 as ebz  # noqa: E402
from paper_1706_03791_b200.device import DeviceBatch  # noqa: E402


def one(shape, nf, reps=3):
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
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-4))
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
    print(json.dumps({"shape": shape, "nf": nf, "mode": os.environ.get("EBZ_SWEEP3B32") and "s3b" or os.environ.get("EBZ_SWEEP3", "auto"),
                      "sweep_c_ms": round(ms[1] / cnt[1], 4),
                      "sweep_d_ms": round(ms[6] / cnt[6], 4)}), flush=True)
    del b


if __name__ == "__main__":
    shapes = [(128, 128, 128), (256, 256, 256), (512, 512, 512), (128, 512, 512),
              (512, 128, 512), (512, 512, 128), (100, 500, 500), (500, 500, 100),
              (64, 1024, 1024), (1024, 64, 256), (32, 32, 2048)]
    for shp in shapes:
        n = shp[0] * shp[1] * shp[2]
        for nf in (1, 2, 4, 8, 16):
            if n * nf * 4 > (2 << 30):
                continue
            one(shp, nf)
