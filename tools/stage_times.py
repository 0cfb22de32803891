"""Isolated per-stage device times (one stream, one field at a time).

    python tools/stage_times.py [cfg5 cfg3 ...] [--reps 5]

Prints, per workload, the average milliseconds of each pipeline stage from
in-stream CUDA events (ebz_profile / ebz_stage_times), plus GB/s of input.
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
from tools.synth import CONFIG_SHAPES, make_torch  # noqa: E402

STAGES = ["range", "sweep_compress", "huffman_build", "encode", "decode", "zero_ranks",
          "sweep_decompress"]


def run(name, reps, layers=1, rel=1e-4, seed=None):
    shape = CONFIG_SHAPES[name]
    f = make_torch(name, shape, seed).reshape(-1)
    out = torch.empty_like(f)
    dims = tuple(reversed(shape))
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=rel), layers=layers)
    b = DeviceBatch(nstreams=1)
    ctx = b.ctx
    for _ in range(2):
        b.roundtrip([f], dims, cfg, [out])
    torch.cuda.synchronize()
    ms = (ctypes.c_double * 8)()
    cnt = (ctypes.c_ulonglong * 8)()
    ctx.lib.ebz_stage_times(ctx.handle, ms, cnt, 8)
    ctx.lib.ebz_profile(ctx.handle, 1)
    tc = td = 0.0
    for _ in range(reps):
        e0, e1, e2 = b.roundtrip([f], dims, cfg, [out])
        torch.cuda.synchronize()
        tc += e0.elapsed_time(e1)
        td += e1.elapsed_time(e2)
    ctx.lib.ebz_profile(ctx.handle, 0)
    ctx.lib.ebz_stage_times(ctx.handle, ms, cnt, 8)
    info = b.info(0)
    nbytes = f.numel() * 4
    err = (out.double() - f.double()).abs().max().item()
    res = {"workload": name, "layers": layers, "rel": rel, "n": f.numel(),
           "compress_ms": tc / reps, "decompress_ms": td / reps,
           "compress_gbs": nbytes / (tc / reps / 1e3) / 1e9,
           "decompress_gbs": nbytes / (td / reps / 1e3) / 1e9,
           "K": int(info.n_unpred), "bits": int(info.bit_length), "status": int(info.status),
           "max_err_over_eb": err / info.eb,
           "stages_ms": {STAGES[i]: round(ms[i] / max(1, cnt[i]), 4) for i in range(7)}}
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["cfg5"])
    ap.add_argument("--reps", type=int, default=5)
    ns = ap.parse_args()
    reps = ns.reps
    names = ns.names
    for nm in names:
        if nm == "cfg2":
            for layers in (1, 2):
                for rel in (1e-3, 1e-4, 1e-5):
                    run(nm, reps, layers, rel)
        else:
            run(nm, reps)
