"""One batched device round trip of the bench workload (for ncu / timing).

    python tools/batch_probe.py [--nfields 64] [--reps 2]

Generates the bench's cfg5 batch on the device (same seeds as bench.py),
runs `reps` batched compress + decompress passes and prints per-phase ms.
"""

import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1706_03791_b200 as ebz  # noqa: E402
from paper_1706_03791_b200.device import DeviceBatch  # noqa: E402
from tools.stage_times import STAGES  # noqa: E402
from tools.synth import CONFIG_SHAPES, make_torch  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--nfields", type=int, default=64)
    p.add_argument("--reps", type=int, default=2)
    p.add_argument("--layers", type=int, default=1)
    p.add_argument("--stages", action="store_true",
                   help="in-stream stage times (averaged over reps after the first)")
    a = p.parse_args()
    shape = CONFIG_SHAPES["cfg5"]
    dims = tuple(reversed(shape))
    fields = [make_torch("cfg5", shape, s).reshape(-1) for s in range(a.nfields)]
    outs = [torch.empty_like(f) for f in fields]
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-4), layers=a.layers)
    db = DeviceBatch()
    ctx = db.ctx
    ms = (ctypes.c_double * 8)()
    cnt = (ctypes.c_ulonglong * 8)()
    for r in range(a.reps):
        if a.stages and r == 1:
            ctx.lib.ebz_stage_times(ctx.handle, ms, cnt, 8)  # clears
            ctx.lib.ebz_profile(ctx.handle, 1)
        e0, e1, e2 = db.roundtrip(fields, dims, cfg, outs)
        torch.cuda.synchronize()
        tc, td = e0.elapsed_time(e1), e1.elapsed_time(e2)
        gb = sum(f.numel() * 4 for f in fields) / 1e9
        print(f"rep {r}: compress {tc:.2f} ms ({gb / tc * 1e3:.1f} GB/s)  "
              f"decompress {td:.2f} ms ({gb / td * 1e3:.1f} GB/s)", flush=True)
    if a.stages and a.reps > 1:
        ctx.lib.ebz_profile(ctx.handle, 0)
        ctx.lib.ebz_stage_times(ctx.handle, ms, cnt, 8)
        print("stages (ms per launch group): " + ", ".join(
            f"{n} {ms[i] / max(1, cnt[i]):.3f}" for i, n in enumerate(STAGES)), flush=True)


if __name__ == "__main__":
    main()
