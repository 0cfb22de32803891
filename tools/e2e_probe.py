"""Host-to-host batched API timing (compress_many / decompress_many).

    python tools/e2e_probe.py [--nfields 64] [--reps 3] [--profile]
"""

import argparse
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1706_03791_b200 as ebz  # noqa: E402
from tools.synth import CONFIG_SHAPES, make_torch  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--nfields", type=int, default=64)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--group", type=int, default=None)
    p.add_argument("--profile", action="store_true")
    a = p.parse_args()
    shape = CONFIG_SHAPES["cfg5"]
    dims = tuple(reversed(shape))
    host = []
    for s in range(a.nfields):
        f = make_torch("cfg5", shape, s).reshape(-1)
        h = torch.empty(f.numel(), dtype=torch.float32, pin_memory=True)
        h.copy_(f)
        host.append(ebz.DataGrid(dims, h.numpy()))
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-4))
    gb = sum(g.values.nbytes for g in host) / 1e9
    for r in range(a.reps):
        t0 = time.perf_counter()
        outs = ebz.compress_many(host, cfg, group=a.group)
        t1 = time.perf_counter()
        recs = ebz.decompress_many([o.stream for o in outs], group=a.group)
        t2 = time.perf_counter()
        print(f"rep {r}: compress_many {1e3 * (t1 - t0):.1f} ms ({gb / (t1 - t0):.1f} GB/s)  "
              f"decompress_many {1e3 * (t2 - t1):.1f} ms ({gb / (t2 - t1):.1f} GB/s)  "
              f"round trip {gb / (t2 - t0):.2f} GB/s", flush=True)
        del outs, recs
    if a.profile:
        pr = cProfile.Profile()
        pr.enable()
        outs = ebz.compress_many(host, cfg, group=a.group)
        recs = ebz.decompress_many([o.stream for o in outs], group=a.group)
        pr.disable()
        pstats.Stats(pr).sort_stats("cumulative").print_stats(18)


if __name__ == "__main__":
    main()
