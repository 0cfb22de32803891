"""Pinned host <-> device copy bandwidth on this box (the e2e path's bound).

    python tools/pcie_probe.py [--gb 2]
"""
import argparse
import json
import time

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=2.0)
    a = ap.parse_args()
    n = int(a.gb * 1e9) // 4
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    d2 = torch.empty_like(d)
    h2 = torch.empty_like(h).pin_memory()
    for _ in range(2):
        d.copy_(h, non_blocking=True)
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h2.copy_(d2, non_blocking=True))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        res[name + "_gbs"] = 3 * 4 * n / (time.perf_counter() - t0) / 1e9
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res["duplex_each_gbs"] = 3 * 4 * n / (time.perf_counter() - t0) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
