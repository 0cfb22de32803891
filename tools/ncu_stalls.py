"""Per-instruction warp-stall samples from an ncu source-page export
(`ncu -i REP --page source --csv --print-source sass > src.csv`).

    python tools/ncu_stalls.py src.csv [--kernel REGEX] [--top 40] [--context 6]

For each kernel in the export: total samples, the stall-reason totals, and
the top instructions by samples with their dominant reasons.  With
--context N, the N preceding instructions of each hot spot are printed too
(a stall is charged to the instruction WAITING, so the producer is usually
a few lines up).
"""

import argparse
import csv
import re


def kernels(path):
    cur = None
    for line in open(path):
        if line.startswith('"Kernel Name"'):
            if cur:
                yield cur
            cur = [line]
        elif cur is not None:
            cur.append(line)
    if cur:
        yield cur


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--kernel", default=".")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--context", type=int, default=0)
    a = ap.parse_args()
    for block in kernels(a.csv):
        name = next(csv.reader([block[0]]))[1]
        if not re.search(a.kernel, name):
            continue
        rows = list(csv.reader(block[1:]))
        hdr = rows[0]
        body = [r for r in rows[1:] if len(r) == len(hdr)]
        ia = hdr.index("Warp Stall Sampling (All Samples)")
        isrc = hdr.index("Source")
        reasons = [(i, h) for i, h in enumerate(hdr)
                   if h.startswith("stall_") and "Not Issued" not in h]

        def num(r, i):
            try:
                return int(r[i] or 0)
            except ValueError:
                return 0

        tot = sum(num(r, ia) for r in body) or 1
        print(f"== {name[:110]}\n   samples {tot}")
        agg = sorted(((sum(num(r, i) for r in body), h) for i, h in reasons), reverse=True)
        print("   " + ", ".join(f"{h[6:]} {100 * v / tot:.1f}%" for v, h in agg if v))
        order = sorted(range(len(body)), key=lambda k: -num(body[k], ia))[:a.top]
        for k in order:
            r = body[k]
            s = num(r, ia)
            why = sorted(((num(r, i), h[6:]) for i, h in reasons), reverse=True)[:3]
            whys = " ".join(f"{h}:{v}" for v, h in why if v)
            if a.context:
                for j in range(max(0, k - a.context), k):
                    print(f"         {body[j][0][-5:]} {body[j][isrc].strip()[:90]}")
            print(f"{s:8d} {100 * s / tot:5.2f}% {r[0][-5:]} {r[isrc].strip()[:70]:70s} {whys}")
            if a.context:
                print()


if __name__ == "__main__":
    main()
