"""Summaries of ncu output for profiles/ (run here, on reports copied back).

    python tools/ncu_summary.py launches LIST.csv STEPS OUT.md
        aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list
        by kernel: launches, total / per-step microseconds, share of the step.
    python tools/ncu_summary.py full REPORT.ncu-rep OUT.md [OUT_TRAFFIC.json NAME=REGEX ...]
        key `--set full` metrics per captured launch (duration, DRAM bytes,
        throughputs, occupancy, registers, IPC); optionally writes the DRAM
        traffic per launch of named kernels (bench.py roofline.traffic).
"""

import collections
import csv
import io
import json
import re
import subprocess
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("<unnamed>::", "")
    return name.strip()


def launches(path, steps, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if not d.get("Metric Name", "").startswith("gpu__time_duration"):
            continue
        k = short(d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", ""))  # ns
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    # torch kernels = synthetic-input generation and host-side parity checks,
    # outside the timed step; ours = libebz200.so
    foreign = re.compile(r"at_cuda_detail|native::|fft|at::|cub::|cutlass|gemm")
    setup = {k: v for k, v in agg.items() if foreign.search(k)}
    agg = {k: v for k, v in agg.items() if k not in setup}
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list summary ({path.split('/')[-1]}, {steps} steps)", "",
             "Per-launch times are cold-cache and serialised (ncu), so the SHARE of the",
             "step is what compares with bench.py, not the absolute time.", "",
             "| kernel | launches | total us | us / step | share |",
             "|---|---:|---:|---:|---:|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {t / 1e3:.1f} | {t / 1e3 / steps:.1f} | "
                     f"{100 * t / tot:.1f}% |")
    lines.append(f"| **all (libebz200)** | {sum(v[0] for v in agg.values())} | {tot / 1e3:.1f} | "
                 f"{tot / 1e3 / steps:.1f} | 100% |")
    lines += ["", f"Not in the timed step (torch: synthetic inputs, parity checks): "
                  f"{sum(v[0] for v in setup.values())} launches, "
                  f"{sum(v[1] for v in setup.values()) / 1e3:.1f} us."]
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = [
    ("gpu__time_duration.sum", "duration_us", 1e-3),
    ("dram__bytes_read.sum", "dram_read_MB", 1e-6),
    ("dram__bytes_write.sum", "dram_write_MB", 1e-6),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct", 1),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_pct", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("sm__inst_executed.avg.per_cycle_active", "ipc", 1),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active_lanes", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__block_size", "block", 1),
]


def full(rep, out, traffic_out=None, named=()):
    if rep.endswith(".csv"):  # an exported `ncu -i REP --page raw --csv`
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    to_base = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9,
               "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    recs = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        rec = {"kernel": short(d.get("Kernel Name", "?"))}
        for m, key, scale in METRICS:
            v = d.get(m, "")
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                rec[key] = None
                continue
            # time -> ns, bytes -> bytes, then the column's own scale
            x *= to_base.get(units.get(m, ""), 1.0)
            rec[key] = x * scale
        recs.append(rec)
    lines = [f"# ncu --set full summary ({rep.split('/')[-1]})", "",
             "| kernel | us | DRAM rd MB | DRAM wr MB | DRAM GB/s | SM % | mem % | occ % | "
             "regs | IPC | lanes |", "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|"]
    for r in recs:
        us = r["duration_us"] or 0
        mb = (r["dram_read_MB"] or 0) + (r["dram_write_MB"] or 0)
        gbs = mb / us * 1e3 if us else 0  # MB/us -> GB/s
        lines.append(
            f"| `{r['kernel'][:60]}` | {us:.1f} | {r['dram_read_MB'] or 0:.1f} | "
            f"{r['dram_write_MB'] or 0:.1f} | {gbs:.0f} | {r['sm_pct'] or 0:.1f} | "
            f"{r['mem_pct'] or 0:.1f} | {r['occupancy_pct'] or 0:.1f} | {r['regs'] or 0:.0f} | "
            f"{r['ipc'] or 0:.2f} | {r['active_lanes'] or 0:.1f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_out:
        traffic = {}
        for spec in named:
            name, rx = spec.split("=", 1)
            hits = [r for r in recs if re.search(rx, r["kernel"])]
            if hits:
                traffic[name] = sum(((h["dram_read_MB"] or 0) + (h["dram_write_MB"] or 0)) * 1e6
                                    for h in hits) / len(hits)
        json.dump(traffic, open(traffic_out, "w"), indent=1)
        print(traffic)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]), sys.argv[4])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None, sys.argv[5:])
