"""Per-CUDA-source-line instruction counts and stall samples of one kernel
from an ncu report (--import-source, -lineinfo builds):

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [POINTS] [TOP]

POINTS (default 64 * 256^3) normalises warp-instructions to thread-
instructions per point (x 32 / POINTS)."""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
pts = float(sys.argv[3]) if len(sys.argv) > 3 else 64 * 256 ** 3
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + rx], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
recs, fname = [], None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] and r[0].isdigit() and len(r) > 7:
        try:
            recs.append((fname, int(r[0]), r[1][:88], int(r[7] or 0), int(r[4] or 0)))
        except ValueError:
            pass
tot = sum(x[3] for x in recs)
ts = sum(x[4] for x in recs) or 1
print(f"thread-instructions per point: {32 * tot / pts:.1f}")
for f, ln, src, ins, smp in sorted(recs, key=lambda x: -x[3])[:top]:
    print(f"{f}:{ln:<5d} {32 * ins / pts:6.2f}  {100 * smp / ts:5.1f}%  {src}")
