"""Golden fixtures for the multi-file driver, produced by
running the REFERENCE CLI itself (build container only):

    python tests/golden/make_golden_files.py

Runs ``ebzip.cli.main`` compress / decompress on the raw files of
files_inputs.make_inputs and records, per run, the exit code, the CSV rows
without their timing columns, the stderr error lines and the SHA-256 of every
output file, with the temporary directory replaced by ``<D>``.  Output:
files.json.
"""

from __future__ import annotations

import contextlib
import hashlib
import io
import json
import os
import sys
import tempfile
from pathlib import Path

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from files_inputs import DIMS, REL, make_inputs  # noqa: E402

# timing columns dropped from the rows: compress seconds, mb_per_s; decompress seconds
DROP = {"compress": (8, 9), "decompress": (2,)}


def norm(text, d):
    return text.replace(str(d), "<D>")


def run(cli, argv, d, kind):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = cli.main(argv)
    lines = out.getvalue().splitlines()
    rows = [",".join(c for k, c in enumerate(r.split(",")) if k not in DROP[kind])
            for r in lines[1:]]
    return {"argv": [norm(a, d) for a in argv], "exit": code, "header": lines[0],
            "rows": [norm(r, d) for r in rows],
            "errors": [norm(e, d) for e in err.getvalue().splitlines()]}


def sha(p):
    return hashlib.sha256(Path(p).read_bytes()).hexdigest()


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    from ebzip import cli  # the reference

    dims = ",".join(str(v) for v in DIMS)
    runs = []
    with tempfile.TemporaryDirectory() as tmp:
        d = Path(tmp)
        f = make_inputs(d / "in")
        o = d / "out"
        names = ["a.raw", "b.raw", "short.raw", "nan.raw"]
        runs.append(run(cli, ["compress", *[str(f[n]) for n in names], "--rel-bound", str(REL),
                              "--dims", dims, "--out", str(o)], d, "compress"))
        runs.append(run(cli, ["compress", str(f["noisy.raw"]), "--rel-bound", str(REL),
                              "--dims", dims, "--out", str(o / "plain")], d, "compress"))
        runs.append(run(cli, ["compress", str(f["noisy.raw"]), "--rel-bound", str(REL),
                              "--dims", dims, "--auto-m", "--out", str(o / "auto")], d,
                        "compress"))
        runs.append(run(cli, ["compress", str(f["wide.raw"]), "--abs-bound", "1e-3",
                              "--layers", "2", "--dims", dims, "--width", "64",
                              "--out", str(o / "wide")], d, "compress"))
        bad = o / "bad.ebz"
        bad.write_bytes((o / "a.raw.ebz").read_bytes()[:100])
        runs.append(run(cli, ["decompress", str(o / "a.raw.ebz"), str(bad),
                              str(o / "b.raw.ebz"), str(o / "wide" / "wide.raw.ebz"),
                              "--out", str(o / "dec")], d, "decompress"))
        outputs = {norm(str(p), d): sha(p) for p in sorted(o.rglob("*")) if p.is_file()
                   and p.name != "bad.ebz"}
    with open(os.path.join(HERE, "files.json"), "w") as fh:
        json.dump({"dims": list(DIMS), "rel": REL, "runs": runs, "outputs": outputs}, fh,
                  indent=1)
    print(json.dumps(runs, indent=1))


if __name__ == "__main__":
    main()
