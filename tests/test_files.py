"""Multi-file driver against the reference CLI's own
output (tests/golden/files.json, tests/golden/make_golden_files.py).

CPU: raw loading and its error messages, the rank / device assignment, the
CSV / exit-code helper and the world-2 gloo gather of per-rank rows.  GPU:
every reference CLI run replayed through compress_files / decompress_files
on the same bytes -- exit codes, rows (timing columns dropped), error lines
and the SHA-256 of every output file identical."""

import hashlib
import io
import json
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1706_03791_b200 as ebz
from paper_1706_03791_b200 import files as F

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from files_inputs import DIMS, REL, make_inputs  # noqa: E402

DROP = {"compress": (8, 9), "decompress": (2,)}


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(HERE, "golden", "files.json")) as fh:
        return json.load(fh)


def _norm(text, d):
    return text.replace(str(d), "<D>")


def _emitted(results, header, d, kind):
    out, err = io.StringIO(), io.StringIO()
    code = F.emit(results, header, out=out, err=err)
    lines = out.getvalue().splitlines()
    rows = [",".join(c for k, c in enumerate(r.split(",")) if k not in DROP[kind])
            for r in lines[1:]]
    return {"exit": code, "header": lines[0], "rows": [_norm(r, d) for r in rows],
            "errors": [_norm(e, d) for e in err.getvalue().splitlines()]}


def test_load_raw_reference_messages(tmp_path, gold):
    f = make_inputs(tmp_path / "in")
    g = F.load_raw(f["a.raw"], DIMS, 32)
    assert g.dims == DIMS and g.values.dtype == np.float32
    assert F.load_raw(f["wide.raw"], DIMS, 64).values.dtype == np.float64
    errs = gold["runs"][0]["errors"]
    with pytest.raises(ValueError) as e:
        F.load_raw(f["short.raw"], DIMS, 32)
    assert f"error: <D>/in/short.raw: {_norm(str(e.value), tmp_path)}" == errs[0]
    with pytest.raises(ValueError) as e:
        F.load_raw(f["nan.raw"], DIMS, 32)
    assert f"error: <D>/in/nan.raw: {e.value}" == errs[1]
    with pytest.raises(OSError):
        F.load_raw(tmp_path / "missing.raw", DIMS, 32)


def test_assignment_round_robin():
    assert F._assignment(7, [0, 1]) == [(0, [0, 2, 4, 6]), (1, [1, 3, 5])]
    assert F._assignment(7, None) == [(None, list(range(7)))]
    # two ranks x two devices: rank 1 owns 1, 3, 5 -> devices alternate
    assert F._assignment(7, [2, 3], rank=1, world=2) == [(2, [1, 5]), (3, [3])]
    every = sorted(i for r in range(3) for _, idx in F._assignment(11, [0, 1], r, 3)
                   for i in idx)
    assert every == list(range(11))


def test_emit_and_exit_code(tmp_path):
    ok = F.FileResult(0, Path("x.raw"), True, "x.raw,1,2")
    bad = F.FileResult(1, Path("y.raw"), False, "boom")
    out, err = io.StringIO(), io.StringIO()
    csv = tmp_path / "s.csv"
    assert F.emit([ok, bad], "h", csv_path=csv, out=out, err=err) == 1
    assert out.getvalue() == "h\nx.raw,1,2\n"
    assert err.getvalue() == "error: y.raw: boom\n"
    assert csv.read_text() == "h\nx.raw,1,2\n"
    assert F.emit([ok], "h", out=io.StringIO(), err=io.StringIO()) == 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # each rank's own share of 9 files (as compress_files would return it)
        mine = [i for _, idx in F._assignment(9, None) for i in idx]
        assert mine == list(range(rank, 9, world))
        local = [F.FileResult(i, Path(f"f{i}.raw"), i % 4 != 3, f"row{i}") for i in mine]
        merged = F.gather_results(local)
        if rank == 0:
            out.put([(r.index, str(r.path), r.ok, r.payload) for r in merged])
    finally:
        dist.destroy_process_group()


def test_gather_results_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == [(i, f"f{i}.raw", i % 4 != 3, f"row{i}") for i in range(9)]


@pytest.mark.gpu
def test_gpu_files_match_reference_cli(tmp_path, gold, gpu):
    _replay(tmp_path, gold, None)


@pytest.mark.gpu
def test_gpu_files_two_host_threads_one_device(tmp_path, gold, gpu):
    """devices=[0, 0]: the files go round robin to two host threads that share
    device 0 (the per-device kernel-attribute records and the context lock
    under concurrent callers); rows, errors and output bytes unchanged."""
    _replay(tmp_path, gold, [0, 0])


@pytest.mark.gpu
def test_gpu_files_two_devices(tmp_path, gold, gpu):
    """devices=[0, 1] (cli.py:100-113 over two GPUs, one host thread each):
    the second device gets its own kernel shared-memory limits."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    _replay(tmp_path, gold, [0, 1])


def _replay(tmp_path, gold, devices):
    kw = {"devices": devices} if devices else {}
    d = tmp_path
    f = make_inputs(d / "in")
    o = d / "out"
    runs = gold["runs"]
    cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=REL))
    names = ["a.raw", "b.raw", "short.raw", "nan.raw"]
    # group=1 and 2 exercise per-group pipelines and the per-file fallback
    got = _emitted(F.compress_files([f[n] for n in names], DIMS, 32, cfg, out_dir=o, group=2,
                                    **kw),
                   F.COMPRESS_COLUMNS, d, "compress")
    assert got == {k: runs[0][k] for k in got}
    got = _emitted(F.compress_files([f["noisy.raw"]], DIMS, 32, cfg, out_dir=o / "plain", **kw),
                   F.COMPRESS_COLUMNS, d, "compress")
    assert got == {k: runs[1][k] for k in got}
    got = _emitted(F.compress_files([f["noisy.raw"]], DIMS, 32, cfg, out_dir=o / "auto",
                                    auto_m=True, **kw), F.COMPRESS_COLUMNS, d, "compress")
    assert got == {k: runs[2][k] for k in got}
    wcfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(absolute=1e-3), layers=2)
    got = _emitted(F.compress_files([f["wide.raw"]], DIMS, 64, wcfg, out_dir=o / "wide", **kw),
                   F.COMPRESS_COLUMNS, d, "compress")
    assert got == {k: runs[3][k] for k in got}
    bad = o / "bad.ebz"
    bad.write_bytes((o / "a.raw.ebz").read_bytes()[:100])
    got = _emitted(F.decompress_files([o / "a.raw.ebz", bad, o / "b.raw.ebz",
                                       o / "wide" / "wide.raw.ebz"], out_dir=o / "dec",
                                      group=1, **kw), F.DECOMPRESS_COLUMNS, d, "decompress")
    assert got == {k: runs[4][k] for k in got}
    outputs = {_norm(str(p), d): hashlib.sha256(p.read_bytes()).hexdigest()
               for p in sorted(o.rglob("*")) if p.is_file() and p.name != "bad.ebz"}
    assert outputs == gold["outputs"]
