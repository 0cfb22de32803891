"""Multi-file driver over the B200 path.

The reference compresses many raw files by mapping one job per file over a
thread pool (``ebzip/cli.py:100-113``; jobs ``:131-212``): load the headerless
little-endian raw grid, compress (with the ``--auto-m`` loop), serialize,
write ``<name>.ebz``; or read, deserialize, decompress and write
``<name>.dec``.  Results keep input order, one CSV row per successful file,
and a failing file (``OSError`` / ``ValueError`` / ``ContainerError``) is
reported without stopping the others; the exit code is 1 when any failed.

This module keeps those semantics and rows but runs the jobs through the
batched device pipelines: files are assigned round robin to the listed GPUs
(file i -> device i mod G, one host thread per device; the ctypes calls
release the GIL), host reads / writes overlap the device work, and each
device processes its valid grids ``group`` at a time with ``compress_many`` /
``decompress_many`` (pinned arenas, overlapped copies).  A group that raises
is re-run file by file so the failure stays with its file.  Under
``torch.distributed`` (one process per GPU) each rank takes the files
``field_shard(len(paths), rank, world)`` and ``gather_results`` collects the
rows on every rank in input order -- no data-path collective.

Per-file ``seconds`` / ``mb_per_s``: a batched file's share of its group's
wall time, in proportion to its raw bytes (the reference times each file on
its own thread).
"""

from __future__ import annotations

import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, replace
from pathlib import Path

import numpy as np

from . import codec
from .batch import compress_many, decompress_many
from .core import ContainerError, DataGrid, deserialize, serialize
from .metrics import bit_rate, compression_factor
from .shard import field_shard

COMPRESSED_SUFFIX = ".ebz"
DECOMPRESSED_SUFFIX = ".dec"
MAX_EXPONENT = codec.MAX_INTERVAL_EXPONENT
COMPRESS_COLUMNS = (
    "file,values,layers,exponent,bound,factor,bit_rate,hitting_rate,"
    "seconds,mb_per_s,output,note"
)
DECOMPRESS_COLUMNS = "file,values,seconds,output"
_JOB_ERRORS = (OSError, ValueError, ContainerError)


@dataclass(frozen=True)
class FileResult:
    """One file's outcome: ``payload`` is the CSV row when ``ok``, else the
    error message (the reference's ``(path, ok, payload)`` triple)."""
    index: int
    path: Path
    ok: bool
    payload: str


def raw_dtype(width: int) -> np.dtype:
    return np.dtype("<f4" if width == 32 else "<f8")


def load_raw(path, dims, width: int) -> DataGrid:
    """Headerless raw grid in scan order (cli.py:69-76, same message)."""
    path = Path(path)
    data = np.fromfile(path, dtype=raw_dtype(width))
    expected = int(np.prod(dims))
    if data.size != expected:
        raise ValueError(f"{path}: holds {data.size} values, dims {tuple(dims)} need {expected}")
    return DataGrid(tuple(dims), data)


def out_path(path: Path, out_dir, name: str) -> Path:
    """Output next to the input or under ``out_dir`` (cli.py:116-120)."""
    directory = Path(out_dir) if out_dir else path.parent
    directory.mkdir(parents=True, exist_ok=True)
    return directory / name


def _assignment(n: int, devices, rank=None, world=None):
    """[(device, [file indices])]: this rank's share, round robin over devices."""
    if world is None:
        try:
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                rank, world = dist.get_rank(), dist.get_world_size()
        except ImportError:
            pass
    mine = field_shard(n, rank or 0, world or 1)
    devices = list(devices) if devices else [None]
    return [(d, mine[k::len(devices)]) for k, d in enumerate(devices)]


def _prefetched(io, fn, idx, size):
    """Chunks of `size` (index, future) pairs; the next chunk's reads are
    submitted before the current one is handed out (one group of read-ahead,
    so host memory holds at most two groups of inputs)."""
    chunks = [idx[i:i + size] for i in range(0, len(idx), size)]
    nxt = [(i, io.submit(fn, i)) for i in chunks[0]] if chunks else []
    for c in range(len(chunks)):
        cur = nxt
        nxt = [(i, io.submit(fn, i)) for i in chunks[c + 1]] if c + 1 < len(chunks) else []
        yield cur


def _compress_row(path, grid, cfg, outcome, payload_len, elapsed, target, note):
    raw_bytes = grid.n_values * grid.element_width // 8
    return ",".join((
        str(path), str(grid.n_values), str(cfg.layers), str(cfg.interval_exponent),
        format(outcome.stream.eb_effective, ".6g"),
        format(compression_factor(raw_bytes, payload_len), ".6g"),
        format(bit_rate(payload_len, grid.n_values), ".6g"),
        format(outcome.hitting_rate, ".6g"),
        format(elapsed, ".6g"),
        format(raw_bytes / 1e6 / elapsed if elapsed > 0 else 0.0, ".6g"),
        str(target), note))


def compress_files(paths, dims, width, config, *, out_dir=None, auto_m=False, devices=None,
                   group: int = 16, rank=None, world=None) -> list[FileResult]:
    """Compress raw files to ``.ebz`` (cli.py:131-188 job semantics); returns
    this rank's results in input order."""
    paths = [Path(p) for p in paths]
    dims = tuple(int(v) for v in dims)
    results: dict[int, FileResult] = {}
    lock = threading.Lock()

    def put(i, ok, payload):
        with lock:
            results[i] = FileResult(i, paths[i], ok, payload)

    def finish(i, grid, outcome, elapsed):
        # the --auto-m loop (cli.py:146-154) and the warning note
        cfg, note = config, ""
        if auto_m:
            while outcome.warning and cfg.interval_exponent < MAX_EXPONENT:
                cfg = replace(cfg, interval_exponent=outcome.warning.suggested_exponent)
                t0 = time.perf_counter()
                outcome = codec.compress(grid, cfg, device=dev_of[i])
                elapsed += time.perf_counter() - t0
            if cfg.interval_exponent != config.interval_exponent:
                note = f"raised exponent to {cfg.interval_exponent}"
        if outcome.warning:
            w = outcome.warning
            note = (f"hitting rate {w.hitting_rate:.3f} < {w.threshold:.3f}; "
                    f"consider exponent {w.suggested_exponent}")
        t0 = time.perf_counter()
        payload = serialize(outcome.stream)
        target = out_path(paths[i], out_dir, paths[i].name + COMPRESSED_SUFFIX)
        target.write_bytes(payload)
        elapsed += time.perf_counter() - t0
        put(i, True, _compress_row(paths[i], grid, cfg, outcome, len(payload), elapsed,
                                   target, note))

    dev_of = {}

    def device_worker(dev, idx):
        for i in idx:
            dev_of[i] = dev
        with ThreadPoolExecutor(max_workers=4) as io:
            for chunk in _prefetched(io, lambda i: load_raw(paths[i], dims, width), idx,
                                     max(1, group)):
                grids = []
                for i, fut in chunk:
                    try:
                        grids.append((i, fut.result()))
                    except _JOB_ERRORS as exc:
                        put(i, False, str(exc))
                if not grids:
                    continue
                t0 = time.perf_counter()
                try:
                    outs = compress_many([g for _, g in grids], config, group=group, device=dev)
                    wall = time.perf_counter() - t0
                    total = sum(g.n_values * g.element_width for _, g in grids) or 1
                    shares = [wall * g.n_values * g.element_width / total for _, g in grids]
                except _JOB_ERRORS:
                    outs, shares = [], []
                    for i, g in grids:  # isolate the failing file(s)
                        t1 = time.perf_counter()
                        try:
                            outs.append(codec.compress(g, config, device=dev))
                        except _JOB_ERRORS as exc:
                            outs.append(exc)
                        shares.append(time.perf_counter() - t1)
                done = []
                for (i, g), out, share in zip(grids, outs, shares):
                    if isinstance(out, Exception):
                        put(i, False, str(out))
                        continue
                    done.append(io.submit(_guard, put, i, finish, i, g, out, share))
                for f in done:
                    f.result()

    _run_devices(_assignment(len(paths), devices, rank, world), device_worker)
    return [results[i] for i in sorted(results)]


def decompress_files(paths, *, out_dir=None, devices=None, group: int = 16, rank=None,
                     world=None) -> list[FileResult]:
    """Decompress ``.ebz`` files to raw ``.dec`` files (cli.py:191-212 job
    semantics); returns this rank's results in input order."""
    paths = [Path(p) for p in paths]
    results: dict[int, FileResult] = {}
    lock = threading.Lock()

    def put(i, ok, payload):
        with lock:
            results[i] = FileResult(i, paths[i], ok, payload)

    def read(i):
        return deserialize(paths[i].read_bytes())

    def finish(i, grid, elapsed):
        name = paths[i].name
        if name.endswith(COMPRESSED_SUFFIX):
            name = name[:-len(COMPRESSED_SUFFIX)]
        t0 = time.perf_counter()
        target = out_path(paths[i], out_dir, name + DECOMPRESSED_SUFFIX)
        grid.values.astype(raw_dtype(grid.element_width), copy=False).tofile(target)
        elapsed += time.perf_counter() - t0
        put(i, True, ",".join((str(paths[i]), str(grid.n_values), format(elapsed, ".6g"),
                               str(target))))

    def device_worker(dev, idx):
        with ThreadPoolExecutor(max_workers=4) as io:
            for chunk in _prefetched(io, read, idx, max(1, group)):
                streams = []
                for i, fut in chunk:
                    try:
                        streams.append((i, fut.result()))
                    except _JOB_ERRORS as exc:
                        put(i, False, str(exc))
                if not streams:
                    continue
                t0 = time.perf_counter()
                try:
                    grids = decompress_many([s for _, s in streams], group=group, device=dev)
                    wall = time.perf_counter() - t0
                    total = sum(s.n_points * s.element_width for _, s in streams) or 1
                    shares = [wall * s.n_points * s.element_width / total for _, s in streams]
                except _JOB_ERRORS:
                    grids, shares = [], []
                    for i, s in streams:
                        t1 = time.perf_counter()
                        try:
                            grids.append(codec.decompress(s, device=dev))
                        except _JOB_ERRORS as exc:
                            grids.append(exc)
                        shares.append(time.perf_counter() - t1)
                done = []
                for (i, _), g, share in zip(streams, grids, shares):
                    if isinstance(g, Exception):
                        put(i, False, str(g))
                        continue
                    done.append(io.submit(_guard, put, i, finish, i, g, share))
                for f in done:
                    f.result()

    _run_devices(_assignment(len(paths), devices, rank, world), device_worker)
    return [results[i] for i in sorted(results)]


def _guard(put, i, fn, *args):
    try:
        fn(*args)
    except _JOB_ERRORS as exc:
        put(i, False, str(exc))


def _run_devices(assignment, worker):
    assignment = [(d, idx) for d, idx in assignment if idx]
    if len(assignment) <= 1:
        for d, idx in assignment:
            worker(d, idx)
        return
    with ThreadPoolExecutor(max_workers=len(assignment)) as pool:
        for f in [pool.submit(worker, d, idx) for d, idx in assignment]:
            f.result()


def gather_results(results: list[FileResult]) -> list[FileResult]:
    """All ranks' results in input order (identity without a process group)."""
    try:
        import torch.distributed as dist
    except ImportError:
        return list(results)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(results)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, [(r.index, str(r.path), r.ok, r.payload) for r in results])
    merged = sorted((t for p in parts for t in p), key=lambda t: t[0])
    return [FileResult(i, Path(p), ok, payload) for i, p, ok, payload in merged]


def emit(results: list[FileResult], header: str, csv_path=None, out=None, err=None) -> int:
    """Print the CSV (and write ``csv_path``), report failures on stderr;
    returns the reference's exit code (cli.py:123-128,183-188)."""
    out = out or sys.stdout
    err = err or sys.stderr
    rows = [r.payload for r in results if r.ok]
    print(header, file=out)
    for row in rows:
        print(row, file=out)
    if csv_path:
        Path(csv_path).write_text(header + "\n" + "".join(r + "\n" for r in rows))
    failed = [r for r in results if not r.ok]
    for r in failed:
        print(f"error: {r.path}: {r.payload}", file=err)
    return 1 if failed else 0
