"""N > 1 host path on CPU: world_size 2 over gloo (127.0.0.1).

Each rank compresses its round-robin shard of a small field batch with the
CPU oracle (standing in for its GPU), the shards together cover every field
exactly once with containers identical to a single-process run, and the
timing reduction is the max over ranks (bench.py's contract)."""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1706_03791_b200.shard import field_shard, reduce_max, reduce_sum

N_FIELDS = 7
DIMS = (12, 9, 5)


def _fields():
    rng = np.random.default_rng(3)
    n = int(np.prod(DIMS))
    return [(np.sin(np.linspace(0, 5 + i, n)) * (i + 1) +
             0.01 * rng.standard_normal(n)).astype(np.float32) for i in range(N_FIELDS)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        fields = _fields()
        mine = field_shard(N_FIELDS, rank, world)
        digests = {i: hashlib.sha256(O.compress_bytes(fields[i], DIMS, relative=1e-3)
                                     ["container"]).hexdigest() for i in mine}
        gathered = [None] * world
        dist.all_gather_object(gathered, digests)
        t_max = reduce_max([10.0 + rank, 5.0 * (world - rank)])
        b_sum = reduce_sum([len(mine)])
        if rank == 0:
            out.put((gathered, t_max, b_sum))
    finally:
        dist.destroy_process_group()


def test_field_shard_round_robin():
    assert field_shard(7, 0, 2) == [0, 2, 4, 6]
    assert field_shard(7, 1, 2) == [1, 3, 5]
    allf = sorted(i for r in range(8) for i in field_shard(64, r, 8))
    assert allf == list(range(64))
    with pytest.raises(ValueError):
        field_shard(4, 2, 2)
    assert reduce_max([1.5, 2.0]) == [1.5, 2.0]   # no group: identity


def test_world2_gloo_shards_and_max_timing():
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, t_max, b_sum = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    merged = {}
    for d in gathered:
        assert not set(d) & set(merged)          # every field exactly once
        merged.update(d)
    assert sorted(merged) == list(range(N_FIELDS))
    fields = _fields()
    for i, f in enumerate(fields):
        want = hashlib.sha256(O.compress_bytes(f, DIMS, relative=1e-3)["container"]).hexdigest()
        assert merged[i] == want
    assert t_max == [11.0, 10.0]                 # max over ranks, element-wise
    assert b_sum == [float(N_FIELDS)]
