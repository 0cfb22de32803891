"""cfg5 -- the headline workload (BASELINE configs[4]: 64 independent 256^3
float32 fields, seeds 0..63, rel eb 1e-4, n = 1, m = 8) -- pinned in full.

* every one of the 64 fields through the public batched API
  (``compress_many`` / ``decompress_many``) equals the CPU oracle byte for
  byte (container) and bit for bit (reconstruction digest);
* the fields sharded round robin over G = 1, 2, 4, 8 ranks (``shard.py``,
  what ``bench.py --gpus G`` runs: each shard one batched device launch)
  give identical containers and reconstructions for every G -- the
  reference's worker-count determinism (tests/test_acceptance.py:333-366);
* the launch-epoch wrap re-zeroes the tagged face buffers: a wrap into an
  epoch whose stale words sit in the same slot stays bit-exact.
"""

import hashlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_1706_03791_b200 as ebz
from paper_1706_03791_b200.device import DeviceBatch
from paper_1706_03791_b200.shard import field_shard
from tools.synth import CONFIG_SHAPES, make_torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SHAPE = CONFIG_SHAPES["cfg5"]
DIMS = tuple(reversed(SHAPE))
NF = 64
CFG = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-4), layers=1, interval_exponent=8)


@pytest.fixture(scope="module")
def fields(gpu):
    return [make_torch("cfg5", SHAPE, s).reshape(-1) for s in range(NF)]


@pytest.fixture(scope="module")
def oracle_out(fields, oracle):
    """(container, recon digest) per field from the oracle, thread-pooled
    (the reference's file-level parallelism); the large arrays are dropped."""
    host = [f.cpu().numpy() for f in fields]

    def one(v):
        r = oracle.compress_bytes(v, DIMS, layers=1, m=8, relative=1e-4)
        return r["container"], r["recon_digest"]

    with ThreadPoolExecutor() as pool:
        return list(pool.map(one, host))


def test_cfg5_all_64_fields_bit_exact(fields, oracle_out):
    grids = [ebz.DataGrid(DIMS, f.cpu().numpy()) for f in fields]
    outs = ebz.compress_many(grids, CFG)
    backs = ebz.decompress_many([o.stream for o in outs])
    for i, (o, b) in enumerate(zip(outs, backs)):
        blob, digest = oracle_out[i]
        assert ebz.serialize(o.stream) == blob, i
        assert hashlib.sha256(b.values.tobytes()).hexdigest() == digest, i


def test_cfg5_shard_count_invariance(fields, oracle_out):
    import torch
    batch = DeviceBatch(nstreams=1)
    outs = [torch.empty_like(f) for f in fields]
    seen = {}
    for G in (1, 2, 4, 8):
        blobs, digests = [None] * NF, [None] * NF
        for rank in range(G):
            idx = field_shard(NF, rank, G)
            mine = [fields[i] for i in idx]
            rec = [outs[i] for i in idx]
            batch.roundtrip(mine, DIMS, CFG, rec)
            torch.cuda.synchronize()
            for j, i in enumerate(idx):
                blobs[i] = batch.container(j)
                st = batch.decode_info(len(idx) + j).status
                assert st == 0, (G, i, st)
                digests[i] = hashlib.sha256(rec[j].cpu().numpy().tobytes()).hexdigest()
        seen[G] = (blobs, digests)
        assert blobs == [b for b, _ in oracle_out], G
        assert digests == [d for _, d in oracle_out], G
    assert seen[1] == seen[2] == seen[4] == seen[8]


def _two_fields(shape, seed):
    a = make_torch("cfg1", shape, seed).reshape(-1)
    b = make_torch("cfg4", shape, seed + 1).reshape(-1)
    return a, b


@pytest.mark.parametrize("shape", [(24, 40, 70), (90, 130), (5, 6, 7, 9)])
def test_epoch_wrap_rezeroes_tagged_buffers(gpu, oracle, shape):
    """Slot S holds face words (or generic progress counters) tagged with
    epoch 1 from field B; the epoch counter is then driven to its maximum
    and wraps back to 1 for field A in the same slot.  Without the wrap's
    re-zeroing, A's consumers would accept B's stale words."""
    import torch
    lib, h = gpu.lib, gpu.handle
    dims = tuple(reversed(shape))
    fa, fb = _two_fields(shape, 7)
    batch = DeviceBatch(nstreams=1)
    slot = 900_000 + len(shape) * 10  # fresh slot: its buffers start zeroed
    emax = lib.ebz_epoch_max()
    old = lib.ebz_debug_set_epoch(h, 0)
    try:
        with gpu.lock:
            batch.compress_async(slot, fb, dims, CFG)          # epoch 1: B's words
            torch.cuda.synchronize()
            lib.ebz_debug_set_epoch(h, emax - 1)
            batch.compress_async(slot, fa, dims, CFG)          # epoch emax
            torch.cuda.synchronize()
            first = batch.container(slot)
            batch.compress_async(slot, fa, dims, CFG)          # wraps to 1
            torch.cuda.synchronize()
            second = batch.container(slot)
            out = torch.empty_like(fa)
            # decompress across the wrap too (its own tagged buffers)
            lib.ebz_debug_set_epoch(h, emax)
            batch.decompress_async(slot, 1, out)
            torch.cuda.synchronize()
    finally:
        lib.ebz_debug_set_epoch(h, max(old, 2))
    ref = oracle.compress_bytes(fa.cpu().numpy(), dims, layers=1, m=8, relative=1e-4)
    assert first == ref["container"]
    assert second == ref["container"]
    assert hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest() == ref["recon_digest"]
