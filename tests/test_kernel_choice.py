"""The 3D n = 1 compress sweep has three kernels that write identical bytes
(one-row 8 x 4 patches with 16-byte face words: shortest ramp; two-row 8 x 8
patches; z-rows 32 x 4 patches: highest throughput).  The dispatch picks by a fitted time model of shape and field
count (csrc/sweep3.cu sweep3_used); EBZ_SWEEP3 = always | never overrides it.
CPU: the choice function.  GPU: every mode equals the oracle."""

import ctypes
import os

import numpy as np
import pytest

from paper_1706_03791_b200 import _native as nat


def _choice(dims, nf, layers=1, compress=1, width=32):
    lib = nat.load_library()
    d = (ctypes.c_uint64 * len(dims))(*dims)
    return lib.ebz_sweep_kernel_choice(width, len(dims), d, layers, nf, compress)


@pytest.fixture
def mode():
    old = os.environ.pop("EBZ_SWEEP3", None)

    def set_mode(v):
        if v is None:
            os.environ.pop("EBZ_SWEEP3", None)
        else:
            os.environ["EBZ_SWEEP3"] = v
    yield set_mode
    set_mode(old)


def test_choice_follows_the_measurements(mode):
    mode(None)
    # lone fields are ramp-bound: two-row kernel (measured 1.33 vs 1.86 ms at 512^3)
    assert _choice((512, 512, 512), 1) == 2
    assert _choice((256, 256, 256), 1) == 5           # shortest ramp: the 16-byte-face one-row kernel
    assert _choice((500, 500, 100), 1) == 5           # cfg3
    assert _choice((256, 256, 256), 1, compress=0) == 1
    assert _choice((256, 64, 1024), 4) == 2
    # batches are throughput-bound: z-rows kernel (cfg5: 4.6 vs 5.6 ms)
    assert _choice((256, 256, 256), 64) == 3
    assert _choice((256, 256, 256), 16) == 3
    assert _choice((512, 512, 512), 4) == 3
    # rows that are not a multiple of 16 cost the two-row kernel twice the time
    assert _choice((500, 500, 100), 8) == 3
    # everything else
    assert _choice((3600, 1800), 1) == 4          # 2D n = 1: the block-speculative kernel
    assert _choice((3600, 1800), 1, layers=2) == 4
    assert _choice((3600, 1800, 4), 1, layers=2) == 1
    assert _choice((256, 256, 256), 64, compress=0) == 1
    assert _choice((256, 256, 256), 64, layers=2) == 1
    assert _choice((254, 256, 256), 64) == 2      # nx % 4 != 0: sweep3c cannot
    assert _choice((32, 32, 32), 1, width=64) == 5    # binary64 3D n = 1: sweep3b
    assert _choice((32, 32, 32), 1, layers=2, width=64) == 0
    assert _choice((3600, 1800), 1, width=64) == 4    # binary64 2D: the block-speculative kernel
    assert _choice((3600, 1800), 1, layers=3, width=64) == 0
    assert _choice((16, 16, 16, 16), 1) == 0
    mode("always")
    assert _choice((512, 512, 512), 1) == 3
    mode("never")
    assert _choice((256, 256, 256), 64) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("force", ["always", "never", None])
def test_both_kernels_equal_the_oracle(gpu, oracle, mode, force):
    import torch
    import paper_1706_03791_b200 as ebz
    from paper_1706_03791_b200.device import DeviceBatch
    mode(force)
    rng = np.random.default_rng(11)
    dev = torch.device("cuda", 0)
    for dims, nf in (((64, 37, 21), 1), ((48, 40, 9), 5), ((132, 33, 6), 2)):
        want = {"always": 3, "never": 2}.get(force)
        got = _choice(dims, nf)
        assert want is None or got == want
        n = int(np.prod(dims))
        fields = []
        for i in range(nf):
            t = np.linspace(0, rng.uniform(3, 40), n)
            v = np.sin(t) * 10 ** rng.uniform(-1, 2) + 0.02 * rng.standard_normal(n)
            v[rng.integers(0, n, n // 50)] += 50.0      # some unpredictable points
            fields.append(v.astype(np.float32))
        cfg = ebz.CompressorConfig(ebz.ErrorBoundSpec(relative=1e-4))
        db = DeviceBatch()
        d_in = [torch.from_numpy(f).to(dev) for f in fields]
        outs = [torch.empty_like(x) for x in d_in]
        with db.ctx.lock:
            db.compress_batch(d_in, dims, cfg)
            db.decompress_batch(outs)
        torch.cuda.synchronize()
        for i, f in enumerate(fields):
            ref = oracle.compress_bytes(f, dims, layers=1, m=8, relative=1e-4)
            assert db.info(i).status == 0
            assert db.container(i) == ref["container"], (force, dims, i)
            assert outs[i].cpu().numpy().tobytes() == \
                oracle.decompress_bytes(ref["container"]).tobytes(), (force, dims, i)
