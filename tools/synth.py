"""Seeded synthetic stand-ins for the five BASELINE configs.

The paper's ATM / Hurricane / cosmology datasets are not available here, so
every config is a deterministic Gaussian-random-field recipe with the
config's shape and value character.  Two backends produce the same recipe:

* ``backend="numpy"`` -- float64 numpy FFTs, bit-reproducible on any host;
  used for golden fixtures and small parity tests.
* ``backend="torch"`` -- the same recipe with torch FFTs on the GPU (fast for
  512^3 and 64 x 256^3); used by ``bench.py``.  Different RNG stream, so the
  bytes differ from the numpy backend, but both bench arms consume the same
  arrays.

All outputs are float32, C-ordered numpy-style shapes (last axis fastest);
``DataGrid.from_array`` reverses them into scan-order dims.
"""

from __future__ import annotations

import math

import numpy as np

CONFIG_SHAPES = {
    "cfg1": (256, 256),
    "cfg2": (1800, 3600),
    "cfg3": (100, 500, 500),
    "cfg4": (512, 512, 512),
    "cfg5": (256, 256, 256),
}


# ----------------------------------------------------------------- numpy ---

def _np_grf(shape, slope, seed, aniso=None, rng=None):
    rng = rng if rng is not None else np.random.default_rng(seed)
    white = rng.standard_normal(shape)
    spec = np.fft.rfftn(white)
    aniso = aniso or (1.0,) * len(shape)
    k2 = np.zeros(spec.shape)
    for ax, n in enumerate(shape):
        f = np.fft.rfftfreq(n) if ax == len(shape) - 1 else np.fft.fftfreq(n)
        f = f * n * aniso[ax]
        view = [1] * len(shape)
        view[ax] = f.size
        k2 = k2 + (f.reshape(view)) ** 2
    with np.errstate(divide="ignore"):
        amp = np.where(k2 > 0, k2 ** (slope / 4.0), 0.0)   # |k|^(slope/2)
    field = np.fft.irfftn(spec * amp, s=shape, axes=tuple(range(len(shape))))
    field -= field.mean()
    field /= field.std()
    return field, rng


def _np_spiky(shape, seed, frac=0.01, scale=5.0):
    field, rng = _np_grf(shape, -3.0, seed)
    n = field.size
    idx = rng.choice(n, int(frac * n), replace=False)
    flat = field.reshape(-1)
    flat[idx] += rng.laplace(0.0, scale, idx.size)
    return field


def _np_lognormal(shape, seed):
    g, _ = _np_grf(shape, -3.0, seed)
    sigma = 6.0 * math.log(10.0) / (g.max() - g.min())
    return np.exp(sigma * g)


def _np_box_mean(a, w=5):
    from scipy.ndimage import uniform_filter
    return uniform_filter(a, size=w, mode="reflect")


def make_numpy(name: str, shape=None, seed=None) -> np.ndarray:
    """Config recipe at an arbitrary shape (defaults: the config's own)."""
    shape = tuple(shape or CONFIG_SHAPES[name])
    if name == "cfg1":
        out = _np_spiky(shape, 0 if seed is None else seed)
    elif name == "cfg2":
        g, _ = _np_grf(shape, -3.0, 1 if seed is None else seed)
        lat = np.linspace(-math.pi / 2, math.pi / 2, shape[0])
        g = g + 3.0 * np.cos(lat).reshape((-1,) + (1,) * (len(shape) - 1))
        lo, hi = g.min(), g.max()
        out = -50.0 + 100.0 * (g - lo) / (hi - lo)
    elif name == "cfg3":
        g, rng = _np_grf(shape, -3.0, 2 if seed is None else seed,
                         aniso=(4.0,) + (1.0,) * (len(shape) - 1))
        mean = _np_box_mean(g)
        local_std = np.sqrt(np.maximum(_np_box_mean((g - mean) ** 2), 0.0))
        n = g.size
        idx = rng.choice(n, int(0.005 * n), replace=False)
        sign = np.where(rng.random(idx.size) < 0.5, -1.0, 1.0)
        flat = g.reshape(-1)
        flat[idx] += sign * 10.0 * local_std.reshape(-1)[idx]
        out = g
    elif name == "cfg4":
        out = _np_lognormal(shape, 3 if seed is None else seed)
    elif name == "cfg5":
        s = 0 if seed is None else seed
        kind = s % 3
        if kind == 0:
            out, _ = _np_grf(shape, -3.0, s)
        elif kind == 1:
            out = _np_spiky(shape, s)
        else:
            out = _np_lognormal(shape, s)
    else:
        raise KeyError(name)
    return np.ascontiguousarray(out, dtype=np.float32)


# ----------------------------------------------------------------- torch ---

def _t_grf(shape, slope, gen, device, aniso=None):
    import torch
    white = torch.randn(shape, generator=gen, device=device, dtype=torch.float64)
    spec = torch.fft.rfftn(white)
    aniso = aniso or (1.0,) * len(shape)
    k2 = torch.zeros(spec.shape, device=device, dtype=torch.float64)
    for ax, n in enumerate(shape):
        if ax == len(shape) - 1:
            f = torch.fft.rfftfreq(n, device=device, dtype=torch.float64)
        else:
            f = torch.fft.fftfreq(n, device=device, dtype=torch.float64)
        f = f * n * aniso[ax]
        view = [1] * len(shape)
        view[ax] = f.numel()
        k2 = k2 + f.reshape(view) ** 2
    amp = torch.where(k2 > 0, k2.clamp_min(1e-300) ** (slope / 4.0),
                      torch.zeros_like(k2))
    del k2
    field = torch.fft.irfftn(spec * amp, s=shape)
    del spec, amp
    field -= field.mean()
    field /= field.std()
    return field


def make_torch(name: str, shape=None, seed=None, device="cuda"):
    """Same recipes on the GPU; returns a float32 CUDA tensor."""
    import torch
    import torch.nn.functional as F
    shape = tuple(shape or CONFIG_SHAPES[name])
    defaults = {"cfg1": 0, "cfg2": 1, "cfg3": 2, "cfg4": 3, "cfg5": 0}
    s = defaults[name] if seed is None else seed
    gen = torch.Generator(device=device)
    gen.manual_seed(1000003 * s + 17)

    def spiky():
        g = _t_grf(shape, -3.0, gen, device)
        n = g.numel()
        idx = torch.randperm(n, generator=gen, device=device)[: int(0.01 * n)]
        u = torch.rand(idx.numel(), generator=gen, device=device, dtype=torch.float64)
        lap = -5.0 * torch.sign(u - 0.5) * torch.log1p(-2.0 * (u - 0.5).abs())
        g.view(-1)[idx] += lap
        return g

    def lognormal():
        g = _t_grf(shape, -3.0, gen, device)
        sigma = 6.0 * math.log(10.0) / float(g.max() - g.min())
        return torch.exp(sigma * g)

    if name == "cfg1":
        out = spiky()
    elif name == "cfg2":
        g = _t_grf(shape, -3.0, gen, device)
        lat = torch.linspace(-math.pi / 2, math.pi / 2, shape[0], device=device,
                             dtype=torch.float64)
        g = g + 3.0 * torch.cos(lat).reshape((-1,) + (1,) * (len(shape) - 1))
        lo, hi = g.min(), g.max()
        out = -50.0 + 100.0 * (g - lo) / (hi - lo)
    elif name == "cfg3":
        g = _t_grf(shape, -3.0, gen, device, aniso=(4.0,) + (1.0,) * (len(shape) - 1))

        def box(a):
            a5 = F.pad(a[None, None], (2, 2, 2, 2, 2, 2), mode="reflect")
            return F.avg_pool3d(a5, 5, stride=1)[0, 0]
        mean = box(g)
        local_std = box((g - mean) ** 2).clamp_min(0).sqrt()
        n = g.numel()
        idx = torch.randperm(n, generator=gen, device=device)[: int(0.005 * n)]
        sign = torch.where(torch.rand(idx.numel(), generator=gen, device=device) < 0.5,
                           -1.0, 1.0).to(torch.float64)
        g.view(-1)[idx] += sign * 10.0 * local_std.view(-1)[idx]
        out = g
    elif name == "cfg4":
        out = lognormal()
    elif name == "cfg5":
        kind = s % 3
        out = _t_grf(shape, -3.0, gen, device) if kind == 0 else (
            spiky() if kind == 1 else lognormal())
    else:
        raise KeyError(name)
    return out.to(torch.float32).contiguous()


# ------------------------------------------------------ small test fields ---

def mixed_field(rng, n, roughness=0.1):
    """Smooth sine + noise (the shape the reference's own codec tests use)."""
    smooth = np.sin(np.linspace(0, 6.0, n)) * 3.0
    return smooth + roughness * rng.standard_normal(n)
