"""Seeded synthetic scalar fields -- the inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no order, gradient or diagram): it only
draws fields.  Every recipe is pinned (numpy PCG64 ``default_rng(seed)``, float64
arithmetic, cast to float32, returned as a C-order array of shape [Lz, Ly, Lx] /
[Ly, Lx] / [Lx], i.e. x fastest -- S:87).  The five BASELINE.json configs stand in for
the paper's public volumes, which are not available (DESIGN.md
"Inputs"):

  c1  32^3   i.i.d. U[0,1) float32                                      (random extreme)
  c2  128^3  32 isotropic Gaussians, centres U[0,128)^3, sigma U[4,16],
             amplitude +-U[0.5,1] (sign p=1/2), + U[0,1e-3) noise
  c3  256^3  i.i.d. U[0,1) float32                                      (worst case)
  c4  512^3  5-octave value noise, base period 64 voxels, gain 0.5,
             lattice U[-1,1), smoothstep trilinear, + N(0, 1e-2)
  c5a 8192^2 fBm, Hurst 0.7, spectral synthesis |k|^-(H+1), unit variance
  c5b 2^27   random walk, cumsum of N(0,1) steps in float64
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    "c1": dict(kind="uniform", shape=(32, 32, 32)),
    "c2": dict(kind="gaussians", shape=(128, 128, 128), n=32),
    "c3": dict(kind="uniform", shape=(256, 256, 256)),
    "c4": dict(kind="value_noise", shape=(512, 512, 512), period=64, octaves=5, gain=0.5, noise=1e-2),
    "c5a": dict(kind="fbm2d", shape=(8192, 8192), hurst=0.7),
    "c5b": dict(kind="random_walk", shape=(1 << 27,)),
}


def uniform(shape, seed=0):
    rng = np.random.default_rng(seed)
    return rng.random(size=tuple(shape), dtype=np.float32)


def gaussians(shape, n=32, seed=0, sigma=(4.0, 16.0), amp=(0.5, 1.0), noise=1e-3):
    """Sum of n isotropic Gaussians a*exp(-|p-c|^2 / (2 sigma^2)) + U[0, noise)."""
    rng = np.random.default_rng(seed)
    shape = tuple(shape)
    d = len(shape)
    out = np.zeros(shape, dtype=np.float64)
    axes = [np.arange(s, dtype=np.float64) for s in shape]  # numpy axis order (z, y, x)
    for _ in range(n):
        c = rng.random(d) * np.array(shape, dtype=np.float64)
        s = rng.uniform(*sigma)
        a = rng.uniform(*amp) * (1.0 if rng.random() < 0.5 else -1.0)
        g = None
        for ax in range(d):
            one = np.exp(-((axes[ax] - c[ax]) ** 2) / (2.0 * s * s))
            sh = [1] * d
            sh[ax] = shape[ax]
            one = one.reshape(sh)
            g = one if g is None else g * one
        out += a * g
    out += rng.random(size=shape) * noise
    return out.astype(np.float32)


def _smoothstep(t):
    return t * t * (3.0 - 2.0 * t)


def _interp_axis(G, n, period, axis):
    """Smoothstep-weighted linear interpolation of lattice values G along `axis` onto
    n grid points, lattice spacing `period` voxels."""
    p = np.arange(n, dtype=np.float64) / period
    c = np.floor(p).astype(np.int64)
    w = _smoothstep(p - c)
    a = np.take(G, c, axis=axis)
    b = np.take(G, c + 1, axis=axis)
    sh = [1] * G.ndim
    sh[axis] = n
    w = w.reshape(sh)
    return a * (1.0 - w) + b * w


def value_noise(shape, seed=0, period=64, octaves=5, gain=0.5, noise=1e-2, slab=32):
    """sum_k gain^k VN_k + N(0, noise); VN_k has lattice period period/2^k, lattice
    values U[-1,1), smoothstep trilinear interpolation (separable)."""
    rng = np.random.default_rng(seed)
    shape = tuple(shape)
    d = len(shape)
    out = np.zeros(shape, dtype=np.float64)
    for k in range(octaves):
        P = period / (2 ** k)
        gsz = [int(np.floor((s - 1) / P)) + 2 for s in shape]
        G = rng.uniform(-1.0, 1.0, size=gsz)
        # interpolate the fastest axes first, the slowest axis slab by slab
        B = G
        for ax in range(d - 1, 0, -1):
            B = _interp_axis(B, shape[ax], P, ax)
        p = np.arange(shape[0], dtype=np.float64) / P
        c = np.floor(p).astype(np.int64)
        w = _smoothstep(p - c)
        amp = gain ** k
        for z0 in range(0, shape[0], slab):
            z1 = min(shape[0], z0 + slab)
            wz = w[z0:z1].reshape((-1,) + (1,) * (d - 1))
            out[z0:z1] += amp * (B[c[z0:z1]] * (1.0 - wz) + B[c[z0:z1] + 1] * wz)
    for z0 in range(0, shape[0], slab):
        z1 = min(shape[0], z0 + slab)
        out[z0:z1] += rng.standard_normal(size=(z1 - z0,) + shape[1:]) * noise
    return out.astype(np.float32)


def fbm2d(shape, hurst=0.7, seed=0):
    """Fractional Brownian surface by spectral synthesis: white N(0,1) noise filtered
    by |k|^-(H+1), DC removed, normalised to unit variance."""
    rng = np.random.default_rng(seed)
    ny, nx = shape
    w = rng.standard_normal(size=(ny, nx))
    W = np.fft.rfft2(w)
    ky = np.fft.fftfreq(ny)[:, None]
    kx = np.fft.rfftfreq(nx)[None, :]
    k = np.sqrt(kx * kx + ky * ky)
    k[0, 0] = 1.0
    filt = k ** (-(hurst + 1.0))
    filt[0, 0] = 0.0
    W *= filt
    del w
    out = np.fft.irfft2(W, s=(ny, nx))
    out /= out.std()
    return out.astype(np.float32)


def random_walk(n, seed=0):
    rng = np.random.default_rng(seed)
    return np.cumsum(rng.standard_normal(size=int(n))).astype(np.float32)


def make(name, seed=0, shape=None):
    """Field of BASELINE config `name` ("c1".."c5b"); `shape` overrides the size (for
    small parity cases of the same recipe)."""
    cfg = dict(CONFIGS[name])
    kind = cfg.pop("kind")
    shp = tuple(shape) if shape is not None else cfg.pop("shape")
    cfg.pop("shape", None)
    if kind == "uniform":
        return uniform(shp, seed)
    if kind == "gaussians":
        return gaussians(shp, n=cfg["n"], seed=seed)
    if kind == "value_noise":
        return value_noise(shp, seed=seed, period=cfg["period"] * min(shp) / 512.0 if shape is not None else cfg["period"],
                           octaves=cfg["octaves"], gain=cfg["gain"], noise=cfg["noise"])
    if kind == "fbm2d":
        return fbm2d(shp, hurst=cfg["hurst"], seed=seed)
    if kind == "random_walk":
        return random_walk(shp[0], seed)
    raise KeyError(name)
