"""Synthetic inputs of the five BASELINE configs, built on the
GPU where they are large (K3 builders) -- workload setup for bench.py and
the tests, not part of the timed hot path.  Small host-side pieces (seeded
numpy factors, Markov parameters, the PSF cube) follow the recipes in
SURVEY.md 8d exactly; ``oracle/configs.py`` holds the numpy twins used to
check these builders at reduced sizes.
"""

from __future__ import annotations

import numpy as np

from . import _dev
from . import _native as N
from .blocks import build_pattern


def c5_factors(i=4096, j=4096, k=1024, r=64, seed=3):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((i, r)), rng.standard_normal((j, r)), rng.standard_normal((k, r))


def c5_build(i=4096, j=4096, k=1024, r=64, noise=1e-4, seed=3, k_slab=None, out=None):
    """X = [[A0, B0, C0]] + noise * Philox normal(linear C-order index) on device;
    ``k_slab=(k0, k1)`` builds only mode-3 rows k0:k1 (global noise indices)."""
    a0, b0, c0 = (_dev.to_device(f) for f in c5_factors(i, j, k, r, seed))
    k0, k1 = (0, k) if k_slab is None else k_slab
    x = out if out is not None else _dev.empty((i, j, k1 - k0))
    N.call("bt_build_cp_model_f64", _dev.ptr(a0), _dev.ptr(b0), _dev.ptr(c0), i, j, k, r, k0, k1,
           float(noise), 3, _dev.ptr(x), 0, 0, _dev.stream())
    return x


def normal_init(dims, r, seed):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((d, r)) for d in dims]


def c1_blocks(nb=32, ell=32, seed=0):
    x = np.linspace(0.0, 1.0, nb)
    base = np.exp(-((x[:, None] - x[None, :]) ** 2) / (2 * 0.1**2))
    rng = np.random.default_rng(seed)
    out = []
    for kk in range(ell):
        g = rng.standard_normal((nb, nb))
        out.append(base * np.exp(-(kk**2) / 32.0) + 1e-3 * (g + g.T) / 2)
    return np.stack(out)


def c1_matrix(nb=32, ell=32):
    """The assembled 1024^2 symmetric block-Toeplitz matrix (device)."""
    from .blocks import struct_assemble

    pat = build_pattern("toeplitz", ell, ell, nb, nb, block_symmetric=True)
    return pat, struct_assemble(pat, _dev.to_device(c1_blocks(nb, ell)))


def c2_markov(state=400, io=32, count=2047, seed=1):
    from scipy.stats import ortho_group

    rng = np.random.default_rng(seed)
    q = ortho_group.rvs(state, random_state=rng)
    lam = rng.uniform(0.5, 0.98, state) * rng.choice([-1, 1], state)
    a = q @ np.diag(lam) @ q.T
    b = rng.standard_normal((state, io)) / 20
    c = rng.standard_normal((io, state)) / 20
    params = np.empty((count, io, io))
    xk = b.copy()
    for kk in range(count):
        params[kk] = c @ xk
        xk = a @ xk
    return params


def c2_build(params):
    """apps.py:186-201 weighted Hankel tensor on device: (d_out, p, d_in)."""
    s = (params.shape[0] + 1) // 2
    pat = build_pattern("hankel", s, s, params.shape[1], params.shape[2])
    d, _, _ = pat.device()
    pd = _dev.to_device(params)
    t = _dev.empty((params.shape[1], params.shape[0], params.shape[2]))
    N.call("bt_build_hankel_f64", _dev.ptr(pd), params.shape[0], params.shape[1], params.shape[2],
           _dev.ptr(d["eta"]), _dev.ptr(t), _dev.stream())
    return pat, t


def c3_points(side=32):
    g = np.linspace(0.0, 1.0, side)
    return np.array([(g[a], g[b]) for b in range(side) for a in range(side)])


def c3_build(side=32, lags=512, lag_scale=None):
    """Weighted Gneiting space-time tensor (npts, lags, npts) on device."""
    lag_scale = float(lags if lag_scale is None else lag_scale)
    npts = side * side
    pat = build_pattern("toeplitz", lags, lags, npts, npts, block_symmetric=True)
    d, _, _ = pat.device()
    pts = _dev.to_device(c3_points(side))
    t = _dev.empty((npts, lags, npts))
    N.call("bt_build_gneiting_f64", _dev.ptr(pts), npts, lags, lag_scale, _dev.ptr(d["eta"]),
           _dev.ptr(t), _dev.stream())
    return pat, t


def c4_psf(k=255, sig=(2.0, 3.0, 4.0), angle_deg=30.0, mix=0.7):
    h = (k - 1) // 2
    dd = np.arange(-h, h + 1, dtype=np.float64)
    d1, d2, d3 = np.meshgrid(dd, dd, dd, indexing="ij")
    s = [2 * v * v for v in sig]
    ga = np.exp(-(d1**2 / s[0] + d2**2 / s[1] + d3**2 / s[2]))
    th = np.deg2rad(angle_deg)
    c, sn = np.cos(th), np.sin(th)
    e1 = c * d1 + sn * d2
    e2 = -sn * d1 + c * d2
    gr = np.exp(-(e1**2 / s[0] + e2**2 / s[1] + d3**2 / s[2]))
    psf = mix * ga + (1.0 - mix) * gr
    return psf / psf.sum()


def gather_standin(nb=256, ell=128):
    """C1's generator scaled up (SURVEY 8d gather/scatter stand-in)."""
    x = np.linspace(0.0, 1.0, nb)
    base = np.exp(-((x[:, None] - x[None, :]) ** 2) / (2 * 0.1**2))
    rng = np.random.default_rng(0)
    out = []
    for kk in range(ell):
        g = rng.standard_normal((nb, nb))
        out.append(base * np.exp(-(kk**2) / 32.0) + 1e-3 * (g + g.T) / 2)
    pat = build_pattern("toeplitz", ell, ell, nb, nb, block_symmetric=True)
    return pat, np.stack(out)
