"""Seeded synthetic inputs for the five BASELINE configs --
numpy generators, TEST/BENCH INFRASTRUCTURE ONLY.

Every generator takes its size parameters so the same recipe serves the
full-size bench workload (built on the GPU by the product's K3 builders,
see ``paper_2105_01170_b200/configs.py``) and the reduced sizes the parity
tests compare at.  The recipes are exactly SURVEY.md section 8d; RHS seeds
``1000 + config#`` are builder choices (flagged there).
"""

from __future__ import annotations

import numpy as np

from .port import assemble, gather, make_pattern, psf_weighted


# ---------------------------------------------------------------------------
# C1 symmetric block Toeplitz 1024^2 -> 32^3, CP R=8 x 50
# ---------------------------------------------------------------------------


def c1_blocks(nb=32, ell=32, seed=0):
    x = np.linspace(0.0, 1.0, nb)
    base = np.exp(-((x[:, None] - x[None, :]) ** 2) / (2 * 0.1**2))
    rng = np.random.default_rng(seed)
    blocks = []
    for k in range(ell):
        g = rng.standard_normal((nb, nb))
        blocks.append(base * np.exp(-(k**2) / 32.0) + 1e-3 * (g + g.T) / 2)
    return np.stack(blocks)


def c1_inputs(nb=32, ell=32):
    pat = make_pattern("toeplitz", ell, ell, nb, nb, block_symmetric=True)
    a = assemble(pat, c1_blocks(nb, ell))
    return pat, a


def normal_init(dims, r, seed):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((d, r)) for d in dims]


# ---------------------------------------------------------------------------
# C2 ERA block Hankel (32, 2047, 32), Tucker (32, 400, 32)
# ---------------------------------------------------------------------------


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
    for k in range(count):          # apps.py:105-114
        params[k] = c @ xk
        xk = a @ xk
    return params


def c2_tensor(params):
    """apps.py:186-201: lateral slices sqrt(eta_k) h_k of the block Hankel."""
    s = (params.shape[0] + 1) // 2
    pat = make_pattern("hankel", s, s, params.shape[1], params.shape[2])
    w = np.sqrt(np.asarray(pat.counts, dtype=np.float64))
    t = np.transpose(params, (1, 0, 2)).copy()
    t *= w[None, :, None]
    return pat, t


# ---------------------------------------------------------------------------
# C3 space-time Gneiting covariance (1024, 512, 1024)
# ---------------------------------------------------------------------------


def c3_points(side=32):
    g = np.linspace(0.0, 1.0, side)
    return np.array([(g[a], g[b]) for b in range(side) for a in range(side)])


def c3_blocks(side=32, lags=512, lag_scale=None):
    from scipy.spatial.distance import cdist

    lag_scale = lags if lag_scale is None else lag_scale
    h = cdist(c3_points(side), c3_points(side))
    out = np.empty((lags, side * side, side * side))
    for k in range(lags):
        u = k / lag_scale
        out[k] = np.exp(-10.0 * h / (u + 1.0) ** 0.25) / (u + 1.0)
    return out


def c3_tensor(side=32, lags=512, lag_scale=None):
    blocks = c3_blocks(side, lags, lag_scale)
    n = side * side
    pat = make_pattern("toeplitz", lags, lags, n, n, block_symmetric=True)
    w = np.sqrt(np.asarray(pat.counts, dtype=np.float64))
    t = np.transpose(blocks, (1, 0, 2)) * w[None, :, None]
    return pat, blocks, np.ascontiguousarray(t)


# ---------------------------------------------------------------------------
# C4 3-D blur: 255^3 PSF on a 128^3 image, CP R=16 x 30
# ---------------------------------------------------------------------------


def c4_psf(k=255, sig=(2.0, 3.0, 4.0), angle_deg=30.0, mix=0.7):
    h = (k - 1) // 2
    d = np.arange(-h, h + 1, dtype=np.float64)
    d1, d2, d3 = np.meshgrid(d, d, d, indexing="ij")
    s = [2 * v * v for v in sig]
    ga = np.exp(-(d1**2 / s[0] + d2**2 / s[1] + d3**2 / s[2]))
    th = np.deg2rad(angle_deg)
    c, sn = np.cos(th), np.sin(th)
    # R^T d for a rotation about axis 3 (z)
    e1 = c * d1 + sn * d2
    e2 = -sn * d1 + c * d2
    gr = np.exp(-(e1**2 / s[0] + e2**2 / s[1] + d3**2 / s[2]))
    psf = mix * ga + (1.0 - mix) * gr
    return psf / psf.sum()


def c4_tensor(k=255, grid=128):
    return np.ascontiguousarray(psf_weighted(c4_psf(k), grid))


# ---------------------------------------------------------------------------
# C5 rank-64 CP model + 1e-4 Philox noise (index addressable)
# ---------------------------------------------------------------------------

_PHILOX_M0 = np.uint64(0xD2511F53)
_PHILOX_M1 = np.uint64(0xCD9E8D57)
_PHILOX_W0 = np.uint32(0x9E3779B9)
_PHILOX_W1 = np.uint32(0xBB67AE85)


def philox_normal(index, key=3):
    """Philox4x32-10 (counter = (lo32(idx), hi32(idx), 0, 0), key = (key, 0)),
    two uint32 outputs -> two uniforms in (0, 1] -> Box-Muller cosine branch.
    Same recipe as ``bt_c5_noise`` in csrc/builders.cu (agrees to the last
    ulp of log/cos, i.e. ~1e-16 relative of a 1e-4 perturbation)."""
    idx = np.asarray(index, dtype=np.uint64)
    c0 = (idx & np.uint64(0xFFFFFFFF)).astype(np.uint64)
    c1 = (idx >> np.uint64(32)).astype(np.uint64)
    c2 = np.zeros_like(c0)
    c3 = np.zeros_like(c0)
    k0 = np.full_like(c0, np.uint64(key))
    k1 = np.zeros_like(c0)
    mask = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = _PHILOX_M0 * c0
        p1 = _PHILOX_M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & mask, lo1, (hi0 ^ c3 ^ k1) & mask, lo0
        k0 = (k0 + np.uint64(_PHILOX_W0)) & mask
        k1 = (k1 + np.uint64(_PHILOX_W1)) & mask
    u1 = (c0.astype(np.float64) + 1.0) * 2.0**-32
    u2 = (c1.astype(np.float64) + 0.5) * 2.0**-32
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def c5_factors(i=4096, j=4096, k=1024, r=64, seed=3):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((i, r)), rng.standard_normal((j, r)), rng.standard_normal((k, r))


def c5_tensor(i, j, k, r, noise=1e-4, seed=3, k_slab=None):
    """X = [[A0, B0, C0]] + noise * eps(linear C-order index).  ``k_slab``
    (k0, k1) restricts to mode-3 rows k0:k1 with the *global* index for eps."""
    a0, b0, c0 = c5_factors(i, j, k, r, seed)
    k0, k1 = (0, k) if k_slab is None else k_slab
    x = np.einsum("ir,jr,kr->ijk", a0, b0, c0[k0:k1], optimize=True)
    ii, jj, kk = np.meshgrid(np.arange(i, dtype=np.uint64), np.arange(j, dtype=np.uint64),
                             np.arange(k0, k1, dtype=np.uint64), indexing="ij")
    lin = (ii * np.uint64(j) + jj) * np.uint64(k) + kk
    return x + noise * philox_normal(lin)


# ---------------------------------------------------------------------------
# gather stand-in: C1's generator scaled up
# ---------------------------------------------------------------------------


def spd_toeplitz(seed, ell=4, nb=5, decay=0.3):
    """Seeded SPD block-Toeplitz input for spd_compress (psd.py:205): an SPD
    anchor on the diagonal, random off-diagonal classes (A_-d = A_d^T), the
    anchor shifted until the assembled matrix has lambda_min >= 1."""
    rng = np.random.default_rng(seed)
    from .port import assemble, make_pattern

    pat = make_pattern("toeplitz", ell, ell, nb, nb)
    g = rng.standard_normal((nb, nb))
    anchor = g @ g.T + nb * np.eye(nb)
    up = [decay * rng.standard_normal((nb, nb)) for _ in range(ell - 1)]
    blocks = [anchor] + up + [u.T for u in up]
    a = assemble(pat, blocks)
    lo = np.linalg.eigvalsh(a).min()
    if lo < 1.0:
        blocks[0] = blocks[0] + (1.0 - lo) * np.eye(nb)
        a = assemble(pat, blocks)
    return pat, a


def detect_cases():
    """Seeded inputs for detect_pattern (blocks.py:266): (name, a, m, n, tol).
    Structured matrices from the named builders with random blocks, plus the
    edge cases the reference handles explicitly: all-zero and -0.0 blocks
    (skipped), NaN blocks (kept; never within tol), near-equal blocks that
    only merge under tol, a ragged 3 x 5 grid of 3 x 2 blocks."""
    from .port import assemble, make_pattern

    rng = np.random.default_rng(41)
    out = []
    for kind, ell in (("toeplitz", 6), ("hankel", 5), ("diagonal", 4)):
        pat = make_pattern(kind, ell, ell, 3, 3)
        blocks = [rng.standard_normal((3, 3)) for _ in range(pat.p)]
        out.append((f"{kind}{ell}", assemble(pat, blocks), 3, 3, 0.0))
    pat = make_pattern("banded", 6, 6, 2, 2, band=1)
    out.append(("banded6", assemble(pat, [rng.standard_normal((2, 2)) for _ in range(pat.p)]),
                2, 2, 0.0))
    # ragged grid with repeats, zeros, -0.0 and a NaN block
    choices = [rng.standard_normal((3, 2)) for _ in range(4)]
    a = np.zeros((9, 10))
    for i in range(3):
        for j in range(5):
            c = (i * 5 + j * 3) % 6
            if c < 4:
                a[i * 3:(i + 1) * 3, j * 2:(j + 1) * 2] = choices[c]
            elif c == 5:
                a[i * 3:(i + 1) * 3, j * 2:(j + 1) * 2] = -0.0
    a[6:9, 8:10] = np.nan
    out.append(("ragged", a, 3, 2, 0.0))
    # near-equal blocks: exact splits them, tol merges them
    base = rng.standard_normal((4, 4))
    b = np.block([[base, base + 1e-9, np.zeros((4, 4))],
                  [base - 2e-9, np.zeros((4, 4)), base + 1e-3],
                  [np.full((4, 4), 5e-7), base, base + 1e-9]])
    for tol in (0.0, 1e-8, 1e-6, 1e-2):
        out.append((f"near_tol{tol:g}", b, 4, 4, tol))
    # C1 matrix, exact and loose
    _, c1 = c1_inputs()
    out.append(("c1", c1, 32, 32, 0.0))
    out.append(("c1_tol", c1, 32, 32, 1e-3))
    return out


def era_system(seed, d=6, n_out=2, n_in=2, rho=0.9):
    """Seeded stable LTI system for the ERA cases (spectral radius rho)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((d, d))
    a *= rho / np.max(np.abs(np.linalg.eigvals(a)))
    return a, rng.standard_normal((d, n_in)), rng.standard_normal((n_out, d))


def gather_standin(nb=256, ell=128):
    x = np.linspace(0.0, 1.0, nb)
    base = np.exp(-((x[:, None] - x[None, :]) ** 2) / (2 * 0.1**2))
    rng = np.random.default_rng(0)
    blocks = []
    for k in range(ell):
        g = rng.standard_normal((nb, nb))
        blocks.append(base * np.exp(-(k**2) / 32.0) + 1e-3 * (g + g.T) / 2)
    pat = make_pattern("toeplitz", ell, ell, nb, nb, block_symmetric=True)
    return pat, np.stack(blocks)


def c1_reference_tensor():
    pat, a = c1_inputs()
    return pat, a, gather(a, pat)


def c5_tensor_rows(factors, i0, i1, dims, noise=1e-4):
    """Mode-1 rows i0:i1 of the C5 tensor of extents ``dims`` (same values as
    ``c5_tensor``: model + noise * eps(global linear C-order index)), so large
    instances can be generated chunk by chunk without the full index grids."""
    a0, b0, c0 = factors
    _, j, k = dims
    x = np.einsum("ir,jr,kr->ijk", a0[i0:i1], b0, c0, optimize=True)
    base = (np.arange(i0, i1, dtype=np.uint64) * np.uint64(j))[:, None] + np.arange(j, dtype=np.uint64)[None, :]
    lin = base[:, :, None] * np.uint64(k) + np.arange(k, dtype=np.uint64)[None, None, :]
    x += noise * philox_normal(lin)
    return x


def c5_tensor_threaded(i, j, k, r, noise=1e-4, seed=3, rows=16, threads=8):
    """``c5_tensor`` for instances too large for its index grids: mode-1 row
    chunks generated on a thread pool (numpy releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    f = c5_factors(i, j, k, r, seed)
    out = np.empty((i, j, k))

    def one(i0):
        out[i0:i0 + rows] = c5_tensor_rows(f, i0, min(i, i0 + rows), (i, j, k), noise)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, range(0, i, rows)))
    return out
