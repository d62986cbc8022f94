"""CPU oracle for the bt200 hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``blockten``
(``/root/reference/pkg/src/blockten``) for exactly the functions on the
hot path.  It exists so that ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` have a checker and a CPU timing arm that travel to the
GPU box (``/root/reference`` does not).  The shipped product
(``paper_2105_01170_b200``) never imports this file.

Pinning: every function here is checked against golden vectors produced by
the *unmodified reference* in this container (``tests/golden/make_golden.py``
writes ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` compares).
Functions the reference does not have (ST-HOSVD, HOOI, CP -> multilevel
Kronecker terms, multilevel matvec, the generalized PSF weighting for an
image larger than the kernel) are restated *only* from the pinned
primitives below and are anchored by the reductions listed in SURVEY.md
section 8c.

Conventions follow the reference: numpy C-order storage, first-index-fastest
unfoldings (tensor.py:1-16), 1-based modes in signatures, fp64 values,
int64 placements.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.linalg import khatri_rao

DENSIFY_LIMIT = 10**8  # reconstruct.py:45


class ShapeError(ValueError):
    pass


class PatternMismatchError(ValueError):
    pass


# ---------------------------------------------------------------------------
# tensor primitives (tensor.py:40-109)
# ---------------------------------------------------------------------------


def unfold(t, mode):
    """tensor.py:40-52 -- rows = mode index, columns first-index-fastest."""
    ax = mode - 1
    if not 0 <= ax < t.ndim:
        raise ShapeError("mode out of range")
    return np.reshape(np.moveaxis(t, ax, 0), (t.shape[ax], -1), order="F")


def fold(mat, mode, dims):
    """tensor.py:55-72."""
    ax = mode - 1
    rest = tuple(dims[:ax]) + tuple(dims[ax + 1:])
    arr = np.reshape(mat, (dims[ax], *rest), order="F")
    return np.moveaxis(arr, 0, ax)


def mode_multiply(t, mode, u):
    """tensor.py:75-90: ``fold(u @ unfold(t, mode))``."""
    dims = list(t.shape)
    dims[mode - 1] = u.shape[0]
    return fold(u @ unfold(t, mode), mode, tuple(dims))


def fro_norm(t):
    """tensor.py:107-109."""
    return float(np.linalg.norm(np.asarray(t).ravel()))


# ---------------------------------------------------------------------------
# block patterns (blocks.py:42-220)
# ---------------------------------------------------------------------------


@dataclass(frozen=True, eq=False)
class Pattern:
    """Minimal stand-in for blocks.py:42-123 ``BlockPattern``."""

    ell: int
    q: int
    m: int
    n: int
    placements: tuple
    structure_class: str = "general"

    @property
    def p(self):
        return len(self.placements)

    @property
    def counts(self):
        return tuple(len(c) for c in self.placements)

    @property
    def shape(self):
        return (self.ell * self.m, self.q * self.n)


def _diag_cells(ell, off):
    """blocks.py:131-137: cells of diagonal ``col - row == off``."""
    r = np.arange(ell - off) if off >= 0 else np.arange(-off, ell)
    return np.column_stack([r, r + off]).astype(np.int64)


def make_pattern(kind, ell, q, m, n, band=None, block_symmetric=False):
    """Restatement of blocks.py:140-220 (class and cell ordering included)."""
    if ell != q:
        raise ShapeError("square block grid required")
    classes = []
    tag = kind
    if kind == "diagonal":
        classes = [np.array([[k, k]], dtype=np.int64) for k in range(ell)]
    elif kind == "banded":
        if band is None or not 0 <= band < ell:
            raise ShapeError("bad band")
        slot = {}
        for i in range(ell):
            for j in range(q):
                if abs(i - j) > band:
                    continue
                key = (min(i, j), max(i, j)) if block_symmetric else (i, j)
                if key not in slot:
                    slot[key] = len(classes)
                    classes.append([])
                classes[slot[key]].append((i, j))
        classes = [np.array(c, dtype=np.int64) for c in classes]
        tag = (f"banded_symmetric:{band}" if block_symmetric else f"banded:{band}")
    elif kind == "toeplitz":
        cut = ell - 1 if band is None else band
        if not 0 <= cut < ell:
            raise ShapeError("bad cutoff")
        classes.append(_diag_cells(ell, 0))
        if block_symmetric:
            for d in range(1, cut + 1):
                classes.append(np.vstack([_diag_cells(ell, -d), _diag_cells(ell, d)]))
            tag = "toeplitz_symmetric"
        else:
            classes += [_diag_cells(ell, -d) for d in range(1, cut + 1)]
            classes += [_diag_cells(ell, d) for d in range(1, cut + 1)]
            tag = "toeplitz"
        if band is not None and band < ell - 1:
            tag += f":{band}"
    elif kind == "hankel":
        for s in range(2 * ell - 1):
            r = np.arange(max(0, s - ell + 1), min(s, ell - 1) + 1)
            classes.append(np.column_stack([r, s - r]).astype(np.int64))
    else:
        raise ValueError(kind)
    return Pattern(ell, q, m, n, tuple(classes), tag)


def kernel_level_pattern(k, bm, bn, grid=None):
    """multilevel.py:247-265 generalised to an image grid of ``grid`` cells
    per side (the reference fixes grid == k).  Class i sits on diagonal
    ``col - row = h - i`` with ``h = (k-1)//2``; ``eta_i = grid - |i - h|``."""
    grid = k if grid is None else grid
    h = (k - 1) // 2
    cells = [_diag_cells(grid, h - i) for i in range(k)]
    return Pattern(grid, grid, bm, bn, tuple(cells), f"toeplitz:{h}")


# ---------------------------------------------------------------------------
# assembly and the tensor maps (blocks.py:351-462)
# ---------------------------------------------------------------------------


def assemble(pat, blocks):
    """blocks.py:351-360: block k verbatim on every cell of class k."""
    out = np.zeros(pat.shape)
    m, n = pat.m, pat.n
    for blk, cells in zip(blocks, pat.placements):
        for i, j in cells:
            out[i * m:(i + 1) * m, j * n:(j + 1) * n] = blk
    return out


def expand(pat, items):
    """blocks.py:363-381: cell value ``item_k / sqrt(eta_k)``."""
    items = [np.atleast_2d(np.asarray(x, dtype=np.float64)) for x in items]
    bm, bn = items[0].shape
    out = np.zeros((pat.ell * bm, pat.q * bn))
    for item, cells in zip(items, pat.placements):
        val = item / np.sqrt(len(cells))
        for i, j in cells:
            out[i * bm:(i + 1) * bm, j * bn:(j + 1) * bn] = val
    return out


def scalars(pat, coeffs):
    """blocks.py:384-392."""
    out = np.zeros((pat.ell, pat.q))
    for c, cells in zip(np.asarray(coeffs, dtype=np.float64), pat.placements):
        out[cells[:, 0], cells[:, 1]] = c / np.sqrt(len(cells))
    return out


def gather(a, pat, tol=0.0, weighted=True):
    """blocks.py:395-449: verify every placement against the first one of its
    class, verify uncovered cells are zero, stack weighted representatives.
    Raises PatternMismatchError naming the first offending cell in the
    reference's scan order (classes in order, then uncovered cells
    row-major)."""
    if a.shape != pat.shape:
        raise ShapeError("shape")
    m, n = pat.m, pat.n
    covered = np.zeros((pat.ell, pat.q), dtype=bool)
    t = np.zeros((m, pat.p, n))
    for k, cells in enumerate(pat.placements):
        i0, j0 = cells[0]
        rep = a[i0 * m:(i0 + 1) * m, j0 * n:(j0 + 1) * n]
        for i, j in cells:
            covered[i, j] = True
            if np.max(np.abs(a[i * m:(i + 1) * m, j * n:(j + 1) * n] - rep)) > tol:
                raise PatternMismatchError(f"class {k + 1}: block at grid cell ({i + 1}, {j + 1})")
        w = np.sqrt(len(cells)) if weighted else 1.0
        t[:, k, :] = w * rep
    for i, j in np.argwhere(~covered):
        if np.max(np.abs(a[i * m:(i + 1) * m, j * n:(j + 1) * n])) > tol:
            raise PatternMismatchError(f"grid cell ({i + 1}, {j + 1}) is outside every class")
    return t


def scatter(t, pat):
    """blocks.py:452-462 -> struct_expand of the lateral slices."""
    return expand(pat, [t[:, k, :] for k in range(pat.p)])


# ---------------------------------------------------------------------------
# decompositions (decomp.py:149-410)
# ---------------------------------------------------------------------------


def _sign_fix(u):
    """decomp.py:176-179: largest-|.| entry of every column made positive."""
    lead = np.argmax(np.abs(u), axis=0)
    s = np.sign(u[lead, np.arange(u.shape[1])])
    s[s == 0] = 1.0
    return s


def svd_trunc(a, r):
    """decomp.py:149-179."""
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    u, vt = u[:, :r], vt[:r, :]
    sg = _sign_fix(u)
    return u * sg, s[:r].copy(), (vt * sg[:, None]).T


def mode_basis(mat, r):
    """decomp.py:220-234 (full_matrices completion when r > min(shape))."""
    if r <= min(mat.shape):
        return svd_trunc(mat, r)[0]
    u = np.linalg.svd(mat, full_matrices=True)[0][:, :r]
    return u * _sign_fix(u)


def hosvd(t, ranks):
    """decomp.py:237-259: bases from the original unfoldings, core by
    sequential projection in mode order."""
    fac = [mode_basis(unfold(t, k + 1), r) for k, r in enumerate(ranks)]
    core = t
    for k, u in enumerate(fac):
        core = mode_multiply(core, k + 1, u.T)
    return core, fac


def tucker_partial(t, ranks, shared=None, shared_from="first"):
    """decomp.py:262-321."""
    fac = [None] * t.ndim
    skip = ()
    if shared is not None:
        a, b = shared
        src = unfold(t, a) if shared_from == "first" else np.hstack([unfold(t, a), unfold(t, b)])
        u = mode_basis(src, int(ranks[a - 1]))
        fac[a - 1] = u
        fac[b - 1] = u
        skip = (a - 1, b - 1)
    for k, r in enumerate(ranks):
        if k in skip or r is None:
            continue
        fac[k] = mode_basis(unfold(t, k + 1), r)
    core = t
    for k, u in enumerate(fac):
        if u is not None:
            core = mode_multiply(core, k + 1, u.T)
    return core, fac


def cp_init_hosvd(t, r):
    """decomp.py:329-341 (the reference's default initialisation)."""
    rng = np.random.default_rng(0)
    out = []
    for k in range(3):
        mat = unfold(t, k + 1)
        keep = min(r, t.shape[k], mat.shape[1])
        u = svd_trunc(mat, keep)[0]
        if keep < r:
            u = np.hstack([u, rng.standard_normal((t.shape[k], r - keep))])
        out.append(u)
    return out


def cp_init_normal(seed):
    """SURVEY 8d generator convention: seeded N(0,1) init drawn in mode order."""
    def init(t, r):
        rng = np.random.default_rng(seed)
        return [rng.standard_normal((t.shape[k], r)) for k in range(3)]
    return init


@dataclass
class CpOut:
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    fit: float
    fit_history: tuple
    n_iters: int
    converged: bool


def cp_als(t, r, max_iters=500, tol=1e-10, init=None):
    """decomp.py:344-410: ALS with pinv of the Hadamard of Grams, column
    normalisation, lambda from the mode-3 update, explicit fit via full
    reconstruction (decomp.py:395-396)."""
    norm_t = fro_norm(t)
    if norm_t == 0.0:
        raise ValueError("zero tensor")
    f = [np.array(x, dtype=np.float64) for x in (init or cp_init_hosvd)(t, r)]
    unf = [unfold(t, k + 1) for k in range(3)]
    g = [x.T @ x for x in f]
    hist = []
    prev = -np.inf
    conv = False
    it = 0
    lam = None
    for it in range(1, max_iters + 1):
        for k in range(3):
            o0, o1 = [j for j in range(3) if j != k]
            f[k] = unf[k] @ khatri_rao(f[o1], f[o0]) @ np.linalg.pinv(g[o0] * g[o1])
            nrm = np.linalg.norm(f[k], axis=0)
            nrm[nrm == 0] = 1.0
            f[k] = f[k] / nrm
            if k == 2:
                lam = nrm
            g[k] = f[k].T @ f[k]
        approx = np.einsum("ir,jr,kr->ijk", f[0] * lam, f[1], f[2])
        fit = 1.0 - fro_norm(t - approx) / norm_t
        hist.append(fit)
        if abs(fit - prev) < tol:
            conv = True
            break
        prev = fit
    return CpOut(f[0] * lam, f[1], f[2], hist[-1], tuple(hist), it, conv)


def cp_sweep_slab(t, f, lam_out=False):
    """One ALS sweep of decomp.py:380-393 on given factors (used to time a
    bounded CPU sample of a large config)."""
    return cp_als(t, f[0].shape[1], max_iters=1, tol=0.0, init=lambda _t, _r: f)


# ---------------------------------------------------------------------------
# restated (no reference function): ST-HOSVD and HOOI
# ---------------------------------------------------------------------------


def st_hosvd_shared13(t, r13, r2):
    """ST-HOSVD for a transpose-closed order-3 tensor with modes 1/3 sharing
    one basis: U from unfold(t,1) (== tucker_partial(shared=(1,3)) step),
    then V from the mode-2 unfolding of t x1 U^T x3 U^T."""
    u = mode_basis(unfold(t, 1), r13)
    y = mode_multiply(mode_multiply(t, 1, u.T), 3, u.T)
    v = mode_basis(unfold(y, 2), r2)
    core = mode_multiply(y, 2, v.T)
    return core, [u, v, u]


def hooi_shared13(t, u, v, sweeps):
    """HOOI sweeps with the shared 1/3 basis: U from unfold(t x2 V^T x3 U^T, 1),
    V from unfold(t x1 U^T x3 U^T, 2); core = t x1 U^T x2 V^T x3 U^T."""
    r13, r2 = u.shape[1], v.shape[1]
    for _ in range(sweeps):
        w = mode_multiply(mode_multiply(t, 2, v.T), 3, u.T)
        u = mode_basis(unfold(w, 1), r13)
        y = mode_multiply(mode_multiply(t, 1, u.T), 3, u.T)
        v = mode_basis(unfold(y, 2), r2)
    core = mode_multiply(mode_multiply(mode_multiply(t, 1, u.T), 2, v.T), 3, u.T)
    return core, [u, v, u]


# ---------------------------------------------------------------------------
# representations (reconstruct.py:170-345, psd.py:51-187)
# ---------------------------------------------------------------------------


def kron_from_kruskal(x, y, z, split="factor"):
    """reconstruct.py:192-226 -> (coeffs (p, r), terms (r, m, n))."""
    r = x.shape[1]
    if split == "factor":
        f, g = y, np.eye(r)
    else:
        q, rr = np.linalg.qr(y, mode="reduced")
        s = np.sign(np.diag(rr))
        s[s == 0] = 1.0
        f, g = q * s, (rr * s[:, None]).T
    terms = np.empty((r, x.shape[0], z.shape[0]))
    for j in range(r):
        terms[j] = (x * g[:, j]) @ z.T
    return f.copy(), terms


def kron_from_tucker(core, fac, p):
    """reconstruct.py:170-189."""
    u, v, w = fac
    coeffs = np.eye(p) if v is None else v.copy()
    terms = np.empty((core.shape[1], u.shape[0] if u is not None else core.shape[0],
                      w.shape[0] if w is not None else core.shape[2]))
    for j in range(core.shape[1]):
        d = core[:, j, :]
        if u is not None:
            d = u @ d
        if w is not None:
            d = d @ w.T
        terms[j] = d
    return coeffs, terms


def blr_from_tucker(core, fac, m, n):
    """reconstruct.py:229-240 -> (left, right, middles)."""
    u, v, w = fac
    left = np.eye(m) if u is None else u.copy()
    right = np.eye(n) if w is None else w.copy()
    mids = (np.ascontiguousarray(np.moveaxis(core, 1, 0)) if v is None
            else np.einsum("ajb,kj->kab", core, v))
    return left, right, mids


def matvec_kron(pat, coeffs, terms, x):
    """reconstruct.py:271-295 (Kron-sum branch); x of length q*n."""
    m, n, ell, q = pat.m, pat.n, pat.ell, pat.q
    xm = x.reshape((n, q), order="F")
    acc = np.zeros((m, ell))
    for j in range(terms.shape[0]):
        cj = scalars(pat, coeffs[:, j])
        acc += (cj @ (terms[j] @ xm).T).T
    return acc.reshape(-1, order="F")


def matvec_blr(pat, left, right, mids, x):
    """reconstruct.py:297-313 (BLR branch)."""
    n, ell, q = pat.n, pat.ell, pat.q
    xm = x.reshape((n, q), order="F")
    z = right.T @ xm
    yb = np.zeros((left.shape[1], ell))
    for k, cells in enumerate(pat.placements):
        s = mids[k] / np.sqrt(len(cells))
        for i, j in cells:
            yb[:, i] += s @ z[:, j]
    return (left @ yb).reshape(-1, order="F")


def matvec_blr_fast(pat, left, right, mids, xs):
    """Vectorised restatement of the BLR branch for many RHS (same
    arithmetic per cell, grouped by class); ``xs`` is (q*n, nrhs)."""
    n, ell, q = pat.n, pat.ell, pat.q
    nrhs = xs.shape[1]
    xm = xs.reshape((q, n, nrhs)).transpose(1, 0, 2)           # (n, q, nrhs)
    z = np.einsum("nr,nqk->rqk", right, xm)                     # (rr, q, nrhs)
    yb = np.zeros((left.shape[1], ell, nrhs))
    for k, cells in enumerate(pat.placements):
        s = mids[k] / np.sqrt(len(cells))
        contrib = np.einsum("ab,bck->ack", s, z[:, cells[:, 1], :])
        np.add.at(yb, (slice(None), cells[:, 0]), contrib)
    y = np.einsum("ma,aik->mik", left, yb)                      # (m, ell, nrhs)
    return y.transpose(1, 0, 2).reshape(ell * left.shape[0], nrhs)


def densify_kron(pat, coeffs, terms):
    """reconstruct.py:318-331."""
    return expand(pat, [np.tensordot(coeffs[k, :], terms, axes=(0, 0)) for k in range(pat.p)])


def densify_blr(pat, left, right, mids):
    """reconstruct.py:332-334."""
    return expand(pat, [left @ mids[k] @ right.T for k in range(pat.p)])


def spsd_blocks(pat, blocks, r):
    """psd.py:164-187 (transpose-closure check omitted: the configs satisfy
    it by construction) -> (basis, projected blocks)."""
    n = pat.m
    t = np.zeros((n, pat.p, n))
    for k, blk in enumerate(blocks):
        t[:, k, :] = np.sqrt(pat.counts[k]) * blk
    u = mode_basis(unfold(t, 1), r)
    proj = np.stack([u.T @ blk @ u for blk in blocks])
    return u, proj


def classify_placements(placements, ell, q):
    """blocks.py:228-263 (descriptive tag, no arithmetic)."""
    allc = np.vstack(placements) if placements else np.zeros((0, 2), dtype=np.int64)
    if len(allc) and np.all(allc[:, 0] == allc[:, 1]):
        return "diagonal"

    def full_diag(cells):
        offs = {int(j - i) for i, j in cells}
        if ell != q:
            return None
        if len(offs) == 1:
            (d,) = offs
            return d if len(cells) == ell - abs(d) else None
        if len(offs) == 2:
            lo, hi = sorted(offs)
            if lo == -hi and hi > 0 and len(cells) == 2 * (ell - hi):
                return hi
        return None

    def full_anti(cells):
        sums = {int(i + j) for i, j in cells}
        if ell != q or len(sums) != 1:
            return None
        (s,) = sums
        return s if len(cells) == min(s + 1, ell, 2 * ell - 1 - s) else None

    if placements and all(full_diag(c) is not None for c in placements):
        return "toeplitz"
    if placements and all(full_anti(c) is not None for c in placements):
        return "hankel"
    if len(allc):
        b = int(np.max(np.abs(allc[:, 0] - allc[:, 1])))
        if b < max(ell, q) - 1:
            return f"banded:{b}"
    return "general"


def markov_from_lti(a, b, c, count):
    """apps.py:105-114."""
    out = np.empty((count, c.shape[0], b.shape[1]))
    x = b.copy()
    for k in range(count):
        out[k] = c @ x
        x = a @ x
    return out


def era_identify(params, ranks, order, tera=False):
    """apps.py:153-237 -> (a, b, c, sing_vals, reduced, u, w)."""
    s = (params.shape[0] + 1) // 2
    pat = make_pattern("hankel", s, s, params.shape[1], params.shape[2])
    r1, r2, r3 = ranks
    t = np.transpose(params, (1, 0, 2)).copy()
    rp = Pattern(pat.ell, pat.q, r1, r3, pat.placements)
    if tera:
        u = mode_basis(unfold(t, 1), r1)
        w = mode_basis(unfold(t, 3), r3)
        reduced = assemble(rp, [u.T @ h @ w for h in params])
    else:
        t *= np.sqrt(np.asarray(pat.counts, dtype=np.float64))[None, :, None]
        core, (u, v, w) = hosvd(t, [r1, r2, r3])
        items = np.einsum("kj,ajb->kab", v, core)
        reduced = expand(rp, items)
    su, sv, svt = np.linalg.svd(reduced, full_matrices=False)
    root = np.sqrt(sv[:order])
    theta = su[:, :order] * root
    gamma_t = root[:, None] * svt[:order]
    a_til = np.linalg.lstsq(theta[: r1 * (s - 1)], theta[r1:], rcond=None)[0]
    return a_til, gamma_t[:, :r3] @ w.T, u @ theta[:r1], sv, reduced, u, w


def detect_pattern(a, m, n, tol=0.0):
    """blocks.py:266-329: row-major scan; tol == 0 groups by the block's bytes
    (all-zero blocks skipped), tol > 0 joins the first representative within
    tol.  Returns (placements, reps, structure_class)."""
    ell, q = a.shape[0] // m, a.shape[1] // n
    reps, cells, by_bytes = [], [], {}
    for i in range(ell):
        for j in range(q):
            blk = np.ascontiguousarray(a[i * m:(i + 1) * m, j * n:(j + 1) * n])
            if tol == 0.0:
                if not blk.any():
                    continue
                k = by_bytes.setdefault(blk.tobytes(), len(reps))
                if k == len(reps):
                    reps.append(blk)
                    cells.append([])
            else:
                if np.max(np.abs(blk)) <= tol:
                    continue
                k = next((kk for kk, r in enumerate(reps) if np.max(np.abs(blk - r)) <= tol),
                         len(reps))
                if k == len(reps):
                    reps.append(blk)
                    cells.append([])
            cells[k].append((i, j))
    placements = tuple(np.array(c, dtype=np.int64) for c in cells)
    return placements, reps, classify_placements(placements, ell, q)


def cholesky(a):
    """decomp.py:196-212 (numpy's LAPACK potrf; asymmetry > 1e-12 max|a|
    is a ShapeError, a failed pivot a ValueError here)."""
    scale = np.max(np.abs(a)) or 1.0
    if np.max(np.abs(a - a.T)) > 1e-12 * scale:
        raise ShapeError("cholesky expects a symmetric matrix")
    return np.linalg.cholesky(a)


def spd_compress(a, pat, r):
    """psd.py:205-271 -> (chol, remainder placements, remainder basis,
    remainder projected blocks)."""
    from scipy.linalg import solve_triangular

    blocks = [a[c[0, 0] * pat.m:(c[0, 0] + 1) * pat.m, c[0, 1] * pat.n:(c[0, 1] + 1) * pat.n]
              for c in pat.placements]
    k0 = next(k for k, c in enumerate(pat.placements)
              if np.any((c[:, 0] == 0) & (c[:, 1] == 0)))
    anchor = blocks[k0]
    low = cholesky(anchor)
    cells_out, rem = [], []
    for k, cells in enumerate(pat.placements):
        on = cells[:, 0] == cells[:, 1]
        for mask, shift in ((on, anchor), (~on, None)):
            if not mask.any():
                continue
            blk = blocks[k] - shift if shift is not None else blocks[k]
            if not blk.any():
                continue
            cells_out.append(cells[mask])
            rem.append(blk)
    scaled = []
    for blk in rem:
        half = solve_triangular(low, blk, lower=True)
        scaled.append(solve_triangular(low, half.T, lower=True).T)
    if not cells_out:
        return low, [], np.eye(pat.m)[:, :r], np.zeros((0, r, r))
    rp = Pattern(pat.ell, pat.q, pat.m, pat.n, tuple(cells_out))
    u, proj = spsd_blocks(rp, scaled, r)
    return low, cells_out, u, proj


def densify_spd(pat, low, cells, u, proj):
    """psd.py:129-138: (I (x) L)(I + M)(I (x) L^T)."""
    n = low.shape[0]
    inner = np.eye(pat.ell * n)
    if cells:
        rp = Pattern(pat.ell, pat.q, n, n, tuple(cells))
        inner = inner + assemble(rp, np.stack([u @ b @ u.T for b in proj]))
    lf = np.kron(np.eye(pat.ell), low)
    return lf @ inner @ lf.T


# ---------------------------------------------------------------------------
# multilevel (multilevel.py:197-298) + restated CP route / matvec
# ---------------------------------------------------------------------------


def psf_weighted(psf, grid=None):
    """multilevel.py:268-298 with the image grid generalised: weight
    sqrt(eta_i1 eta_i2 eta_i3) times psf[i3, i2, i1]."""
    k = psf.shape[0]
    grid = k if grid is None else grid
    h = (k - 1) // 2
    eta = (grid - np.abs(np.arange(k) - h)).astype(np.float64)
    w = np.sqrt(np.einsum("a,b,c->abc", eta, eta, eta))
    return w * np.transpose(psf, (2, 1, 0))


def ml_kron_from_kruskal(levels, x, y, z):
    """CP route to multilevel terms (restated): term r = (S1(x_r), S2(y_r),
    S3(z_r)) with S_t = struct_scalars(level_t, .) and a 1x1 innermost block
    (the squeezed order-5 tensor has singleton innermost modes)."""
    return [(scalars(levels[0], x[:, r]), scalars(levels[1], y[:, r]),
             scalars(levels[2], z[:, r])) for r in range(x.shape[1])]


def ml_matvec(terms, vols):
    """Restated multilevel Kronecker matvec: y = sum_r (S1 (x) S2 (x) S3) x with
    x the first-image-axis-fastest vectorisation.  ``vols`` is
    (nrhs, N3, N2, N1) C-order, i.e. vol[b, a3, a2, a1] = x[a1 + N1 a2 + N1 N2 a3]
    -- level 1 (outermost Kronecker factor) acts on a3."""
    out = np.zeros(vols.shape[:1] + (terms[0][0].shape[0], terms[0][1].shape[0],
                                     terms[0][2].shape[0]))
    for s1, s2, s3 in terms:
        out += np.einsum("ia,jb,kc,nabc->nijk", s1, s2, s3, vols, optimize=True)
    return out
