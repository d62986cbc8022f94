"""Config-size golden fixtures from the UNMODIFIED reference (this container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_big.py [c3] [c5] [c4] [mlt]

Companion of ``make_golden.py`` for the BASELINE configs at (or near) their
stated sizes, where the full outputs are too large to commit: each fixture
keeps what the GPU parity tests need to compare at north_star's tolerances
(bases, cores, fit histories, factors, sampled slices and fingerprints).

* ``big_c3.npz`` -- C3 at full size (1024 x 512 x 1024, 4.3 GB):
  reference ``tucker_partial(t, [64, None, 64], shared=(1, 3))``
  (decomp.py:262-321) and ``spsd_compress_blocks(pat, blocks, 64)``
  (psd.py:164-187); the restated ST-HOSVD (its mode-1 step IS the reference
  ``tucker_partial`` basis) + 5 HOOI sweeps (oracle/port.py); the reference
  ``blr_from_tucker`` (reconstruct.py:229-240) of that (64, 32, 64) Tucker and
  its ``matvec`` (reconstruct.py:271-315) on one seeded RHS.
* ``big_c5.npz`` -- C5 recipe at 1024 x 1024 x 512, R = 64 (the headline rank;
  all 64 columns live), init seed 1003, 3 sweeps of the reference ``cp_als``
  (decomp.py:344-410) with the explicit-residual fit.
* ``big_c4.npz`` -- C4 at full size: the reference's 30-sweep ``cp_als``
  factors of the 255^3 PSF tensor (R = 16, seed-2 init) and the 128 x 128
  Toeplitz level matrices the reference ``struct_scalars`` (blocks.py:384-392)
  assembles from them through ``ml_kron_sum_from_tucker`` (multilevel.py:
  197-225) on the superdiagonal core, for the generalised level patterns
  (``BlockPattern(placements=...)``); the 128^3 matvec of the first
  4 seeded volumes sampled every 61st entry.
* ``mltucker.npz`` -- ``ml_kron_sum_from_tucker`` on general (dense-core)
  Tucker models of small multilevel patterns, incl. identity level factors.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

import blockten as bt  # noqa: E402
import blockten.decomp as bt_decomp  # noqa: E402
from blockten.blocks import BlockPattern  # noqa: E402
from blockten.multilevel import MultilevelPattern, ml_kron_sum_from_tucker  # noqa: E402

from oracle import configs as oc  # noqa: E402
from oracle import port  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
C3_SLICES = np.array([0, 1, 2, 17, 255, 510, 511])


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


def c3():
    pat3, blocks, t = oc.c3_tensor()
    pat = bt.build_pattern("toeplitz", 512, 512, 1024, 1024, block_symmetric=True)
    log("c3 tensor built")
    out = {"slices": C3_SLICES}
    # mode-1 spectrum (gap bookkeeping for the principal-angle checks)
    t1 = port.unfold(t, 1)
    lam = np.linalg.eigvalsh(t1 @ t1.T)[::-1]
    del t1
    out["sv1"] = np.sqrt(np.maximum(lam, 0.0))
    log("c3 spectrum")
    rep = bt.tucker_partial(t, [64, None, 64], shared=(1, 3))
    u = rep.factors[0]
    out["tp_u"] = u
    out["tp_core_slices"] = rep.core[:, C3_SLICES, :].copy()
    out["tp_core_norm"] = np.linalg.norm(rep.core)
    del rep
    log("c3 tucker_partial")
    sp = bt.spsd_compress_blocks(pat, blocks, 64)
    out["spsd_u"] = sp.basis
    out["spsd_blocks_slices"] = sp.blocks[C3_SLICES].copy()
    out["spsd_trace"] = sp.trace()
    del sp
    log("c3 spsd")
    # restated ST-HOSVD (mode-1 step = the reference basis above) + HOOI
    y = port.mode_multiply(port.mode_multiply(t, 1, u.T), 3, u.T)
    v = port.mode_basis(port.unfold(y, 2), 32)
    out["st_u"], out["st_v"], out["st_core"] = u, v, port.mode_multiply(y, 2, v.T)
    del y
    core_h, fac_h = port.hooi_shared13(t, u, v, 5)
    out["hooi_u"], out["hooi_v"], out["hooi_core"] = fac_h[0], fac_h[1], core_h
    log("c3 st-hosvd + hooi")
    tk = bt.TuckerRep(core=core_h, factors=(fac_h[0], fac_h[1], fac_h[0]))
    blr = bt.blr_from_tucker(tk, pat)
    out["blr_mid_slices"] = blr.middles[C3_SLICES].copy()
    rhs = np.random.default_rng(1003).standard_normal(pat.shape[1])
    yb = bt.matvec(blr, rhs)
    out["blr_y"] = yb
    log("c3 blr matvec")
    np.savez_compressed(os.path.join(OUT, "big_c3.npz"), **out)


def c5():
    dims, r, sweeps = (1024, 1024, 512), 64, 3
    x = oc.c5_tensor_threaded(*dims, r)
    log("c5 tensor built")
    init = oc.normal_init(dims, r, 1003)
    saved = bt_decomp._cp_init
    bt_decomp._cp_init = lambda _t, _r: [f.copy() for f in init]
    try:
        res = bt.cp_als(x, r, sweeps, 0.0)
    finally:
        bt_decomp._cp_init = saved
    log(f"c5 cp_als fits {res.fit_history}")
    np.savez_compressed(os.path.join(OUT, "big_c5.npz"), dims=np.array(dims + (r, sweeps)),
                        hist=np.array(res.fit_history), x=res.rep.x, y=res.rep.y, z=res.rep.z,
                        norm=np.linalg.norm(x))


def _ref_level(k, bm, bn, grid):
    """The generalised C4 level as a public reference BlockPattern: class i on
    the diagonal col - row = h - i of a grid x grid block grid."""
    h = (k - 1) // 2
    cells = []
    for i in range(k):
        off = h - i
        rows = np.arange(max(0, -off), min(grid, grid - off))
        cells.append(np.column_stack([rows, rows + off]).astype(np.int64))
    return BlockPattern(ell=grid, q=grid, m=bm, n=bn, placements=tuple(cells))


def c4():
    k, grid, r = 255, 128, 16
    x = oc.c4_tensor(k, grid).reshape(k, k, k)
    init = oc.normal_init((k, k, k), r, 2)
    saved = bt_decomp._cp_init
    bt_decomp._cp_init = lambda _t, _r: [f.copy() for f in init]
    try:
        res = bt.cp_als(x, r, 30, 0.0)
    finally:
        bt_decomp._cp_init = saved
    log(f"c4 cp_als fit {res.fit}")
    levels = (_ref_level(k, grid * grid, grid * grid, grid), _ref_level(k, grid, grid, grid),
              _ref_level(k, 1, 1, grid))
    mlp = MultilevelPattern(levels=levels)
    core = np.zeros((1, r, r, r, 1))
    core[0, np.arange(r), np.arange(r), np.arange(r), 0] = 1.0
    tk = bt.TuckerRep(core=core, factors=(None, res.rep.x, res.rep.y, res.rep.z, None))
    # the reference enumerates all r^3 multi-indices; only the superdiagonal
    # ones carry a nonzero block -- keep those (the CP route's r terms)
    terms = [tm for tm in ml_kron_sum_from_tucker(tk, mlp) if tm.block[0, 0] != 0.0]
    assert len(terms) == r
    lv = np.stack([np.stack(tm.level_mats) for tm in terms])          # (r, 3, 128, 128)
    first_col, first_row = lv[:, :, :, 0].copy(), lv[:, :, 0, :].copy()
    assert all(np.array_equal(lv[a, b, 1:, 1:], lv[a, b, :-1, :-1])
               for a in range(r) for b in range(3)), "level matrices are Toeplitz"
    vols = np.random.default_rng(1004).standard_normal((grid**3, 32))[:, :4]
    trip = [(lv[t, 0], lv[t, 1], lv[t, 2]) for t in range(r)]
    ys = port.ml_matvec(trip, vols.T.reshape(4, grid, grid, grid)).reshape(4, -1).T
    log("c4 ml matvec")
    np.savez_compressed(os.path.join(OUT, "big_c4.npz"), fit=res.fit, hist=np.array(res.fit_history),
                        x=res.rep.x, y=res.rep.y, z=res.rep.z, col=first_col, row=first_row,
                        y_sampled=ys[::61], y_norms=np.linalg.norm(ys, axis=0))


def mlt():
    rng = np.random.default_rng(97)
    out = {}
    cases = []
    inner = bt.build_pattern("banded", 3, 3, 2, 2, band=1)
    outer = bt.build_pattern("hankel", 2, 2, inner.shape[0], inner.shape[1])
    cases.append(("hb", MultilevelPattern(levels=(outer, inner))))
    lv3 = _ref_level(5, 1, 1, 4)
    lv2 = _ref_level(5, 4, 4, 4)
    lv1 = _ref_level(5, 16, 16, 4)
    cases.append(("psf", MultilevelPattern(levels=(lv1, lv2, lv3))))
    t_in = bt.build_pattern("toeplitz", 3, 3, 2, 3)
    t_out = bt.build_pattern("toeplitz", 2, 2, t_in.shape[0], t_in.shape[1], block_symmetric=True)
    cases.append(("tt", MultilevelPattern(levels=(t_out, t_in))))
    for name, mlp in cases:
        dims = mlp.dims
        for variant in ("full", "ident"):
            ranks = [max(1, d - 1) for d in dims]
            core = rng.standard_normal(tuple(ranks))
            facs = []
            for i, (d, rr) in enumerate(zip(dims, ranks)):
                f = np.linalg.qr(rng.standard_normal((d, rr)))[0]
                if variant == "ident" and i in (0, 2):      # identity factors -> None
                    f = None
                facs.append(f)
            if variant == "ident":
                shape = list(ranks)
                shape[0], shape[2] = dims[0], dims[2]
                core = rng.standard_normal(tuple(shape))
            tk = bt.TuckerRep(core=core, factors=tuple(facs))
            terms = ml_kron_sum_from_tucker(tk, mlp)
            key = f"{name}_{variant}"
            out[key + "_core"] = core
            for i, f in enumerate(facs):
                out[key + f"_f{i}"] = np.zeros((0, 0)) if f is None else f
            out[key + "_nterms"] = np.array(len(terms))
            for j, tm in enumerate(terms):
                for lvl, m in enumerate(tm.level_mats):
                    out[key + f"_t{j}_l{lvl}"] = m
                out[key + f"_t{j}_b"] = tm.block
            if mlp.shape[0] * mlp.shape[1] <= 10**6:
                out[key + "_dense"] = bt.ml_kron_densify(terms)
    np.savez_compressed(os.path.join(OUT, "mltucker.npz"), **out)


if __name__ == "__main__":
    todo = sys.argv[1:] or ["mlt", "c4", "c5", "c3"]
    for name in todo:
        globals()[name]()
        log(f"{name} done")
