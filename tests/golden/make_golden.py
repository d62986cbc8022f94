"""Generate golden fixtures from the UNMODIFIED reference (this container only).

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

Imports ``blockten`` read-only from ``/root/reference`` and records its
outputs on seeded inputs into ``tests/golden/*.npz``.  The fixtures travel to
the GPU box; the reference does not.  Every array here was produced by a
reference function (named in the key) -- nothing is computed by this repo's
code except the config input recipes of ``oracle/configs.py``, whose outputs
are themselves cross-checked against reference builders below.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

import blockten as bt  # noqa: E402
import blockten.decomp as bt_decomp  # noqa: E402
from blockten.multilevel import _kernel_level_pattern  # noqa: E402
from helpers import random_blocks, random_pattern, random_ranks, PATTERN_KINDS  # noqa: E402

from oracle import configs as oc  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def flat_placements(pat):
    cells = np.vstack(pat.placements) if pat.p else np.zeros((0, 2), np.int64)
    offs = np.cumsum([0] + list(pat.counts)).astype(np.int64)
    return cells.astype(np.int64), offs


def with_init(init):
    saved = bt_decomp._cp_init
    bt_decomp._cp_init = lambda t, r: [f.copy() for f in init]
    return saved


def patterns():
    specs = []
    for ell in (1, 2, 3, 5, 8):
        for kind in ("diagonal", "toeplitz", "hankel"):
            specs.append((kind, ell, None, False))
        specs.append(("toeplitz", ell, None, True))
        for band in range(ell):
            specs.append(("banded", ell, band, False))
            specs.append(("banded", ell, band, True))
            specs.append(("toeplitz", ell, band, False))
            specs.append(("toeplitz", ell, band, True))
    small = {}
    meta = []
    for idx, (kind, ell, band, sym) in enumerate(specs):
        pat = bt.build_pattern(kind, ell, ell, 2, 3, band=band, block_symmetric=sym)
        cells, offs = flat_placements(pat)
        small[f"cells_{idx}"] = cells
        small[f"offs_{idx}"] = offs
        meta.append({"kind": kind, "ell": ell, "band": band, "sym": sym,
                     "tag": pat.structure_class})
    # configuration-size patterns: bit-exactness via hashes
    big = []
    for kind, ell, m, n, sym in (("toeplitz", 32, 32, 32, True), ("hankel", 1024, 32, 32, False),
                                 ("toeplitz", 512, 1024, 1024, True),
                                 ("toeplitz", 128, 256, 256, True)):
        pat = bt.build_pattern(kind, ell, ell, m, n, block_symmetric=sym)
        cells, offs = flat_placements(pat)
        big.append({"kind": kind, "ell": ell, "m": m, "n": n, "sym": sym, "p": pat.p,
                    "cells_sha": sha(cells), "offs_sha": sha(offs), "tag": pat.structure_class})
    # C4 level patterns (reference builder, grid == K) for K = 7, 255
    for k in (7, 255):
        pat = _kernel_level_pattern(k, 1, 1)
        cells, offs = flat_placements(pat)
        big.append({"kind": "kernel_level", "ell": k, "m": 1, "n": 1, "sym": False, "p": pat.p,
                    "cells_sha": sha(cells), "offs_sha": sha(offs), "tag": pat.structure_class})
    np.savez_compressed(os.path.join(OUT, "patterns.npz"), **small)
    with open(os.path.join(OUT, "patterns.json"), "w") as fh:
        json.dump({"small": meta, "big": big}, fh, indent=1)


def maps():
    """Gather / scatter on random patterns of every class (helpers.py:13-46)."""
    rng = np.random.default_rng(2024)
    out = {}
    n_cases = 0
    for rep in range(6):
        for kind in PATTERN_KINDS:
            pat = random_pattern(rng, kind, max_grid=6, max_block=5)
            blocks = random_blocks(rng, pat)
            a = bt.struct_assemble(pat, blocks)
            t = bt.mat_to_tensor(a, pat)
            tu = bt.mat_to_tensor(a, pat, weighted=False)
            back = bt.tensor_to_mat(t, pat)
            cells, offs = flat_placements(pat)
            key = f"c{n_cases}"
            out[key + "_dims"] = np.array([pat.ell, pat.q, pat.m, pat.n], np.int64)
            out[key + "_cells"] = cells
            out[key + "_offs"] = offs
            out[key + "_a"] = a
            out[key + "_t"] = t
            out[key + "_tu"] = tu
            out[key + "_back"] = back
            coeffs = rng.standard_normal(pat.p)
            out[key + "_coeffs"] = coeffs
            out[key + "_scalars"] = bt.struct_scalars(pat, coeffs)
            n_cases += 1
    out["n_cases"] = np.array(n_cases)
    np.savez_compressed(os.path.join(OUT, "maps.npz"), **out)


def cp_cases():
    out = {}
    # reference test cases (test_decomp.py:154-174) with the reference init
    rng = np.random.default_rng(10)
    t = np.einsum("i,j,k->ijk", rng.standard_normal(4), rng.standard_normal(6), rng.standard_normal(3))
    res = bt.cp_als(t, 1)
    out.update(rank1_t=t, rank1_fit=res.fit, rank1_x=res.rep.x, rank1_y=res.rep.y,
               rank1_z=res.rep.z, rank1_iters=res.n_iters)
    t = np.random.default_rng(12).standard_normal((2, 5, 3))
    res = bt.cp_als(t, 4, max_iters=200)
    out.update(pad_t=t, pad_fit=res.fit, pad_hist=np.array(res.fit_history),
               pad_init=np.array(0))
    init = bt_decomp._cp_init(t, 4)
    out.update(pad_init0=init[0], pad_init1=init[1], pad_init2=init[2])
    # C1 at full size with the N(0,1) seed-0 init
    pat, a = oc.c1_inputs()
    pat_ref = bt.build_pattern("toeplitz", 32, 32, 32, 32, block_symmetric=True)
    a_ref = bt.struct_assemble(pat_ref, oc.c1_blocks())
    assert np.array_equal(a, a_ref)
    t = bt.mat_to_tensor(a_ref, pat_ref)
    init = oc.normal_init(t.shape, 8, 0)
    saved = with_init(init)
    try:
        res = bt.cp_als(t, 8, 50, 0.0)
    finally:
        bt_decomp._cp_init = saved
    ks = bt.kron_sum_from_kruskal(res.rep, pat_ref)
    relerr = bt.error_fro(a_ref, ks)
    rhs = np.random.default_rng(1001).standard_normal((1024, 16))
    mv = np.stack([bt.matvec(ks, rhs[:, c]) for c in range(16)], axis=1)
    cnt = bt.FlopCounter()
    bt.matvec(ks, rhs[:, 0], cnt)
    out.update(c1_a_sha=sha(a_ref), c1_t=t, c1_fit=res.fit, c1_hist=np.array(res.fit_history),
               c1_x=res.rep.x, c1_y=res.rep.y, c1_z=res.rep.z, c1_relerr=relerr,
               c1_coeffs=ks.coeffs, c1_terms=ks.terms, c1_rhs=rhs, c1_mv=mv,
               c1_flops_per_rhs=cnt.flops)
    # a mid-size random CP case (R > some extents excluded): shapes like C4/C5
    rng = np.random.default_rng(77)
    for name, dims, r, iters in (("mid", (24, 20, 28), 5, 15), ("odd", (17, 9, 13), 3, 12)):
        t = rng.standard_normal(dims)
        init = oc.normal_init(dims, r, 5)
        saved = with_init(init)
        try:
            res = bt.cp_als(t, r, iters, 0.0)
        finally:
            bt_decomp._cp_init = saved
        out.update({f"{name}_t": t, f"{name}_r": r, f"{name}_iters": iters,
                    f"{name}_fit": res.fit, f"{name}_hist": np.array(res.fit_history),
                    f"{name}_x": res.rep.x, f"{name}_y": res.rep.y, f"{name}_z": res.rep.z})
    # C5 recipe at reduced size (K-slab regeneration semantics checked in tests)
    i, j, k, r = 48, 40, 32, 6
    x = oc.c5_tensor(i, j, k, r)
    init = oc.normal_init((i, j, k), r, 1003)
    saved = with_init(init)
    try:
        res = bt.cp_als(x, r, 10, 0.0)
    finally:
        bt_decomp._cp_init = saved
    out.update(c5s_t=x, c5s_dims=np.array([i, j, k, r]), c5s_fit=res.fit,
               c5s_hist=np.array(res.fit_history), c5s_x=res.rep.x, c5s_y=res.rep.y,
               c5s_z=res.rep.z)
    np.savez_compressed(os.path.join(OUT, "cp.npz"), **out)


def tucker_cases():
    out = {}
    rng = np.random.default_rng(31)
    n = 0
    for dims in ((3, 5, 2), (4, 4, 3), (6, 9, 5), (5, 3, 7)):
        t = rng.standard_normal(dims)
        ranks = random_ranks(rng, dims)
        rep = bt.hosvd(t, ranks)
        out.update({f"h{n}_t": t, f"h{n}_ranks": np.array(ranks), f"h{n}_core": rep.core,
                    f"h{n}_u0": rep.factors[0], f"h{n}_u1": rep.factors[1],
                    f"h{n}_u2": rep.factors[2]})
        n += 1
    out["n_hosvd"] = np.array(n)
    # svd_truncated sign convention + _mode_basis completion (decomp.py:149-234)
    a = rng.standard_normal((7, 5))
    u, s, v = bt.svd_truncated(a, 3)
    out.update(svd_a=a, svd_u=u, svd_s=s, svd_v=v)
    wide = rng.standard_normal((6, 3))
    out.update(mb_a=wide, mb_u=bt_decomp._mode_basis(wide, 5))
    # C2 at reduced size: s = 64 Hankel (32, 127, 32), ranks (32, 40, 32)
    params = oc.c2_markov(state=60, io=8, count=127, seed=1)
    seq = bt.MarkovSequence(params=params)
    pat, blocks = bt.hankel_pattern_from_markov(seq)
    w = np.sqrt(np.asarray(pat.counts, dtype=np.float64))
    t = np.transpose(blocks, (1, 0, 2)).copy() * w[None, :, None]
    _, t_mine = oc.c2_tensor(params)
    assert np.array_equal(t, t_mine)
    rep = bt.hosvd(t, [8, 40, 8])
    blr = bt.blr_from_tucker(rep, pat)
    rhs = np.random.default_rng(1002).standard_normal((pat.shape[1], 4))
    mv = np.stack([bt.matvec(blr, rhs[:, c]) for c in range(4)], axis=1)
    cnt = bt.FlopCounter()
    bt.matvec(blr, rhs[:, 0], cnt)
    out.update(c2s_params=params, c2s_t=t, c2s_core=rep.core, c2s_u=rep.factors[0],
               c2s_v=rep.factors[1], c2s_w=rep.factors[2], c2s_mid=blr.middles,
               c2s_rhs=rhs, c2s_mv=mv, c2s_flops=cnt.flops)
    # C3 at reduced size: 6x6 grid (n = 36), 10 lags; tucker_partial shared + SPSD
    pat3, blocks3, t3 = oc.c3_tensor(side=6, lags=10)
    pat_ref = bt.build_pattern("toeplitz", 10, 10, 36, 36, block_symmetric=True)
    rep = bt.tucker_partial(t3, [8, 4, 8], shared=(1, 3))
    sp = bt.spsd_compress_blocks(pat_ref, blocks3, 8)
    out.update(c3s_t=t3, c3s_blocks=blocks3, c3s_core=rep.core, c3s_u=rep.factors[0],
               c3s_v=rep.factors[1], c3s_spsd_u=sp.basis, c3s_spsd_blocks=sp.blocks,
               c3s_trace=sp.trace())
    np.savez_compressed(os.path.join(OUT, "tucker.npz"), **out)


def rep_cases():
    """Converters + matvec + FlopCounter on random patterns (test_reconstruct.py)."""
    rng = np.random.default_rng(555)
    out = {}
    n = 0
    for rep_i in range(3):
        for kind in PATTERN_KINDS:
            pat = random_pattern(rng, kind, max_grid=6, max_block=5)
            a = bt.struct_assemble(pat, random_blocks(rng, pat))
            t = bt.mat_to_tensor(a, pat)
            ranks = random_ranks(rng, t.shape)
            tk = bt.hosvd(t, ranks)
            ks = bt.kron_sum_from_tucker(tk, pat)
            blr = bt.blr_from_tucker(tk, pat)
            x = rng.standard_normal(pat.shape[1])
            c1, c2 = bt.FlopCounter(), bt.FlopCounter()
            y_k = bt.matvec(ks, x, c1)
            y_b = bt.matvec(blr, x, c2)
            cells, offs = flat_placements(pat)
            key = f"r{n}"
            out.update({key + "_dims": np.array([pat.ell, pat.q, pat.m, pat.n]),
                        key + "_cells": cells, key + "_offs": offs, key + "_core": tk.core,
                        key + "_u": tk.factors[0], key + "_v": tk.factors[1],
                        key + "_w": tk.factors[2], key + "_kc": ks.coeffs, key + "_kt": ks.terms,
                        key + "_bl": blr.left, key + "_br": blr.right, key + "_bm": blr.middles,
                        key + "_x": x, key + "_yk": y_k, key + "_yb": y_b,
                        key + "_fk": c1.flops, key + "_fb": c2.flops,
                        key + "_dk": bt.densify(ks), key + "_a": a})
            # CP-based converters where the rank fits the block extents
            r = int(min(pat.m, pat.n, 2))
            init = oc.normal_init(t.shape, r, 9)
            saved = with_init(init)
            try:
                res = bt.cp_als(t, r, 8, 0.0)
            finally:
                bt_decomp._cp_init = saved
            kf = bt.kron_sum_from_kruskal(res.rep, pat)
            out.update({key + "_cx": res.rep.x, key + "_cy": res.rep.y, key + "_cz": res.rep.z,
                        key + "_kfc": kf.coeffs, key + "_kft": kf.terms})
            if pat.p >= r:
                kq = bt.kron_sum_from_kruskal(res.rep, pat, split="qr")
                out.update({key + "_kqc": kq.coeffs, key + "_kqt": kq.terms})
            bk = bt.blr_from_kruskal(res.rep, pat)
            out.update({key + "_bkl": bk.left, key + "_bkr": bk.right, key + "_bkm": bk.middles})
            n += 1
    out["n_cases"] = np.array(n)
    np.savez_compressed(os.path.join(OUT, "reps.npz"), **out)


def psf_cases():
    out = {}
    rng = np.random.default_rng(8)
    for k in (3, 5, 7):
        psf = rng.standard_normal((k, k, k))
        x, mlp = bt.psf_weighted_tensor(psf)
        out[f"psf{k}"] = psf
        out[f"x{k}"] = x
        if k <= 5:
            out[f"dense{k}"] = bt.blur_operator_dense(psf)
    # C4 recipe at K = 7 (grid == K so the reference builder applies)
    psf = oc.c4_psf(7)
    x, mlp = bt.psf_weighted_tensor(psf)
    out["c4s_psf"] = psf
    out["c4s_x"] = x
    t = x[0, :, :, :, 0]
    init = oc.normal_init(t.shape, 3, 2)
    saved = with_init(init)
    try:
        res = bt.cp_als(t, 3, 30, 0.0)
    finally:
        bt_decomp._cp_init = saved
    out.update(c4s_fit=res.fit, c4s_hist=np.array(res.fit_history), c4s_cx=res.rep.x,
               c4s_cy=res.rep.y, c4s_cz=res.rep.z)
    # multilevel terms from the (diagonal-core) Tucker form of the CP result,
    # densified by the reference -> anchors ml_kron_sum_from_kruskal + ml_matvec
    r = res.rep.rank
    core = np.zeros((1, r, r, r, 1))
    for i in range(r):
        core[0, i, i, i, 0] = 1.0
    tk = bt.TuckerRep(core=core, factors=(None, res.rep.x, res.rep.y, res.rep.z, None))
    terms = bt.ml_kron_sum_from_tucker(tk, mlp)
    dense = bt.ml_kron_densify(terms)
    out["c4s_dense_cp"] = dense
    vols = np.random.default_rng(1004).standard_normal((7**3, 3))
    out["c4s_vols"] = vols
    out["c4s_mv"] = dense @ vols
    np.savez_compressed(os.path.join(OUT, "psf.npz"), **out)


def spd_cases():
    """psd.py:205-271 spd_compress and decomp.py:196 cholesky on seeded SPD
    block-Toeplitz inputs (oracle/configs.spd_toeplitz) at every rank."""
    out = {}
    for case, (seed, ell, nb) in enumerate(((21, 4, 5), (22, 3, 8), (23, 6, 3))):
        pat_o, a = oc.spd_toeplitz(seed, ell, nb)
        pat = bt.build_pattern("toeplitz", ell, ell, nb, nb)
        out[f"s{case}_a"] = a
        for r in range(1, nb + 1):
            rep = bt.spd_compress(a, pat, r)
            key = f"s{case}_r{r}"
            out[key + "_dense"] = rep.densify()
            out[key + "_basis"] = rep.remainder.basis
            out[key + "_blocks"] = rep.remainder.blocks
            if r == 1:
                out[f"s{case}_chol"] = rep.chol
                out[f"s{case}_rem_cells"] = np.concatenate(rep.remainder.pattern.placements)
                out[f"s{case}_rem_counts"] = np.array(rep.remainder.pattern.counts)
                out[f"s{case}_rem_class"] = np.array(rep.remainder.pattern.structure_class)
    # block diagonal input: empty remainder
    g = np.random.default_rng(24).standard_normal((4, 4))
    t0 = g @ g.T + 4 * np.eye(4)
    cells = np.column_stack([np.arange(3), np.arange(3)])
    pat = bt.BlockPattern(ell=3, q=3, m=4, n=4, placements=(cells,), structure_class="diagonal")
    a = bt.struct_assemble(pat, np.stack([t0]))
    rep = bt.spd_compress(a, pat, 2)
    out.update(bd_a=a, bd_dense=rep.densify(), bd_chol=rep.chol)
    g = np.random.default_rng(25).standard_normal((7, 7))
    out["chol_in"] = g @ g.T + 7 * np.eye(7)
    out["chol_out"] = bt.cholesky(out["chol_in"])
    np.savez_compressed(os.path.join(OUT, "spd.npz"), **out)


def detect_cases():
    """blocks.py:266-329 detect_pattern on oracle/configs.detect_cases()."""
    out = {}
    meta = []
    for name, a, m, n, tol in oc.detect_cases():
        pat, reps = bt.detect_pattern(a, m, n, tol=tol)
        cells, offs = flat_placements(pat)
        out[f"{name}_cells"] = cells
        out[f"{name}_offs"] = offs
        out[f"{name}_reps"] = np.stack(reps)
        meta.append({"name": name, "structure_class": pat.structure_class})
    np.savez_compressed(os.path.join(OUT, "detect.npz"), **out)
    with open(os.path.join(OUT, "detect.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def container_cases():
    """container.py writer output for every representation kind, from seeded
    inputs; the device reader/writer must reproduce these bytes."""
    from blockten.decomp import tucker_partial
    from blockten.multilevel import MultilevelTuckerRep, ml_mat_to_tensor, ml_tensor_to_mat
    from blockten.psd import spd_compress, spsd_compress
    from blockten.reconstruct import TuckerBlockRep, blr_from_tucker, kron_sum_from_tucker

    root = os.path.join(OUT, "containers")
    os.makedirs(root, exist_ok=True)
    rng = np.random.default_rng(61)
    pat = bt.build_pattern("toeplitz", 4, 4, 3, 5)
    a = bt.struct_assemble(pat, rng.standard_normal((pat.p, 3, 5)))
    tk = bt.hosvd(bt.mat_to_tensor(a, pat), [3, 5, 4])
    bt.container_write(os.path.join(root, "kron_sum.btc"), kron_sum_from_tucker(tk, pat),
                       seed=7, ranks=(3, 5, 4))
    bt.container_write(os.path.join(root, "blr.btc"), blr_from_tucker(tk, pat))
    patb = bt.build_pattern("banded", 5, 5, 2, 3, band=1)
    ab = bt.struct_assemble(patb, rng.standard_normal((patb.p, 2, 3)))
    tkp = tucker_partial(bt.mat_to_tensor(ab, patb), [None, 3, None])
    bt.container_write(os.path.join(root, "tucker_raw.btc"), TuckerBlockRep(pattern=patb, tucker=tkp))
    pat_s, a_s = oc.spd_toeplitz(62, 3, 4)
    pat_s = bt.build_pattern("toeplitz", 3, 3, 4, 4)
    bt.container_write(os.path.join(root, "spsd.btc"), spsd_compress(a_s, pat_s, 3))
    bt.container_write(os.path.join(root, "spd.btc"), spd_compress(a_s, pat_s, 2))
    inner = bt.build_pattern("banded", 3, 3, 2, 2, band=1)
    outer = bt.build_pattern("hankel", 2, 2, inner.shape[0], inner.shape[1])
    mlp = bt.MultilevelPattern(levels=(outer, inner))
    tm = rng.standard_normal(mlp.dims)
    am = ml_tensor_to_mat(tm, mlp)
    tkm = bt.hosvd(ml_mat_to_tensor(am, mlp), [2, 3, 3, 2])
    bt.container_write(os.path.join(root, "multilevel.btc"), MultilevelTuckerRep(pattern=mlp, tucker=tkm))


ERA_CASES = (  # (name, system seed, d, n_out, n_in, s, ranks, order, tera)
    ("full", 71, 6, 2, 2, 20, (2, 39, 2), 6, False),
    ("cut", 72, 5, 3, 2, 16, (3, 12, 2), 5, False),
    ("tera", 73, 4, 3, 3, 12, (2, 0, 2), 4, True),
    ("siso", 74, 2, 1, 1, 10, (1, 19, 1), 2, False),
)


def era_cases():
    """apps.py:153-237 era_identify_compressed on seeded stable systems."""
    from blockten.apps import LtiSystem, era_identify_compressed, markov_from_lti

    out = {}
    for name, seed, d, no, ni, s, ranks, order, tera in ERA_CASES:
        a, b, c = oc.era_system(seed, d, no, ni)
        seq = markov_from_lti(LtiSystem(a=a, b=b, c=c), 2 * s - 1)
        res = era_identify_compressed(seq, ranks, order, tera=tera)
        out[f"{name}_params"] = seq.params
        out[f"{name}_sv"] = res.sing_vals
        out[f"{name}_eig"] = np.linalg.eigvals(res.system.a)
        out[f"{name}_markov"] = markov_from_lti(res.system, 2 * s - 1).params
        out[f"{name}_reduced"] = res.reduced_hankel
        out[f"{name}_u"] = res.basis_left
        out[f"{name}_w"] = res.basis_right
        out[f"{name}_approx"] = res.hankel_approx()
    np.savez_compressed(os.path.join(OUT, "era.npz"), **out)


if __name__ == "__main__":
    np.seterr(all="ignore")
    patterns()
    maps()
    cp_cases()
    tucker_cases()
    rep_cases()
    psf_cases()
    spd_cases()
    detect_cases()
    container_cases()
    era_cases()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
