#!/usr/bin/env python
"""bt200 benchmark -- BASELINE.json metric "CP-ALS MTTKRP GFLOP/s & ST-HOSVD
time ...; % FP64/HBM roofline".

Headline workload (config C5, the largest config that fits one B200):
CP-ALS at rank 64 for 10 sweeps (tol 0: exactly 10) on the 4096x4096x1024
fp64 tensor [[A0,B0,C0]] + 1e-4 noise (seed 3, init seed 1003), built on the
GPU.  One *step* = one full ``cp_als(X, 64, max_iters=10, tol=0.0)`` call
(fro norm, 10 sweeps, fits, final KruskalRep).  ``value`` = reference-
equivalent MTTKRP GFLOP/s = 10 sweeps x 3 modes x 2*I*J*K*R / step time
(the reference's ``unfold @ khatri_rao`` count, decomp.py:385-387).  The
tensor (137 GB) is far larger than L2, so no flush is needed between steps.

Also reported: roofline of the dominant kernel (the P = X x3 C DMMA GEMM,
timed live with CUDA events inside the library), the e2e number through the
public API with host buffers, the CPU reference (oracle port, all host
threads) on a bounded mode-3 slab, clocks, launch counts, and secondary
configs (C3 ST-HOSVD+HOOI time, C1/C2/C4 pipelines, gather stand-in GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

I_, J_, K_, R_, ITERS = 4096, 4096, 1024, 64, 10
CPU_SLAB = 8          # mode-3 rows in the bounded CPU sample
REF_SLAB = 4          # rows per step for --impl reference


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="bt200", choices=["bt200", "reference"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--small", action="store_true", help="reduced C5 (smoke runs)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------


class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.dev = dev_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *exc):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        import numpy as np

        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# FP64 peak (DMMA) -- the roofline denominator MEASURED_PEAKS.json lacks
# ---------------------------------------------------------------------------


def fp64_peaks(torch):
    import ctypes as C

    from paper_2105_01170_b200 import _native as N

    lib = N.load()
    sink = torch.zeros(8192, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    out = {}
    for name, fn in (("dmma", lib.bt_peak_dmma), ("dfma", lib.bt_peak_dfma)):
        fl = C.c_double()
        fn(2000, 148 * 8, 256, sink.data_ptr(), C.byref(fl), st)
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(40000, 148 * 8, 256, sink.data_ptr(), C.byref(fl), st)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, fl.value / e0.elapsed_time(e1) / 1e9)
        out[name] = best
    return out


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of decomp.py:344-410, all host threads)
# ---------------------------------------------------------------------------


def cpu_slab_sweep(x_slab, init, threads):
    from oracle import port

    t0 = time.perf_counter()
    port.cp_als(x_slab, init[0].shape[1], max_iters=1, tol=0.0,
                init=lambda _t, _r: [f.copy() for f in init])
    return time.perf_counter() - t0


def build_slab_host(torch, k_rows):
    from paper_2105_01170_b200 import configs

    xs = configs.c5_build(I_, J_, K_, R_, k_slab=(0, k_rows))
    host = xs.cpu().numpy()
    del xs
    torch.cuda.empty_cache()
    return host


def run_reference(args, rank, world):
    nproc = os.cpu_count() or 1
    if rank != 0:
        return
    import numpy as np

    from paper_2105_01170_b200 import configs

    if args.small:
        global I_, J_, K_
        I_, J_, K_ = 512, 512, 128
    from oracle import configs as oc

    host = oc.c5_tensor(I_, J_, K_, R_, k_slab=(0, REF_SLAB))   # numpy generator, untimed
    init = configs.normal_init((I_, J_, K_), R_, 1003)
    init = [init[0], init[1], init[2][:REF_SLAB].copy()]
    for _ in range(args.warmup):
        cpu_slab_sweep(host, init, nproc)
    times = [cpu_slab_sweep(host, init, nproc) for _ in range(args.steps)]
    per = float(np.mean(times))
    gflops = 6 * I_ * J_ * REF_SLAB * R_ / per / 1e9
    line = {
        "metric": "CP-ALS MTTKRP GFLOP/s (reference-equivalent 6*I*J*K*R per sweep)",
        "value": gflops, "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"C5 CP-ALS R={R_} one sweep on a {I_}x{J_}x{REF_SLAB} mode-3 slab "
                               f"of the {I_}x{J_}x{K_} tensor (bounded CPU sample)"},
        "cpu_baseline": {"value": gflops, "unit": "GFLOP/s", "cores": nproc, "kind": "port",
                         "sample": f"1 ALS sweep on a {I_}x{J_}x{REF_SLAB} slab per step; "
                                   "numpy restatement of decomp.py:344-410 (oracle/port.py), "
                                   "OpenBLAS threads = all cores, einsum fit single-threaded"},
        "e2e": {"value": gflops, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# bt200 arm
# ---------------------------------------------------------------------------


def local_device(torch):
    """This rank's GPU: LOCAL_RANK (one process per GPU), folded onto the
    visible devices so the gloo test hook can stack ranks on one GPU."""
    n = max(torch.cuda.device_count(), 1)
    return int(os.environ.get("LOCAL_RANK", 0)) % n


def timed(torch, fn, steps, warmup):
    """Secondary-config timing: median over `steps` calls, each bracketed by
    CUDA events with a synchronize.  The latency-bound configs (C1, C4 CP) take
    11 calls: single calls on the box show rare 20-500 ms host-side stalls with
    SM/memory clocks steady at max (tools/probe_spikes2.py), so the median, not
    the mean, is the statistic."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    log(f"[bench] timed: {[round(t, 3) for t in ts]} ms")
    ts.sort()
    return ts[len(ts) // 2] if len(ts) % 2 else 0.5 * (ts[len(ts) // 2 - 1] + ts[len(ts) // 2])


def extras_run(torch, budget_s=240.0):
    """Secondary configs, each device resident, timed with CUDA events."""
    import numpy as np

    import paper_2105_01170_b200 as bt
    from paper_2105_01170_b200 import configs, decomp, multilevel, reconstruct

    out = {}
    t_start = time.time()

    def left():
        return budget_s - (time.time() - t_start)

    # C3: ST-HOSVD (shared 1/3) + 5 HOOI sweeps -> (64, 32, 64), SPSD blocks
    try:
        pat3, t3 = configs.c3_build()
        torch.cuda.synchronize()

        def c3():
            rep = decomp.st_hosvd(t3, [64, 32, 64], shared=(1, 3))
            return decomp.hooi(t3, rep, 5, shared=(1, 3))

        ms = timed(torch, c3, 3, 1)
        rep = c3()
        ms_st = timed(torch, lambda: decomp.st_hosvd(t3, [64, 32, 64], shared=(1, 3)), 3, 0)
        out["c3_st_hosvd_ms"] = ms_st
        out["c3_st_hosvd_plus_5_hooi_ms"] = ms
        from paper_2105_01170_b200.tensor import fro_norm_dev

        out["c3_core_norm_ratio"] = fro_norm_dev(rep.core) / fro_norm_dev(t3)
        # C3's two outputs: the PSD-preserving SpsdRep from the
        # unweighted blocks (psd.py:164-187) and the BLR operator of the
        # (64, 32, 64) Tucker (reconstruct.py:229-240) with its matvec
        from paper_2105_01170_b200 import psd

        eta3 = torch.tensor(pat3.counts, dtype=torch.float64, device="cuda")
        blocks3 = (t3.permute(1, 0, 2) / eta3.sqrt()[:, None, None]).contiguous()
        out["c3_spsd_ms"] = timed(torch, lambda: psd.spsd_compress_blocks(pat3, blocks3, 64), 3, 1)
        del blocks3
        torch.cuda.empty_cache()
        out["c3_blr_from_tucker_ms"] = timed(torch, lambda: reconstruct.blr_from_tucker(rep, pat3), 3, 1)
        blr3 = reconstruct.blr_from_tucker(rep, pat3)
        rhs3 = torch.from_numpy(np.random.default_rng(1003).standard_normal((pat3.shape[1], 16))).cuda()
        ms_mv = timed(torch, lambda: reconstruct.matvec(blr3, rhs3), 3, 1)
        out["c3_blr_matvec16_ms"] = ms_mv
        out["c3_blr_matvec_tflops"] = 16 * reconstruct.flops_blr(pat3, 64, 64) / ms_mv / 1e9
        del blr3, rhs3
        # K7 / K9 kernel rooflines at C3: the mode-1 unfolding Gram (SYRK over
        # the 1024 x 524288 unfolding, unique-half work n(n+1)N/n flops, SURVEY
        # 8d) and the first TTM t x1 U^T (2 r N flops)
        from paper_2105_01170_b200 import _linalg
        from paper_2105_01170_b200.tensor import ttm_dev

        n1 = int(t3.shape[0])
        big_n = t3.numel() // n1
        ms_g = timed(torch, lambda: _linalg.unfold_gram_dev(t3, 1), 3, 1)
        u = rep.factors[0] if torch.is_tensor(rep.factors[0]) else torch.from_numpy(
            np.ascontiguousarray(rep.factors[0])).cuda()
        ms_t = timed(torch, lambda: ttm_dev(t3, 1, u, int(u.shape[1]), transpose=True), 3, 1)
        out["c3_gram_mode1_ms"] = ms_g
        out["c3_gram_mode1_tflops"] = n1 * (n1 + 1) * big_n / ms_g / 1e9
        out["c3_ttm_mode1_ms"] = ms_t
        out["c3_ttm_mode1_tflops"] = 2.0 * int(u.shape[1]) * t3.numel() / ms_t / 1e9
        del t3, rep
        torch.cuda.empty_cache()
    except Exception as exc:  # pragma: no cover - reported, not fatal
        out["c3_error"] = repr(exc)[:300]
    # C1 full pipeline
    if left() > 0:
        try:
            pat, a = configs.c1_matrix()
            init = configs.normal_init((32, 32, 32), 8, 0)
            rhs = torch.from_numpy(np.random.default_rng(1001).standard_normal((1024, 16))).cuda()

            def c1():
                t = bt.mat_to_tensor(a, pat)
                saved = decomp._cp_init
                decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
                try:
                    res = decomp.cp_als(t, 8, 50, 0.0)
                finally:
                    decomp._cp_init = saved
                ks = reconstruct.kron_sum_from_kruskal(res.rep, pat)
                err = reconstruct.error_fro(a, ks)
                y = reconstruct.matvec(ks, rhs)
                return res, err, y

            out["c1_pipeline_ms"] = timed(torch, c1, 11, 3)
            res, err, _ = c1()
            out["c1_fit"] = res.fit
            out["c1_relerr"] = err
            # the 50-sweep CP-ALS alone (fused one-CTA kernel), per sweep
            t1 = bt.mat_to_tensor(a, pat)
            t1 = t1 if torch.is_tensor(t1) else torch.from_numpy(t1).cuda()

            def c1cp():
                saved = decomp._cp_init
                decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
                try:
                    return decomp.cp_als(t1, 8, 50, 0.0)
                finally:
                    decomp._cp_init = saved

            ms_cp = timed(torch, c1cp, 11, 3)
            out["c1_cp_ms"] = ms_cp
            out["c1_cp_us_per_sweep"] = ms_cp * 1e3 / 50
        except Exception as exc:  # pragma: no cover
            out["c1_error"] = repr(exc)[:300]
    # C4: CP R=16 x 30 on the 255^3 weighted PSF + multilevel matvec on 32 volumes
    if left() > 0:
        try:
            x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(),
                                                    grid=128)
            x3 = x.reshape(255, 255, 255)
            init = configs.normal_init((255, 255, 255), 16, 2)

            def c4cp():
                saved = decomp._cp_init
                decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
                try:
                    return decomp.cp_als(x3, 16, 30, 0.0)
                finally:
                    decomp._cp_init = saved

            out["c4_cp_ms"] = timed(torch, c4cp, 11, 3)
            res = c4cp()
            out["c4_fit"] = res.fit
            terms = multilevel.ml_kron_sum_from_kruskal(res.rep, mlp)
            stacks = multilevel.stack_level_mats(terms)
            vols = torch.from_numpy(np.random.default_rng(1004).standard_normal((128**3, 32))).cuda()
            ms = timed(torch, lambda: multilevel.ml_matvec(terms, vols, stacks), 2, 1)
            out["c4_matvec32_ms"] = ms
            out["c4_matvec_tflops"] = 16 * 32 * 3 * 2 * 128**4 / ms / 1e9
            del vols
            torch.cuda.empty_cache()
        except Exception as exc:  # pragma: no cover
            out["c4_error"] = repr(exc)[:300]
    # C2: HOSVD (32, 400, 32) of the weighted Hankel tensor + BLR matvec on 64 RHS
    if left() > 0:
        try:
            params = configs.c2_markov()
            pat2, t2 = configs.c2_build(params)

            def c2():
                return decomp.hosvd(t2, [32, 400, 32])

            out["c2_hosvd_ms"] = timed(torch, c2, 3, 1)
            rep = c2()
            blr = reconstruct.blr_from_tucker(rep, pat2)
            rhs = torch.from_numpy(np.random.default_rng(1002).standard_normal((32768, 64))).cuda()
            ms = timed(torch, lambda: reconstruct.matvec(blr, rhs), 2, 1)
            out["c2_matvec64_ms"] = ms
            out["c2_matvec_tflops"] = 64 * reconstruct.flops_blr(pat2, 32, 32) / ms / 1e9
        except Exception as exc:  # pragma: no cover
            out["c2_error"] = repr(exc)[:300]
    # gather / scatter stand-in (A 32768^2 = 8.6 GB)
    if left() > 0:
        try:
            patg, blocks = configs.gather_standin()
            a = bt.struct_assemble(patg, torch.from_numpy(blocks).cuda())
            del blocks
            ms_g = timed(torch, lambda: bt.mat_to_tensor(a, patg), 3, 1)
            t = bt.mat_to_tensor(a, patg)
            ms_s = timed(torch, lambda: bt.tensor_to_mat(t, patg), 3, 1)
            nbytes = a.numel() * 8 + t.numel() * 8
            out["gather_standin_ms"] = ms_g
            out["gather_standin_gbs"] = nbytes / ms_g / 1e6
            out["scatter_standin_ms"] = ms_s
            out["scatter_standin_gbs"] = nbytes / ms_s / 1e6
            del t
            # detect_pattern (digest pass + bit-exact verify pass: A read twice)
            ms_d = timed(torch, lambda: bt.detect_pattern(a, patg.m, patg.n), 2, 1)
            pd, _ = bt.detect_pattern(a, patg.m, patg.n)
            out["detect_standin_ms"] = ms_d
            out["detect_standin_gbs"] = 2 * a.numel() * 8 / ms_d / 1e6
            out["detect_standin_classes"] = pd.p
            del a
            torch.cuda.empty_cache()
        except Exception as exc:  # pragma: no cover
            out["gather_error"] = repr(exc)[:300]
    return out


def extras_cpu(budget_s=120.0):
    """The reference path timed on the host beside each secondary config:
    the oracle port (numpy restatement of the reference, oracle/port.py) with
    all host threads, on bounded samples scaled to the full config where the
    full run would take minutes (stated per entry)."""
    import numpy as np

    from oracle import configs as oc
    from oracle import port

    out = {}
    t_start = time.time()

    def left():
        return budget_s - (time.time() - t_start)

    def clock(fn):
        t0 = time.perf_counter()
        r = fn()
        return (time.perf_counter() - t0) * 1e3, r

    try:   # C1 full pipeline, full size
        pat, a = oc.c1_inputs()
        init = oc.normal_init((32, 32, 32), 8, 0)
        rhs = np.random.default_rng(1001).standard_normal((1024, 16))

        def c1():
            t = port.gather(a, pat)
            res = port.cp_als(t, 8, 50, 0.0, init=lambda _t, _r: [f.copy() for f in init])
            coeffs, terms = port.kron_from_kruskal(res.x, res.y, res.z)
            err = np.linalg.norm(a - port.densify_kron(pat, coeffs, terms)) / np.linalg.norm(a)
            y = np.stack([port.matvec_kron(pat, coeffs, terms, rhs[:, j]) for j in range(16)], 1)
            return err, y

        out["c1_pipeline_ms"], _ = clock(c1)
        out["c1_sample"] = "full C1 pipeline (gather, 50 sweeps, Kron sum, error, 16 matvecs)"
    except Exception as exc:  # pragma: no cover
        out["c1_error"] = repr(exc)[:200]
    if left() > 0:
        try:   # C2 HOSVD full size; BLR matvec: 1 RHS x 64
            params = oc.c2_markov()
            pat2, t2 = oc.c2_tensor(params)
            ms, (core, fac) = clock(lambda: port.hosvd(t2, [32, 400, 32]))
            out["c2_hosvd_ms"] = ms
            left_, right_, mids = port.blr_from_tucker(core, fac, pat2.m, pat2.n)
            x = np.random.default_rng(1002).standard_normal(32768)
            ms1, _ = clock(lambda: port.matvec_blr(pat2, left_, right_, mids, x))
            out["c2_matvec64_ms"] = 64 * ms1
            out["c2_sample"] = "HOSVD full size; BLR matvec timed on 1 RHS, x64"
        except Exception as exc:  # pragma: no cover
            out["c2_error"] = repr(exc)[:200]
    if left() > 0:
        try:   # C3 ST-HOSVD on the first 64 lags (same u_k), x8
            _, _, t3 = oc.c3_tensor(side=32, lags=64, lag_scale=512)
            ms, _ = clock(lambda: port.st_hosvd_shared13(t3, 64, 32))
            out["c3_st_hosvd_ms"] = 8 * ms
            out["c3_sample"] = "ST-HOSVD on a (1024, 64, 1024) lag prefix, x8 (extrapolated)"
            del t3
        except Exception as exc:  # pragma: no cover
            out["c3_error"] = repr(exc)[:200]
    if left() > 0:
        try:   # C4 one sweep x30
            x4 = oc.c4_tensor().reshape(255, 255, 255)
            init4 = oc.normal_init((255, 255, 255), 16, 2)
            ms, _ = clock(lambda: port.cp_als(x4, 16, 1, 0.0, init=lambda _t, _r: init4))
            out["c4_cp_ms"] = 30 * ms
            out["c4_sample"] = "1 ALS sweep x30 (extrapolated)"
            del x4
        except Exception as exc:  # pragma: no cover
            out["c4_error"] = repr(exc)[:200]
    if left() > 0:
        try:   # gather stand-in: 8 of 128 block rows (2048 x 32768), x16
            nb, ell = 256, 128
            pat, blocks = oc.gather_standin(nb, ell)
            rows = 8
            sub = port.Pattern(rows, ell, nb, nb, tuple(c[c[:, 0] < rows] for c in pat.placements))
            sub = port.Pattern(rows, ell, nb, nb, tuple(c for c in sub.placements if len(c)))
            a = port.assemble(sub, [blocks[k] for k, c in enumerate(pat.placements)
                                    if np.any(c[:, 0] < rows)])
            ms, _ = clock(lambda: port.gather(a, sub))
            out["gather_standin_ms"] = (ell // rows) * ms
            out["gather_sample"] = "8 of 128 block rows (2048 x 32768), x16 (extrapolated)"
        except Exception as exc:  # pragma: no cover
            out["gather_error"] = repr(exc)[:200]
    out["cores"] = os.cpu_count()
    return out


def run_bt200(args, rank, world):
    import numpy as np
    import torch

    import paper_2105_01170_b200 as bt
    from paper_2105_01170_b200 import _dev, configs, decomp
    from paper_2105_01170_b200 import _native as N

    global I_, J_, K_
    if args.small:
        I_, J_, K_ = 512, 512, 128
    torch.cuda.set_device(local_device(torch))
    lib = N.load()
    peaks = fp64_peaks(torch)
    log(f"[bench] fp64 peaks (TFLOP/s): {peaks}")

    from paper_2105_01170_b200.parallel import (NativeCpOps, cp_als_sharded, shard_bounds,
                                                torch_allreduce)

    k0, k1 = shard_bounds(K_, world, rank)
    x = configs.c5_build(I_, J_, K_, R_, k_slab=(k0, k1))   # this rank's mode-3 slab
    init = configs.normal_init((I_, J_, K_), R_, 1003)
    init_dev = [torch.from_numpy(init[0]).cuda(), torch.from_numpy(init[1]).cuda(),
                torch.from_numpy(init[2][k0:k1].copy()).cuda()]
    f = [torch.empty_like(v) for v in init_dev]
    lam = torch.empty(R_, dtype=torch.float64, device="cuda")
    from paper_2105_01170_b200.decomp import cp_als_device
    phase = [0.0] * 4
    hist_holder = {}
    allreduce = torch_allreduce()

    # the sharded run's phase state (workspace, handle) is built once, outside
    # the timed steps; each step re-seeds the factors and re-runs init_local
    ops = NativeCpOps(x, R_, f[0], f[1], f[2], ITERS) if world > 1 else None

    def step():
        for k in range(3):
            f[k].copy_(init_dev[k])
        if world == 1:
            hist, n_it, conv = cp_als_device(x, R_, f, lam, ITERS, 0.0, "auto", 0.0, ws_holder(),
                                             phase_ms=phase)
        else:
            hist, n_it, conv = cp_als_sharded(ops, ITERS, 0.0, allreduce)
        hist_holder["h"] = hist

    ws_cache = {}

    def ws_holder():
        if "ws" not in ws_cache:
            import ctypes as C

            pb = N.CpProblem(_dev.ptr(x), I_, J_, k1 - k0, R_, 0.0)
            ws_cache["ws"] = _dev.workspace(lib.bt_cp_als_ws_bytes(C.byref(pb)))
        return ws_cache["ws"]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    phase_tot = [0.0] * 4
    l0 = lib.bt_launch_count()
    with Clocks(local_device(torch)) as clk:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
            phase_tot = [a + b for a, b in zip(phase_tot, phase)]
        e1.record()
        torch.cuda.synchronize()
    launches = (lib.bt_launch_count() - l0) / args.steps
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    ref_flops = ITERS * 6.0 * I_ * J_ * K_ * R_
    value = ref_flops / (ms / 1e3) / 1e9     # whole job: the global tensor, max-over-ranks time
    kloc = k1 - k0
    import ctypes as C

    variant = int(lib.bt_cp_tree_variant(C.byref(N.CpProblem(_dev.ptr(x), I_, J_, kloc, R_, 0.0))))
    per = args.steps * ITERS
    tree_ms = phase_tot[0] / per
    # the second full pass over X: the Q GEMM (+ mode-2 reduction, phase 1) on
    # the Q tree, the mode-3 GEMM (phase 2) on the P tree
    gemm2_ms = (phase_tot[1] if variant == 1 else phase_tot[2]) / per
    if tree_ms == 0.0:
        # sharded run: time this rank's mode-1 tree kernel and second GEMM separately (CUDA events)
        for k in range(3):
            f[k].copy_(init_dev[k])
        buf = ops.init_local()
        allreduce(buf)
        ops.init_finish(buf)
        tree_ms = timed(torch, lambda: ops.mttkrp(1), 3, 1)
        gemm2_ms = timed(torch, lambda: ops.mttkrp(2 if variant == 1 else 3), 3, 1)
    if ops is not None:
        ops.close()
    achieved = 2.0 * I_ * J_ * kloc * R_ / (tree_ms / 1e3) / 1e12
    peak = peaks["dmma"]
    fit = hist_holder["h"][-1]
    log(f"[bench] C5 step {ms:.1f} ms, tree variant {'Q' if variant else 'P'}, phases/sweep "
        f"{[round(v / per, 2) for v in phase_tot]} ms, fit {fit}")
    traffic = None
    ncu_file = "r02_ncu_c5q.json" if variant == 1 else "r01_ncu_c5.json"
    try:
        prof = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                           "profiles", ncu_file)))
        if prof["config"] == {"I": I_, "J": J_, "K": kloc, "R": R_}:
            tk = prof["tree_p_kernel"]
            traffic = tk["dram_bytes_read"] + tk["dram_bytes_write"]
    except (OSError, KeyError, ValueError):
        pass
    if variant == 1:
        phases = {"mode1_tree_no_p_store": tree_ms, "q_gemm_plus_mode2": gemm2_ms,
                  "mode3_from_q": phase_tot[2] / per, "solves_fit": phase_tot[3] / per}
        kname = ("tree_p_tma_kernel (X x3 C tiles by TMA, mode-1 reduction fused, no P store; "
                 "DMMA) -- Q dimension tree") if kloc > 256 else (
                 "gemm_at_tma_kernel (T = X[i]^T B batched over i, TMA + DMMA; mode 1 streamed "
                 "from T) -- Q dimension tree, short mode-3 slab")
        alg_bytes = 8.0 * I_ * J_ * kloc
        alg_note = "algorithmic X = "
    else:
        phases = {"p_tree": tree_ms, "mode2": phase_tot[1] / per, "mode3": gemm2_ms,
                  "solves_fit": phase_tot[3] / per}
        kname = "tree_p_tma_kernel (P = X x3 C by TMA, mode-1 reduction fused; DMMA) -- P dimension tree"
        alg_bytes = 8.0 * I_ * J_ * (kloc + R_)
        alg_note = "algorithmic X + P = "
    if world > 1:
        # sharded: only this rank's two full-pass kernels are timed (separately,
        # CUDA events); the sweep's other phases are not instrumented
        phases = {k: v for k, v in phases.items() if v > 0.0}
    result = {
        "metric": "CP-ALS MTTKRP GFLOP/s (reference-equivalent 6*I*J*K*R per sweep)",
        "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"C5: cp_als(X {I_}x{J_}x{K_} fp64 = [[A0,B0,C0]] + 1e-4 noise, "
                               f"R={R_}, max_iters={ITERS}, tol=0) per step; init seed 1003",
                   "global_batch": 1,
                   "parallelism": (f"mode-3 sharded x{world} (NCCL allreduce of MTTKRP partials "
                                   f"and R x R Grams)") if world > 1 else "1 GPU",
                   "l2": "inputs (137 GB) >> L2; no flush needed",
                   "per_sweep_ms": ms / ITERS, "final_fit": fit,
                   "executed_mttkrp_flops_per_sweep": 4.0 * I_ * J_ * K_ * R_,
                   "dimension_tree": "Q = X x1 A" if variant == 1 else "P = X x3 C",
                   "phase_ms_per_sweep": phases},
        "roofline": {"bound": "tensor", "kernel": kname,
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_note": ("bytes per launch, ncu dram__bytes_read+write "
                                      f"(profiles/{ncu_file}); {alg_note}{alg_bytes:.4g} B"),
                     "peak_source": "measured in this run: DMMA.8x8x4 chains on all SMs "
                                    "(MEASURED_PEAKS.json has no FP64 figure)",
                     "second_gemm": ("Q GEMM gemm_at_tma_kernel (+ mode-2 reduction)" if variant == 1
                                     else "mode-3 GEMM"),
                     "second_gemm_achieved": 2.0 * I_ * J_ * kloc * R_ / (gemm2_ms / 1e3) / 1e12},
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "fp64_peaks_tflops": dict(peaks),
    }
    if world > 1:
        result["comm"] = {"backend": os.environ.get("BT_DIST_BACKEND", "nccl"), "nranks": world,
                          "nccl_algo": os.environ.get("NCCL_ALGO"),
                          "nccl_proto": os.environ.get("NCCL_PROTO")}
    # the secondary configs get the whole HBM: the headline tensor is released
    # here and rebuilt on the device for the e2e run
    x = None
    ws_cache.clear()
    torch.cuda.empty_cache()
    # ---- N > 1: the C3 ST-HOSVD (+5 HOOI) sharded along the time mode over
    # all ranks (parallel.tucker_c3_distributed: NCCL allreduce of the mode-1
    # Grams, allgather of the projected mode-2 slabs), max over ranks
    if world > 1 and not args.no_extras:
        try:
            result["extras_distributed"] = c3_distributed(torch, world, rank)
        except Exception as exc:  # pragma: no cover
            result["extras_distributed"] = {"c3_error": repr(exc)[:300]}
    # ---- GPU secondary configs first: the host-side numpy work of the CPU
    # baselines below leaves OpenBLAS threads spinning, which would steal
    # the host cores the latency-bound configs (C1) launch from
    ex = None
    if not args.no_extras and rank == 0:
        ex = extras_run(torch)
        for key in ("c3_gram_mode1", "c3_ttm_mode1"):
            if isinstance(ex.get(key + "_tflops"), float):
                ex[key + "_frac_dmma"] = ex[key + "_tflops"] / peak
        result["extras"] = ex
    # ---- e2e: public API with host buffers (H2D of X + init, D2H of factors).
    # After the GPU secondary configs: pinning and unpinning 137 GB of host
    # memory left single-call latencies of the light configs (C1, C4) 10-30x
    # slow on some boxes when they ran after it
    ws_cache.clear()
    torch.cuda.empty_cache()
    if not args.no_e2e:
        try:
            x = configs.c5_build(I_, J_, K_, R_, k_slab=(k0, k1))
            result["e2e"] = e2e_run(args, torch, x, init, world, rank, k0, k1)
        except Exception as exc:  # pragma: no cover
            result["e2e"] = {"value": None, "unit": "GFLOP/s", "error": repr(exc)[:300]}
        x = None
    ws_cache.clear()
    torch.cuda.empty_cache()
    # ---- CPU baseline (bounded slab, rank 0, N=1)
    if not args.no_cpu and rank == 0 and world == 1:
        try:
            host = build_slab_host(torch, CPU_SLAB)
            init_s = [init[0], init[1], init[2][:CPU_SLAB].copy()]
            nproc = os.cpu_count() or 1
            secs = cpu_slab_sweep(host, init_s, nproc)
            full = secs * (K_ / CPU_SLAB)
            result["cpu_baseline"] = {
                "value": 6.0 * I_ * J_ * K_ * R_ / full / 1e9, "unit": "GFLOP/s",
                "cores": nproc, "kind": "port",
                "sample": f"1 ALS sweep of oracle/port.py cp_als (numpy restatement of "
                          f"decomp.py:344-410) on a {I_}x{J_}x{CPU_SLAB} mode-3 slab: {secs:.2f} s, "
                          f"extrapolated x{K_ // CPU_SLAB} to the full tensor; einsum fit single-threaded"}
            del host
        except Exception as exc:  # pragma: no cover
            result["cpu_baseline"] = {"value": None, "error": repr(exc)[:300]}
    if ex is not None and not args.no_cpu and world == 1:
        cpu = extras_cpu()
        result["extras_cpu_reference"] = cpu
        result["extras_speedup_vs_cpu"] = {
            k: cpu[k] / ex[k] for k in ("c1_pipeline_ms", "c2_hosvd_ms", "c2_matvec64_ms",
                                        "c3_st_hosvd_ms", "c4_cp_ms", "gather_standin_ms")
            if isinstance(cpu.get(k), float) and isinstance(ex.get(k), float) and ex[k] > 0}
    if rank == 0:
        print(json.dumps(result), flush=True)


def c3_distributed(torch, world, rank):
    """ST-HOSVD and ST-HOSVD + 5 HOOI of C3 on this rank's lag slab; CUDA
    events bracketed by barriers, max over ranks."""
    from paper_2105_01170_b200 import configs
    from paper_2105_01170_b200.parallel import shard_bounds, tucker_c3_distributed

    _, t = configs.c3_build()
    p0, p1 = shard_bounds(int(t.shape[1]), world, rank)
    x_local = t[:, p0:p1, :].contiguous()
    del t
    torch.cuda.empty_cache()
    out = {"workload": f"C3 (1024, 512, 1024) sharded along the 512 lags over {world} GPUs"}
    for key, sweeps in (("c3_st_hosvd_ms", 0), ("c3_st_hosvd_plus_5_hooi_ms", 5)):
        tucker_c3_distributed(x_local, 64, 32, hooi_sweeps=sweeps, p_offset=p0)   # warm-up
        torch.cuda.synchronize()
        torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tucker_c3_distributed(x_local, 64, 32, hooi_sweeps=sweeps, p_offset=p0)
        e1.record()
        torch.cuda.synchronize()
        tt = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        out[key] = float(tt.item())
    del x_local
    torch.cuda.empty_cache()
    return out


def e2e_run(args, torch, x_dev, init, world, rank, k0, k1):
    """Same metric through the public API with host buffers: every step copies
    this rank's X slab (and the init factors) host->device and reads the
    factors + fit history back (1 GPU: ``cp_als``; N GPUs:
    ``parallel.cp_als_distributed`` on mode-3 slabs)."""
    import numpy as np

    from paper_2105_01170_b200 import decomp, parallel

    nbytes = x_dev.numel() * 8
    try:
        host = torch.empty(tuple(x_dev.shape), dtype=torch.float64, pin_memory=True)
        pinned = True
    except RuntimeError:
        host = torch.empty(tuple(x_dev.shape), dtype=torch.float64)
        pinned = False
    host.copy_(x_dev)
    torch.cuda.synchronize()
    x_dev.set_()          # release the resident copy: the API call allocates its own
    torch.cuda.empty_cache()
    init_l = [init[0], init[1], init[2][k0:k1].copy()]
    saved = decomp._cp_init
    decomp._cp_init = lambda _t, _r: [v.copy() for v in init_l]

    def once():
        if world == 1:
            return decomp.cp_als(host, R_, ITERS, 0.0)
        return parallel.cp_als_distributed(host, R_, ITERS, 0.0, init=init_l)

    steps = max(1, min(args.steps, 5))
    try:
        once()  # warm-up
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            res = once()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        wall = (time.perf_counter() - t0) / steps * 1e3
    finally:
        decomp._cp_init = saved
    if world > 1:
        t = torch.tensor([ms, wall], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, wall = float(t[0]), float(t[1])
    h2d = nbytes + sum(v.nbytes for v in init_l)
    d2h = sum(np.asarray(v).nbytes for v in (res.rep.x, res.rep.y, res.rep.z)) + 8 * ITERS
    # give the 137 GB of pinned host memory back (torch caches pinned blocks):
    # held, it slows the launch-bound secondary configs timed after this
    del host
    import gc

    gc.collect()
    if hasattr(torch._C, "_host_emptyCache"):
        torch._C._host_emptyCache()
    return {"value": ITERS * 6.0 * I_ * J_ * K_ * R_ / (ms / 1e3) / 1e9, "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
            "ms_per_step": ms, "wall_ms_per_step": wall, "steps": steps,
            "host_buffer": "pinned" if pinned else "pageable",
            "path": ("paper_2105_01170_b200.cp_als(torch CPU tensor)" if world == 1 else
                     "paper_2105_01170_b200.parallel.cp_als_distributed(host slab per rank)") +
                    " -> H2D, device ALS, D2H of factors + fit history"}


def relaunch(args):
    """``--gpus N`` (N > 1) without a launcher: re-execute this script under
    ``torch.distributed.run`` with one process per GPU (the driver's own
    launch line), so ``n_gpus`` always equals the ranks that ran."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    log(f"[bench] --gpus {args.gpus} without a launcher: {' '.join(cmd)}")
    return subprocess.call(cmd)


def nccl_env():
    """Fixed reduction order (bit-reproducible sums across
    runs) and communicator evidence in the log."""
    os.environ.setdefault("NCCL_ALGO", "Ring")
    os.environ.setdefault("NCCL_PROTO", "Simple")
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")


def main():
    args = parse()
    if args.impl == "reference":
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
        os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    if world > 1:
        import torch
        import torch.distributed as dist

        if args.impl == "bt200":
            torch.cuda.set_device(local_device(torch))
            # BT_DIST_BACKEND=gloo is a test hook only: it runs the N > 1 code
            # path as several ranks on one GPU (host-mediated sums, so no
            # kernel waits on another rank's); the product path is NCCL
            backend = os.environ.get("BT_DIST_BACKEND", "nccl")
            if backend == "nccl":
                nccl_env()
                dist.init_process_group("nccl", device_id=torch.device("cuda", local_device(torch)))
            else:
                dist.init_process_group(backend)
            probe = torch.ones(1, device="cuda")
            dist.all_reduce(probe)          # creates the communicator now
            log(f"[bench] rank {rank}: {backend} communicator nranks={dist.get_world_size()} "
                f"(allreduce of ones = {int(probe.item())}), device cuda:{local_device(torch)}, "
                f"NCCL_ALGO={os.environ.get('NCCL_ALGO')} NCCL_PROTO={os.environ.get('NCCL_PROTO')}")
        else:
            dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_bt200(args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
