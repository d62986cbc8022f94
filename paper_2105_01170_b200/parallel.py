"""Multi-GPU CP-ALS: the tensor sharded along mode 3 across ranks (one process
per GPU, torch.distributed over NCCL for the sums).

Decomposition: A and B are replicated, C and the tensor are
row-sharded along mode 3.  The only exchanges per sweep are sums of
  * the mode-1 and mode-2 MTTKRP partials (I x R, J x R: each rank holds a
    K-slab, the MTTKRP sums over it),
  * the mode-3 solve's Gram / inner-product buffer (R x R + 2), because C's
    column norms, Gram and the fit need all rows,
  * the explicit-residual scalar (when the fit takes that route),
plus one sum of the local C Gram and ||X||^2 at start.  Everything else --
the pinv solves, normalisations, lambda, the fit -- is computed redundantly
and bit-identically on every rank (NCCL's allreduce returns the same bits to
all ranks, and the kernels are deterministic).

``cp_als_sharded`` is backend-agnostic: ``ops`` supplies the phases (the
native C-ABI here, ``NativeCpOps``; the CPU tests plug in a numpy stand-in)
and ``allreduce`` sums a buffer in place across ranks.
"""

from __future__ import annotations

import ctypes as C

from . import _dev
from . import _native as N
from .decomp import _FIT_MODES


class NativeCpOps:
    """The C-ABI CP phase API (include/bt200.h bt_cp_*) on device buffers."""

    def __init__(self, x_local, r, a, b, c_local, max_iters, fit="auto", norm_x=0.0):
        t = _dev.require_cuda()
        self.x = x_local
        I, J, K = (int(s) for s in x_local.shape)
        self.I, self.J, self.K, self.R = I, J, K, int(r)
        self.f = [a, b, c_local]
        self.lam = t.empty(self.R, dtype=t.float64, device="cuda")
        self.norm_x = float(norm_x)
        self.pb = N.CpProblem(_dev.ptr(x_local), I, J, K, self.R, 0.0)
        lib = N.load()
        self.ws = _dev.workspace(lib.bt_cp_state_ws_bytes(C.byref(self.pb)))
        self.h = C.c_void_p()
        N.call("bt_cp_state_create", C.byref(self.pb), _dev.ptr(a), _dev.ptr(b), _dev.ptr(c_local),
               _dev.ptr(self.lam), int(max_iters), _FIT_MODES[fit], _dev.ptr(self.ws),
               int(self.ws.numel()) * 8, _dev.stream(), C.byref(self.h))
        RR2 = self.R * self.R + 2
        self.buf = {"m1": _dev.empty((I, self.R)), "m2": _dev.empty((J, self.R)),
                    "m3": _dev.empty((max(K, 1), self.R)), "g": _dev.empty((RR2,)),
                    "init": _dev.empty((RR2,)), "r": _dev.empty((2,))}

    def init_local(self):
        N.call("bt_cp_init_local", self.h, self.norm_x, _dev.ptr(self.buf["init"]))
        return self.buf["init"]

    def init_finish(self, buf):
        N.call("bt_cp_init_finish", self.h, _dev.ptr(buf))

    def mttkrp(self, mode):
        out = self.buf[f"m{mode}"]
        N.call("bt_cp_mttkrp", self.h, int(mode), _dev.ptr(out))
        return out

    def solve(self, mode, m):
        N.call("bt_cp_solve", self.h, int(mode), _dev.ptr(m), _dev.ptr(self.buf["g"]))
        return self.buf["g"]

    def solve_finish(self, mode, it, g):
        N.call("bt_cp_solve_finish", self.h, int(mode), int(it), _dev.ptr(g))

    def residual(self):
        N.call("bt_cp_residual", self.h, _dev.ptr(self.buf["r"]))
        return self.buf["r"]

    def residual_finish(self, it, r):
        N.call("bt_cp_residual_finish", self.h, int(it), _dev.ptr(r))

    def read_fit(self, it):
        v = C.c_double()
        N.call("bt_cp_read_fit", self.h, int(it), C.byref(v))
        return v.value

    def finish(self, n_iters):
        hist = (C.c_double * max(int(n_iters), 1))()
        N.call("bt_cp_state_finish", self.h, int(n_iters), hist)
        return [hist[k] for k in range(int(n_iters))]

    def close(self):
        if self.h:
            N.load().bt_cp_state_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def cp_als_sharded(ops, max_iters: int, tol: float, allreduce):
    """Run the ALS sweeps over ``ops`` with ``allreduce(buf)`` (in-place sum
    across ranks) at the exchange points.  Returns (fit_history, n_iters,
    converged); the factors/lambda live in ``ops``."""
    buf = ops.init_local()
    allreduce(buf)
    ops.init_finish(buf)
    prev = float("-inf")
    conv = False
    it = 0
    for it in range(1, int(max_iters) + 1):
        ix = it - 1
        m1 = ops.mttkrp(1)
        allreduce(m1)
        ops.solve_finish(1, ix, ops.solve(1, m1))
        m2 = ops.mttkrp(2)
        allreduce(m2)
        ops.solve_finish(2, ix, ops.solve(2, m2))
        m3 = ops.mttkrp(3)
        g = ops.solve(3, m3)
        allreduce(g)
        ops.solve_finish(3, ix, g)
        r = ops.residual()
        allreduce(r)
        ops.residual_finish(ix, r)
        if tol > 0.0:
            fit = ops.read_fit(ix)
            if abs(fit - prev) < tol:
                conv = True
                break
            prev = fit
    hist = ops.finish(it)
    return hist, it, conv


def torch_allreduce(group=None):
    """In-place SUM over the default (or given) process group; identity for a
    single process."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return lambda buf: None

    def red(buf):
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)

    return red


def shard_bounds(K: int, world: int, rank: int):
    """Contiguous mode-3 slab [k0, k1) of rank (first K % world ranks get one more)."""
    base, extra = divmod(int(K), int(world))
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def cp_als_distributed(x_local, r: int, max_iters: int = 500, tol: float = 1e-10, init=None,
                       fit: str = "auto", group=None):
    """Public multi-GPU CP-ALS (decomp.py:344-410 semantics) for a tensor
    sharded along mode 3: ``x_local`` is this rank's (I, J, K_local) slab
    (numpy / CPU or CUDA tensor), ``init`` the (A, B, C_local) initial factors.
    Returns ``(CpResult-like rep with x, y replicated and z local, fit history)``
    as numpy when x_local is host memory."""
    from .decomp import CpResult, KruskalRep

    xd = _dev.to_device(x_local)
    if init is None:
        raise ValueError("cp_als_distributed needs explicit initial factors (A, B, C_local)")
    f = [_dev.to_device(v).clone() for v in init]
    ops = NativeCpOps(xd, r, f[0], f[1], f[2], max_iters, fit=fit)
    try:
        hist, n_it, conv = cp_als_sharded(ops, max_iters, tol, torch_allreduce(group))
    finally:
        ops.close()
    rep = KruskalRep(x=_dev.like_input(x_local, f[0]), y=_dev.like_input(x_local, f[1]),
                     z=_dev.like_input(x_local, f[2]))
    return CpResult(rep=rep, fit=hist[-1], fit_history=tuple(hist), n_iters=n_it, converged=conv)


# ---------------------------------------------------------------------------
# ST-HOSVD / HOOI sharded along the time (class) mode -- C3, SURVEY.md 8e
# ---------------------------------------------------------------------------


class NativeTuckerOps:
    """Device kernels behind the sharded Tucker driver: mode bases (DMMA
    Gram + eigensolver, optional cross-rank Gram sum) and mode products."""

    def mode_basis(self, x, mode, r, reduce=None, start=None):
        from . import _linalg as L

        return L.mode_basis_dev(x, mode, int(r), reduce=reduce, start=start)

    def ttm_t(self, x, mode, u):
        """x x_mode u^T (u: extent x r)."""
        from .tensor import ttm_dev

        return ttm_dev(x, mode, u, int(u.shape[1]), transpose=True)

    def rows(self, u, r0, r1):
        return u[r0:r1].contiguous()


def torch_allgather_mode2(group=None):
    """Gather an order-3 tensor sharded along mode 2 (uneven slabs allowed)
    into the full tensor on every rank: slabs are exchanged as contiguous
    (P_local, a, b) blocks (padded to the largest slab) and re-interleaved."""
    import torch.distributed as dist

    t = _dev.torch()
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return lambda y: y

    def gather(y):
        world = dist.get_world_size(group)
        a, pl, b = (int(s) for s in y.shape)
        sizes = t.tensor([pl], dtype=t.int64, device=y.device)
        all_sizes = [t.zeros_like(sizes) for _ in range(world)]
        dist.all_gather(all_sizes, sizes, group=group)
        counts = [int(s.item()) for s in all_sizes]
        pmax = max(counts)
        blk = t.zeros((pmax, a, b), dtype=y.dtype, device=y.device)
        blk[:pl] = y.permute(1, 0, 2)
        outs = [t.empty_like(blk) for _ in range(world)]
        dist.all_gather(outs, blk, group=group)
        full = t.cat([o[:c] for o, c in zip(outs, counts)], dim=0)
        return full.permute(1, 0, 2).contiguous()

    return gather


def st_hosvd_sharded(ops, x_local, r13: int, r2: int, allreduce, allgather):
    """ST-HOSVD of an (I, P, J) tensor with modes 1 and 3 sharing one basis
    (the C3 recipe; decomp.st_hosvd with shared=(1, 3)), the tensor sharded
    along mode 2.  Exchanges: the I x I mode-1 Gram (sum, once per deflation
    pass) and the projected (r13, P, r13) tensor (all-gather).  Returns
    (U, V, core), replicated on every rank."""
    u = ops.mode_basis(x_local, 1, r13, reduce=allreduce)
    y = allgather(ops.ttm_t(ops.ttm_t(x_local, 1, u), 3, u))
    v = ops.mode_basis(y, 2, r2)
    return u, v, ops.ttm_t(y, 2, v)


def hooi_sharded(ops, x_local, u, v, sweeps: int, p0: int, p1: int, allreduce, allgather):
    """HOOI sweeps (decomp.hooi, shared=(1, 3)) on the mode-2-sharded tensor.
    U-step: the local partial of x x2 V^T x3 U^T over this rank's rows
    [p0, p1) of V is summed across ranks (I x r2 x r13); V-step: the projected
    (r13, P_local, r13) slabs are all-gathered.  Returns (U, V, core)."""
    y = None
    tb = None   # x_local x3 U^T for the current U: one full pass per sweep serves
                # this sweep's V-step and the next sweep's U-step (decomp._hooi_shared3)
    for _ in range(int(sweeps)):
        if tb is None:
            z = ops.ttm_t(ops.ttm_t(x_local, 2, ops.rows(v, p0, p1)), 3, u)
        else:
            z = ops.ttm_t(tb, 2, ops.rows(v, p0, p1))
        allreduce(z)
        u = ops.mode_basis(z, 1, int(u.shape[1]), start=u)
        tb = ops.ttm_t(x_local, 3, u)
        y = allgather(ops.ttm_t(tb, 1, u))
        v = ops.mode_basis(y, 2, int(v.shape[1]), start=v)
    if y is None:
        y = allgather(ops.ttm_t(ops.ttm_t(x_local, 1, u), 3, u))
    return u, v, ops.ttm_t(y, 2, v)


def tucker_c3_distributed(x_local, r13: int, r2: int, hooi_sweeps: int = 0, p_offset: int = 0,
                          group=None):
    """Public multi-GPU ST-HOSVD (+ HOOI) for the C3 shape: ``x_local`` is
    this rank's (I, P_local, J) slab of the weighted tensor (rows
    [p_offset, p_offset + P_local) of mode 2).  Returns a TuckerRep with
    factors (U, V, U) and the core, replicated, as numpy for host input."""
    from .decomp import TuckerRep

    xd = _dev.to_device(x_local)
    ops = NativeTuckerOps()
    red = torch_allreduce(group)
    gat = torch_allgather_mode2(group)
    u, v, core = st_hosvd_sharded(ops, xd, r13, r2, red, gat)
    if hooi_sweeps:
        pl = int(xd.shape[1])
        u, v, core = hooi_sharded(ops, xd, u, v, hooi_sweeps, p_offset, p_offset + pl, red, gat)
    fu = _dev.like_input(x_local, u)
    return TuckerRep(core=_dev.like_input(x_local, core),
                     factors=(fu, _dev.like_input(x_local, v), fu))


# ---------------------------------------------------------------------------
# RHS-sharded matvec (independent units, no data-path collective)
# ---------------------------------------------------------------------------


def matvec_sharded(rep, x, world: int, rank: int):
    """Columns [c0, c1) of rep @ x for this rank (reconstruct.matvec on a
    shard of the right-hand sides; SURVEY.md 8e "shard RHS columns")."""
    from .reconstruct import matvec

    c0, c1 = shard_bounds(int(x.shape[1]), world, rank)
    return matvec(rep, x[:, c0:c1])
