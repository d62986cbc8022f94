"""CPU stand-in for NativeCpOps (test double): the same CP phases restated in
numpy on a local mode-3 slab, so the sharded orchestration
(paper_2105_01170_b200.parallel.cp_als_sharded) can be checked with gloo on
CPU.  Mirrors decomp.py:380-396 per phase."""

import numpy as np
from scipy.linalg import khatri_rao

from oracle import port


class NumpyCpOps:
    def __init__(self, x_local, r, a, b, c_local, max_iters, norm_x=0.0):
        import torch

        self.torch = torch
        self.x = x_local
        self.R = r
        self.f = [a.copy(), b.copy(), c_local.copy()]
        self.g = [None, None, None]
        self.lam = np.ones(r)
        self.hist = np.zeros(max_iters)
        self.x2 = 0.0
        self.norm_x = norm_x
        self.unf = [port.unfold(x_local, k + 1) for k in range(3)]

    def _t(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))

    def init_local(self):
        self.g[0] = self.f[0].T @ self.f[0]
        self.g[1] = self.f[1].T @ self.f[1]
        gc = self.f[2].T @ self.f[2]
        x2 = self.norm_x ** 2 if self.norm_x > 0 else float(np.sum(self.x * self.x))
        return self._t(np.concatenate([gc.ravel(), [x2, 0.0]]))

    def init_finish(self, buf):
        b = buf.numpy()
        R = self.R
        self.g[2] = b[:R * R].reshape(R, R).copy()
        self.x2 = float(b[R * R])

    def mttkrp(self, mode):
        k = mode - 1
        o0, o1 = [j for j in range(3) if j != k]
        return self._t(self.unf[k] @ khatri_rao(self.f[o1], self.f[o0]))

    def solve(self, mode, m):
        k = mode - 1
        o0, o1 = [j for j in range(3) if j != k]
        mm = m.numpy()
        fu = mm @ np.linalg.pinv(self.g[o0] * self.g[o1])
        self._fu = fu
        inner = float(np.sum(fu * mm)) if mode == 3 else 0.0
        return self._t(np.concatenate([(fu.T @ fu).ravel(), [inner, 0.0]]))

    def solve_finish(self, mode, it, g):
        k = mode - 1
        R = self.R
        gb = g.numpy()
        gu = gb[:R * R].reshape(R, R)
        nrm = np.sqrt(np.diag(gu)).copy()
        nrm[nrm == 0] = 1.0
        self.f[k] = self._fu / nrm
        self.g[k] = gu / np.outer(nrm, nrm)
        if mode == 3:
            self.lam = nrm
            xh2 = float(nrm @ (self.g[0] * self.g[1] * self.g[2]) @ nrm)
            res2 = max(self.x2 - 2.0 * gb[R * R] + xh2, 0.0)
            self.hist[it] = 1.0 - np.sqrt(res2 / self.x2)

    def residual(self):
        approx = np.einsum("ir,jr,kr->ijk", self.f[0] * self.lam, self.f[1], self.f[2])
        return self._t(np.array([float(np.sum((self.x - approx) ** 2)), 0.0]))

    def residual_finish(self, it, r):
        self.hist[it] = 1.0 - np.sqrt(float(r.numpy()[0])) / np.sqrt(self.x2)

    def read_fit(self, it):
        return float(self.hist[it])

    def finish(self, n_iters):
        self.f[0] = self.f[0] * self.lam
        return list(self.hist[:n_iters])
