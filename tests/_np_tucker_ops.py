"""CPU stand-in for parallel.NativeTuckerOps (test double): mode bases from
the (optionally cross-rank summed) unfolding Gram and mode products, on CPU
torch tensors so the gloo collectives apply.  Mirrors decomp.py:220-234 (sign
rule) with a Gram eigensolve in place of the SVD."""

import numpy as np
import torch


def _unfold(x, mode):
    return torch.movedim(x, mode - 1, 0).reshape(x.shape[mode - 1], -1)


class TorchCpuTuckerOps:
    def mode_basis(self, x, mode, r, reduce=None, start=None):
        m = _unfold(x, mode)
        g = (m @ m.T).contiguous()
        if reduce is not None:
            reduce(g)
        w, v = np.linalg.eigh(g.numpy())
        u = v[:, ::-1][:, :r]
        lead = np.argmax(np.abs(u), axis=0)
        s = np.sign(u[lead, np.arange(r)])
        s[s == 0] = 1.0
        return torch.from_numpy(np.ascontiguousarray(u * s))

    def ttm_t(self, x, mode, u):
        y = torch.tensordot(u.T, torch.movedim(x, mode - 1, 0), dims=1)
        return torch.movedim(y, 0, mode - 1).contiguous()

    def rows(self, u, r0, r1):
        return u[r0:r1].contiguous()
