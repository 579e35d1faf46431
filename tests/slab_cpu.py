"""Test-only CPU executor of paper_2404_19249_b200.slab.slab_block_solve: the phases of the fused two-phase
Jacobi-PCG (include/ks.h ks_slab_*) over one rank's rows, in numpy/torch on the host, with the operators from
the oracle (A = 1/2 K + M_V + mu M, M, diag A). It lets the multi-process driver (partition, halo exchange,
all-gathered dots, coefficients, freezing, stopping) run on CPU processes over gloo. It is test
infrastructure, never a product path."""
import numpy as np
import torch


class CpuSlab:
    def __init__(self, A, M, lam, mu, U, bounds, rank):
        self.A, self.M = A.tocsr(), M.tocsr()
        self.d = self.A.diagonal().copy()
        self.bounds, self.rank = bounds, rank
        self.row0, self.row1 = bounds[rank][0], bounds[rank][1]
        n, N = U.shape
        self.N = N
        self.NP = 1 << max(0, (N - 1).bit_length())
        self.U = np.zeros((n, self.NP))
        self.U[:, :N] = U
        self.sh = np.zeros(self.NP)
        self.sh[:N] = np.asarray(lam) + mu
        self.z = torch.zeros((n, self.NP), dtype=torch.float64)   # exchanged by the driver (gloo)
        self.q = np.zeros((n, self.NP))
        self.p = np.zeros((n, self.NP))
        self.x = np.zeros((n, self.NP))

    def _rows(self, Op, X):
        return Op[self.row0:self.row1] @ X   # only the referenced (own + halo) rows of X matter

    def init(self):
        a, b = self.row0, self.row1
        bvec = self.sh * self._rows(self.M, self.U)
        r = bvec - self._rows(self.A, self.U)
        z = r / self.d[a:b, None]
        self.z[a:b] = torch.from_numpy(z)
        self.p[a:b] = z
        return torch.from_numpy(np.concatenate([(bvec * bvec).sum(0), (r * z).sum(0), (r * r).sum(0)]))

    def spmm(self, first, ax, beta, xwritten):
        a, b = self.row0, self.row1
        zf = self.z.numpy()
        w = self._rows(self.A, zf)
        if first:
            self.q[a:b] = w
            return torch.from_numpy((self.p[a:b] * w).sum(0))
        xin = self.x if xwritten else self.U
        self.x[a:b] = xin[a:b] + ax * self.p[a:b]
        self.p[a:b] = zf[a:b] + beta * self.p[a:b]
        self.q[a:b] = w + beta * self.q[a:b]
        return torch.from_numpy((self.p[a:b] * self.q[a:b]).sum(0))

    def update(self, alpha):
        a, b = self.row0, self.row1
        z = self.z.numpy()[a:b] - alpha * (self.q[a:b] / self.d[a:b, None])
        self.z[a:b] = torch.from_numpy(z)
        r = self.d[a:b, None] * z
        return torch.from_numpy(np.concatenate([(r * z).sum(0), (r * r).sum(0)]))

    def finish(self, ax, xwritten, iterated):
        a, b = self.row0, self.row1
        if not iterated:
            self.x[a:b] = self.U[a:b]
            return
        xin = self.x if xwritten else self.U
        self.x[a:b] = xin[a:b] + ax * self.p[a:b]

    def result(self):
        return self.x[self.row0:self.row1, :self.N]
