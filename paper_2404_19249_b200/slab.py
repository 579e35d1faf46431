"""Row-slab partition of ONE block solve over several processes.

The N BVPs of Algorithm 3 (Aux_Linear_Problem) are one sparse operator applied to an
[n][N] block. The paper distributes the work over processes (the scaling runs of
PAPER.md:1410-1418); here each rank (one GPU) owns a contiguous slab of rows of the free numbering:

  * partition  slab bounds balanced by nonzeros; the halo of a slab is the window of rows its rows reference
               (lexicographic numbering: about one grid plane on each side), received from the two
               neighbouring ranks only;
  * exchange   before every S phase the neighbours' boundary rows of z (one point-to-point message each way);
  * reduction  after every phase the per-column dot products of all ranks are all-gathered and summed in rank
               order, so every rank derives bitwise the same alpha_i, beta_i and the same stopping decisions.

The arithmetic of every phase runs in libks's kernels (ks_slab_init / spmm / update / finish: the fused
two-phase Jacobi-PCG of ks_block_solve over a row range, include/ks.h); this module is the host driver only:
partition, exchange schedule, coefficients, per-column freezing and the stopping rule of ks_block_solve
(DESIGN.md §7). The driver takes an executor object, so the multi-process logic is tested on CPU processes
(gloo, tests/test_slab.py) with a test-only executor, and on the GPU with `GpuSlab`.
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def slab_bounds(row_ptr, col, world: int):
    """[(row0, row1, halo0, halo1)] of every rank: rows [row0, row1) whose first nonzero index lies in
    [r nnz / world, (r+1) nnz / world), and the window [halo0, halo1) of rows they reference (columns are
    sorted within a row). Raises ValueError when a slab is empty or its halo reaches past a neighbour."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    n, nnz = len(row_ptr) - 1, int(row_ptr[-1])
    cuts = [0] + [int(np.searchsorted(row_ptr[:-1], int(nnz * r / world), side="left")) for r in range(1, world)]
    cuts.append(n)
    out = []
    for r in range(world):
        a, b = cuts[r], cuts[r + 1]
        if b <= a:
            raise ValueError(f"slab {r} of {world} is empty (n_free = {n})")
        lo = min(a, int(col[row_ptr[a:b]].min()))
        hi = max(b, int(col[row_ptr[a + 1:b + 1] - 1].max()) + 1)
        out.append((a, b, lo, hi))
    for r, (a, b, lo, hi) in enumerate(out):
        if r > 0 and lo < out[r - 1][0]:
            raise ValueError(f"slab {r}: halo row {lo} lies beyond the lower neighbour (too many ranks)")
        if r + 1 < world and hi > out[r + 1][1]:
            raise ValueError(f"slab {r}: halo row {hi - 1} lies beyond the upper neighbour (too many ranks)")
    return out


def halo_schedule(bounds, rank: int):
    """(sends, recvs) of one rank: lists of (peer, row0, row1). The lower neighbour needs my rows
    [row0, its halo1), the upper one my rows [its halo0, row1); I receive my halo rows from them."""
    a, b, lo, hi = bounds[rank]
    sends, recvs = [], []
    if rank > 0:
        pa, pb, plo, phi = bounds[rank - 1]
        if phi > a:
            sends.append((rank - 1, a, phi))
        if lo < a:
            recvs.append((rank - 1, lo, a))
    if rank + 1 < len(bounds):
        na, nb, nlo, nhi = bounds[rank + 1]
        if nlo < b:
            sends.append((rank + 1, nlo, b))
        if hi > b:
            recvs.append((rank + 1, b, hi))
    return sends, recvs


class _Comm:
    """torch.distributed plumbing of the driver: halo rows and the all-gather of the dots. With a gloo group
    and CUDA tensors the messages are staged through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.host = dist.get_backend(group) == "gloo"

    def gsum(self, t):
        """sum over ranks of the per-rank vector t (torch), in rank order -> numpy float64."""
        import torch
        x = t.detach().to("cpu") if self.host else t.detach()
        parts = [torch.empty_like(x) for _ in range(self.world)]
        self.dist.all_gather(parts, x.contiguous(), group=self.group)
        s = np.zeros(x.numel())
        for p in parts:   # fixed order: every rank gets bitwise the same sum
            s = s + p.cpu().numpy().astype(np.float64)
        return s

    def halo(self, z, sends, recvs):
        """z[rows] <- neighbours' rows (recvs), my rows -> neighbours (sends)."""
        import torch
        ops, bufs = [], []
        for peer, r0, r1 in sends:
            buf = z[r0:r1].contiguous()
            if self.host:
                buf = buf.cpu()
            ops.append(self.dist.P2POp(self.dist.isend, buf, peer, group=self.group))
        for peer, r0, r1 in recvs:
            buf = torch.empty_like(z[r0:r1], device="cpu" if self.host else z.device)
            ops.append(self.dist.P2POp(self.dist.irecv, buf, peer, group=self.group))
            bufs.append((buf, r0, r1))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        for buf, r0, r1 in bufs:
            z[r0:r1].copy_(buf)


def slab_block_solve(ex, lam, tol: float = 1e-10, max_iter: int = 2000, group=None):
    """Algorithm 3's N BVPs  A u~_i = (lambda_i + mu) M u_i with rows split over the ranks of
    `group`; the iteration is that of ks_block_solve (fused two-phase Jacobi-PCG, x0 = u, per-column alpha,
    beta, stop on ||r||_2 <= tol ||b||_2, converged columns frozen, p.Ap <= 0 -> NOT_SPD for that column).
    `ex` executes the phases on this rank's rows (GpuSlab, or a test executor). Returns dict(status, iters,
    relres, block_iters); the solution rows are ex.result()."""
    comm = _Comm(group)
    lam = np.asarray(lam, dtype=np.float64)
    N, NP = len(lam), ex.NP
    sends, recvs = halo_schedule(ex.bounds, comm.rank)
    d = comm.gsum(ex.init())
    bb, rz, rr = d[:NP][:N], d[NP:2 * NP][:N], d[2 * NP:3 * NP][:N]
    bnorm = np.sqrt(bb)
    rho, rr_last = rz.copy(), rr.copy()
    finite = np.isfinite(bnorm) & np.isfinite(rz) & np.isfinite(rr)
    status = "ok" if finite.all() else "nonfinite"
    active = finite & ~(np.sqrt(rr) <= tol * bnorm)
    iters = np.zeros(N, dtype=np.int32)
    ax = np.zeros(NP)      # alpha of the deferred x update
    beta = np.zeros(NP)
    it, first, xwritten = 0, True, False
    if active.any():
        comm.halo(ex.z, sends, recvs)
        while True:
            pq = comm.gsum(ex.spmm(first, ax, beta, xwritten))[:N]
            if not first:
                xwritten = True
            first = False
            alpha = np.zeros(NP)
            bad = active & ~(pq > 0.0)
            if bad.any():
                status = "not_spd" if np.all(np.isfinite(pq[bad])) else "nonfinite"
                active &= ~bad
            alpha[:N] = np.where(active, rho / np.where(active, pq, 1.0), 0.0)
            ax = alpha.copy()
            d = comm.gsum(ex.update(alpha))
            rz, rr = d[:NP][:N], d[NP:2 * NP][:N]
            beta = np.zeros(NP)
            for c in np.nonzero(active)[0]:
                iters[c] += 1
                if not (np.isfinite(rz[c]) and np.isfinite(rr[c])):
                    status = "nonfinite"
                    active[c] = False
                    continue
                beta[c] = rz[c] / rho[c]
                rho[c], rr_last[c] = rz[c], rr[c]
                if np.sqrt(rr[c]) <= tol * bnorm[c]:
                    beta[c] = 0.0
                    active[c] = False
            it += 1
            if not active.any():
                break
            if it >= max_iter:
                if status == "ok":
                    status = "not_converged"
                break
            comm.halo(ex.z, sends, recvs)
    ex.finish(ax, xwritten, it > 0)
    relres = np.where(bnorm > 0, np.sqrt(rr_last) / np.where(bnorm > 0, bnorm, 1.0), np.sqrt(rr_last))
    return dict(status=status, iters=iters, relres=relres, block_iters=it)


class GpuSlab:
    """Executor of slab_block_solve on this rank's GPU through libks (ks_slab_*). Vectors are [n_free][NP]
    torch CUDA tensors in the global numbering; only this rank's rows (and the halo rows of z) are used."""

    def __init__(self, ctx, lam, U, bounds, rank: int):
        import torch
        from . import ks as _ks
        self.ctx, self.L = ctx, ctx._L
        self.bounds, self.rank = bounds, rank
        self.row0, self.row1 = bounds[rank][0], bounds[rank][1]
        N = int(U.shape[1])
        self.N = N
        self.NP = 1 << max(0, (N - 1).bit_length())
        n, NP, dev = ctx.n_free, self.NP, U.device
        _ks._check_cuda_tensor(U, torch.float64, (n, N), "U")
        self.U = torch.zeros((n, NP), dtype=torch.float64, device=dev)
        self.U[:, :N] = U
        self.lam = torch.zeros(NP, dtype=torch.float64, device=dev)
        self.lam[:N] = torch.as_tensor(np.asarray(lam, dtype=np.float64), device=dev)
        self.z = torch.zeros((n, NP), dtype=torch.float64, device=dev)
        self.q, self.p, self.x = (torch.zeros_like(self.z) for _ in range(3))
        self.dots = torch.zeros(3 * NP, dtype=torch.float64, device=dev)

    def _call(self, st):
        self.ctx._call(st)

    @staticmethod
    def _h(a):
        return np.ascontiguousarray(a, dtype=np.float64)

    def init(self):
        self._call(self.L.ks_slab_init(self.ctx._h, self.NP, self.row0, self.row1, self.lam.data_ptr(),
                                       self.U.data_ptr(), self.z.data_ptr(), self.p.data_ptr(), self.dots.data_ptr()))
        return self.dots[:3 * self.NP].clone()

    def spmm(self, first, ax, beta, xwritten):
        a, b = self._h(ax), self._h(beta)
        xin = self.x if xwritten else self.U
        self._call(self.L.ks_slab_spmm(self.ctx._h, self.NP, self.row0, self.row1, int(first), a.ctypes.data,
                                       b.ctypes.data, self.z.data_ptr(), self.q.data_ptr(), self.p.data_ptr(),
                                       xin.data_ptr(), self.x.data_ptr(), self.dots.data_ptr()))
        return self.dots[:self.NP].clone()

    def update(self, alpha):
        a = self._h(alpha)
        self._call(self.L.ks_slab_update(self.ctx._h, self.NP, self.row0, self.row1, a.ctypes.data,
                                         self.z.data_ptr(), self.q.data_ptr(), self.dots.data_ptr()))
        return self.dots[:2 * self.NP].clone()

    def finish(self, ax, xwritten, iterated):
        if not iterated:
            self.x[self.row0:self.row1] = self.U[self.row0:self.row1]
            return
        a = self._h(ax)
        xin = self.x if xwritten else self.U
        self._call(self.L.ks_slab_finish(self.ctx._h, self.NP, self.row0, self.row1, a.ctypes.data,
                                         self.p.data_ptr(), xin.data_ptr(), self.x.data_ptr()))

    def result(self):
        """This rank's rows of u~: [row1 - row0][N]."""
        return self.x[self.row0:self.row1, :self.N]


def gpu_slab_bounds(ctx, world: int):
    """slab_bounds of a context's pattern (copied to the host once)."""
    rp, col = ctx.pattern()[:2]
    return slab_bounds(rp.cpu().numpy(), col.cpu().numpy(), world)
