#!/usr/bin/env python
"""NEXT-4 experiment: a two-level preconditioner for the Hartree Poisson solve (K x = b, the stiffness
matrix on the free nodes), built from the method's own coarse space P (the nonnested interpolation):
    additive:        z = D^-1 r + P K_H^-1 P^T r,            K_H = P^T K P  (dense Cholesky, n_H small)
    balanced / deflated variants are printed for comparison.
K comes from the library's assembly (ks_values, on the GPU), P from gen (the structured coarse Kuhn mesh of
the config). Right-hand side: the P1 load of a Gaussian charge (what ks_hartree solves). PCG to 1e-10 on the
host (scipy). Prints one JSON line per config with the iteration counts."""
import json
import os
import sys

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2404_19249_b200 as ks  # noqa: E402


def pcg(K, b, prec, tol=1e-10, maxit=5000):
    x = np.zeros_like(b)
    r = b.copy()
    z = prec(r)
    p = z.copy()
    rz = r @ z
    bn = np.linalg.norm(b)
    for it in range(1, maxit + 1):
        q = K @ p
        al = rz / (p @ q)
        x += al * p
        r -= al * q
        if np.linalg.norm(r) <= tol * bn:
            return it
        z = prec(r)
        rzn = r @ z
        p = z + (rzn / rz) * p
        rz = rzn
    return maxit


def main():
    cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "3,4").split(",")]
    for c in cfgs:
        p = gen.make_problem(c)
        ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
        ctx.assemble_veff(torch.from_numpy(p.V).cuda(), p.mu)
        rp, col = (t.cpu().numpy() for t in ctx.pattern()[:2])
        v = {k: t.cpu().numpy() for k, t in ctx.values().items()}
        n = p.n_free
        K = sp.csr_matrix((v["K"], col, rp), shape=(n, n))
        M = sp.csr_matrix((v["M"], col, rp), shape=(n, n))
        P = sp.csr_matrix((p.P_val, p.P_col, p.P_rowptr), shape=(n, p.n_H))
        xf = p.xyz[p.free_nodes]
        rho = np.exp(-((xf - np.array([0.3, -0.2, 0.1])) ** 2).sum(1) / 2.0)
        b = 4 * np.pi * (M @ rho)
        Dinv = 1.0 / K.diagonal()
        KH = (P.T @ K @ P).toarray()
        cho = sla.cho_factor(KH)
        coarse = lambda r: P @ sla.cho_solve(cho, P.T @ r)
        jac = lambda r: Dinv * r
        add = lambda r: Dinv * r + coarse(r)

        def balanced(r):   # deflation-type (coarse first, then smoother on the remainder, symmetrised)
            y = coarse(r)
            w = r - K @ y
            z = y + Dinv * w
            w2 = r - K @ z
            return z + coarse(w2)
        res = {"config": f"C{c}", "n": n, "n_H": p.n_H, "jacobi": pcg(K, b, jac), "two_level_additive": pcg(K, b, add),
               "two_level_balanced": pcg(K, b, balanced)}
        print(json.dumps(res), flush=True)
        del ctx


if __name__ == "__main__":
    main()
