#!/usr/bin/env python
"""NEXT-4 experiment: would O'Leary block PCG cut the iterations of the N shifted
BVPs A u~_i = (lambda_i + mu) M u_i enough to pay for its extra bytes? A and M come from the library's
own assembly (ks_values, on the GPU); both solvers run on the host in numpy/scipy with the same Jacobi
preconditioner, x0 = u and stopping rule (||r_i|| <= tol ||b_i||, every column). Prints one JSON line per
config with the iteration counts."""
import json
import os
import sys

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2404_19249_b200 as ks  # noqa: E402


def jacobi_pcg(A, Dinv, B, X, tol, maxit=1000):
    bn = np.linalg.norm(B, axis=0)
    R = B - A @ X
    Z = Dinv[:, None] * R
    P = Z.copy()
    rho = (R * Z).sum(0)
    act = np.linalg.norm(R, axis=0) > tol * bn
    it = 0
    while act.any() and it < maxit:
        Q = A @ P
        al = np.where(act, rho / (P * Q).sum(0), 0.0)
        X = X + P * al
        R = R - Q * al
        Z = Dinv[:, None] * R
        rn = (R * Z).sum(0)
        be = rn / rho
        rho = rn
        it += 1
        act = act & (np.linalg.norm(R, axis=0) > tol * bn)
        P = Z + P * be
    return it


def block_pcg(A, Dinv, B, X, tol, maxit=1000):
    """O'Leary (1980) block PCG: alpha = (P^T A P)^-1 (Z^T R), beta = (Z_old^T R_old)^-1 (Z^T R)."""
    bn = np.linalg.norm(B, axis=0)
    R = B - A @ X
    Z = Dinv[:, None] * R
    P = Z.copy()
    G = Z.T @ R
    it = 0
    while it < maxit:
        Q = A @ P
        al = np.linalg.solve(P.T @ Q, G)
        X = X + P @ al
        R = R - Q @ al
        it += 1
        if np.all(np.linalg.norm(R, axis=0) <= tol * bn):
            break
        Z = Dinv[:, None] * R
        Gn = Z.T @ R
        P = Z + P @ np.linalg.solve(G, Gn)
        G = Gn
    return it


def main():
    cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4").split(",")]
    for c in cfgs:
        p = gen.make_problem(c)
        ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
        ctx.assemble_veff(torch.from_numpy(p.V).cuda(), p.mu)
        rp, col = (t.cpu().numpy() for t in ctx.pattern()[:2])
        v = {k: t.cpu().numpy() for k, t in ctx.values().items()}
        n = p.n_free
        A = sp.csr_matrix((v["A"], col, rp), shape=(n, n))
        M = sp.csr_matrix((v["M"], col, rp), shape=(n, n))
        B = M @ (p.U * (p.lam + p.mu)[None, :])
        Dinv = 1.0 / A.diagonal()
        it_j = jacobi_pcg(A, Dinv, B, p.U.copy(), 1e-10)
        it_b = block_pcg(A, Dinv, B, p.U.copy(), 1e-10)
        print(json.dumps({"config": f"C{c}", "n": n, "N": p.N, "mu": p.mu, "jacobi_pcg_iterations": it_j,
                          "block_pcg_iterations": it_b}), flush=True)
        del ctx


if __name__ == "__main__":
    main()
