#!/usr/bin/env python
"""NEXT-4 experiment: a stronger preconditioner for the BVPs of Algorithm 3 (A u~ = (lambda + mu) M u,
A = H + mu M; the paper uses GAMG). Jacobi (what ks_block_solve runs)
against the two-level preconditioners on the method's own coarse space P:
    additive:  z = D^-1 r + P A_H^-1 P^T r,        A_H = P^T A P  (dense Cholesky, n_H small)
    balanced:  coarse, smoother, coarse (symmetrised deflation)
Operators from the CPU oracle (test infrastructure: this is an offline experiment, not a product path), P from gen,
x0 = u (the warm start of ks_block_solve), PCG to 1e-10 on the host. One JSON line per config and column."""
import json
import os
import sys

import numpy as np
import scipy.linalg as sla

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import oracle  # noqa: E402
import scipy.sparse as sp  # noqa: E402


def pcg(A, b, x0, prec, tol=1e-10, maxit=5000):
    x = x0.copy()
    r = b - A @ x
    z = prec(r)
    p = z.copy()
    rz = r @ z
    bn = np.linalg.norm(b)
    if np.linalg.norm(r) <= tol * bn:
        return 0
    for it in range(1, maxit + 1):
        q = A @ p
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
    cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4").split(",")]
    cols = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    for c in cfgs:
        p = gen.make_problem(c)
        om = oracle.Mesh.from_problem(p)
        om.assemble_veff(p.V, p.mu)
        A, M = om.csr("A"), om.csr("M")
        n = p.n_free
        P = sp.csr_matrix((p.P_val, p.P_col, p.P_rowptr), shape=(n, p.n_H))
        Dinv = 1.0 / A.diagonal()
        AH = (P.T @ A @ P).toarray()
        cho = sla.cho_factor(AH)
        coarse = lambda r: P @ sla.cho_solve(cho, P.T @ r)
        jac = lambda r: Dinv * r
        add = lambda r: Dinv * r + coarse(r)

        def balanced(r):
            y = coarse(r)
            z = y + Dinv * (r - A @ y)
            return z + coarse(r - A @ z)
        for j in range(min(cols, p.N)):
            u = np.ascontiguousarray(p.U[:, j])
            b = (p.lam[j] + p.mu) * (M @ u)
            res = {"config": f"C{c}", "column": j, "n": n, "n_H": p.n_H, "mu": p.mu,
                   "jacobi": pcg(A, b, u, jac), "two_level_additive": pcg(A, b, u, add),
                   "two_level_balanced": pcg(A, b, u, balanced)}
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
