"""Per-entry parity bounds for the projected matrices (test helper; no product or oracle arithmetic).

F_A = W^T H W and F_B = W^T M W with W = [P | U~] (st1-st7). Every entry is a sum of
products w_ki Op_kl w_lj, so a computation in another summation order differs from the oracle by at most
(number of terms) x u x (|W|^T |Op| |W|)_ij. DESIGN.md reading Q12' states the per-entry tolerance
|dF_ij| <= 1e-9 (|W|^T |Op| |W|)_ij that the GPU parity tests apply to every entry (not a block norm), so a
wrong small entry (e.g. a b_H row of a coarse node next to the boundary) cannot hide under a large one.
"""
import numpy as np
import scipy.sparse as sp


def abs_gram(P_abs, U_abs, Op_abs):
    """(|W|^T |Op| |W|) for W = [P | U] as a dense (n_H + N)^2 array; P_abs sparse, U_abs dense."""
    OpP = (Op_abs @ P_abs).tocsr()
    OpU = Op_abs @ U_abs
    n_H, N = P_abs.shape[1], U_abs.shape[1]
    B = np.zeros((n_H + N, n_H + N))
    B[:n_H, :n_H] = (P_abs.T @ OpP).toarray()
    B[:n_H, n_H:] = P_abs.T @ OpU
    B[n_H:, :n_H] = B[:n_H, n_H:].T
    B[n_H:, n_H:] = U_abs.T @ OpU
    return B


def projection_bounds(om, n_H, P_rowptr, P_col, P_val, Ut):
    """Per-entry bounds (bound_FA, bound_FB) for the oracle mesh `om` (H unshifted, M)."""
    n = Ut.shape[0]
    P_abs = sp.csr_matrix((np.abs(P_val), P_col, P_rowptr), shape=(n, n_H))
    U_abs = np.abs(Ut)
    return (abs_gram(P_abs, U_abs, abs(om.csr("H"))), abs_gram(P_abs, U_abs, abs(om.csr("M"))))


def assert_entrywise(F, Fo, bound, tol=1e-9, what="F"):
    """|F - Fo| <= tol * bound on every entry (entries with bound 0 must agree exactly)."""
    err = np.abs(F - Fo)
    bad = err > tol * bound
    if np.any(bad):
        i, j = np.unravel_index(np.argmax(np.where(bad, err / np.maximum(bound, 1e-300), 0)), F.shape)
        raise AssertionError(f"{what}[{i},{j}]: gpu {F[i, j]!r} oracle {Fo[i, j]!r} |d| {err[i, j]:.3e} "
                             f"> {tol:g} x bound {bound[i, j]:.3e} ({int(bad.sum())} entries)")
