"""Pins of the NEXT-1 oracle functions: the small generalized eigenproblem of Algorithm 3
(oracle.pencil_eig: Cholesky + cyclic Jacobi) and the lift of its eigenvectors (Mesh.lift), and the
linear outer loop they close (oracle.augmented_step). Each pin compares with an
independent construction: closed forms of 2x2 / diagonal pencils, eigen-residual and F_B-orthonormality
invariants, the columns of P and U~ picked out by unit coefficient vectors, and a brute-force dense
eigensolve of the fine operators (scipy) for the converged outer loop."""
import numpy as np
import pytest
import scipy.linalg as sl

import gen
import oracle


def test_pencil_eig_2x2_closed_form():
    a, b, c = 2.0, -0.75, 5.5
    FA = np.array([[a, b], [b, c]])
    ev, Y = oracle.pencil_eig(FA, np.eye(2), 2)
    m, r = 0.5 * (a + c), np.hypot(0.5 * (a - c), b)
    assert np.allclose(ev, [m - r, m + r], rtol=0, atol=1e-14)
    # eigenvector of the lower eigenvalue: (b, lambda - a) normalised, up to sign
    v = np.array([b, m - r - a])
    v /= np.linalg.norm(v)
    assert abs(abs(v @ Y[:, 0]) - 1.0) < 1e-14


def test_pencil_eig_diagonal_pencil():
    d = np.array([3.0, -1.0, 7.0, 0.5, 2.0])
    e = np.array([2.0, 0.5, 1.0, 4.0, 8.0])
    ev, Y = oracle.pencil_eig(np.diag(d), np.diag(e), 5)
    assert np.allclose(ev, np.sort(d / e), rtol=0, atol=1e-14)
    # F_B-normalised unit vectors: |y| = 1/sqrt(e) on the matching coordinate
    for j in range(5):
        i = int(np.argmax(np.abs(Y[:, j])))
        assert abs(abs(Y[i, j]) - 1.0 / np.sqrt(e[i])) < 1e-14
        assert abs(d[i] / e[i] - ev[j]) < 1e-14


@pytest.mark.parametrize("D,k", [(7, 3), (40, 40), (90, 12)])
def test_pencil_eig_invariants(D, k):
    rng = np.random.default_rng(D)
    A = rng.standard_normal((D, D))
    A = A + A.T
    B = rng.standard_normal((D, D))
    B = B @ B.T + D * np.eye(D)
    ev, Y = oracle.pencil_eig(A, B, k)
    assert np.all(np.diff(ev) >= 0)
    scale = np.abs(A).max() + np.abs(ev).max() * np.abs(B).max()
    assert np.abs(A @ Y - (B @ Y) * ev).max() <= 1e-12 * scale * D
    assert np.abs(Y.T @ B @ Y - np.eye(k)).max() <= 1e-12 * D
    # Courant-Fischer: the lowest eigenvalue is the minimum Rayleigh quotient (spot check vs random vectors)
    X = rng.standard_normal((D, 200))
    rq = np.einsum("ij,ij->j", X, A @ X) / np.einsum("ij,ij->j", X, B @ X)
    assert ev[0] <= rq.min() + 1e-12


def test_pencil_eig_rejects_indefinite_mass():
    FA = np.eye(3)
    FB = np.diag([1.0, -1.0, 2.0])
    with pytest.raises(oracle.OracleError):
        oracle.pencil_eig(FA, FB, 2)


def small(n=6, N=3, **kw):
    cfg = dict(L=3.0, n=n, grading=None, jitter=0.2, nuclei=[((0.3, -0.2, 0.1), 2)], vnoise=0.05, N=N,
               orbitals="gauss", lam=("uniform", -2.0, -0.5), nc=2, seed=5)
    cfg.update(kw)
    return gen.make_problem(cfg)


def test_lift_picks_columns_of_P_and_Ut():
    p = small()
    m = oracle.Mesh.from_problem(p)
    rng = np.random.default_rng(1)
    Ut = rng.standard_normal((p.n_free, p.N))
    D = p.n_H + p.N
    import scipy.sparse as sp
    P = sp.csr_matrix((p.P_val, p.P_col, p.P_rowptr), shape=(p.n_free, p.n_H)).toarray()
    # Y = unit vectors on coarse columns 0 and n_H-1 -> those columns of P
    Y = np.zeros((D, 2))
    Y[0, 0] = 1.0
    Y[p.n_H - 1, 1] = 1.0
    assert np.array_equal(m.lift(p.n_H, p.P_rowptr, p.P_col, p.P_val, Ut, Y), P[:, [0, p.n_H - 1]])
    # Y = [0; I] -> U~ itself
    Y = np.vstack([np.zeros((p.n_H, p.N)), np.eye(p.N)])
    assert np.array_equal(m.lift(p.n_H, p.P_rowptr, p.P_col, p.P_val, Ut, Y), Ut)


def test_augmented_outer_loop_converges_to_fine_eigenpairs():
    """Algorithm 3 with a fixed (linear) potential: BVPs, projection onto [P_H | U~], small eigenproblem,
    lift. The Ritz values are upper bounds of the fine eigenvalues (Rayleigh-Ritz in a subspace of S_h) and
    converge to the brute-force dense eigenvalues of (H, M) on the same mesh."""
    p = gen.make_problem(dict(L=5.0, n=10, grading=None, jitter=0.15, nuclei=[((0.0, 0.0, 0.0), 1)],
                              vnoise=0.0, N=4, orbitals="gauss", lam=("const", 2.0), nc=5, seed=9,
                              potential="harmonic"))
    mu = 0.0   # V = |x|^2/2 >= 0: H itself is SPD, so the BVPs are plain inverse iterations
    # four independent starting orbitals: Gaussians at the centre and one unit step along each axis
    xf = p.xyz[p.free_nodes]
    ctr = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    p.U = np.ascontiguousarray(np.stack([np.exp(-0.5 * ((xf - c) ** 2).sum(1)) for c in ctr], axis=1))
    m = oracle.Mesh.from_problem(p)
    m.assemble_veff(p.V, mu)
    H, M = m.csr("H").toarray(), m.csr("M").toarray()
    w = sl.eigh(H, M, eigvals_only=True)[:p.N]
    lam, U = p.lam.copy(), p.U.copy()
    errs = []
    for it in range(40):
        lam, U, info = oracle.augmented_step(m, p.n_H, p.P_rowptr, p.P_col, p.P_val, lam, U, tol=1e-12)
        assert np.all(lam >= w - 1e-10)          # Ritz values bound the fine eigenvalues from above
        errs.append(np.max(np.abs(lam - w)))
        if errs[-1] < 1e-10 * np.abs(w).max():
            break
    assert errs[-1] < 1e-10 * np.abs(w).max(), errs
    assert errs[-1] < 1e-3 * errs[0]
    # linear convergence, rate of the order of ((lambda_N + mu) / (lambda_{N+1} + mu))^2 (Rayleigh-Ritz
    # squares the vector error; paper: "rate -> 2/3")
    w6 = sl.eigh(H, M, eigvals_only=True)[:p.N + 1]
    rate = (errs[-2] / errs[-6]) ** 0.25
    assert rate < ((w6[p.N - 1] + mu) / (w6[p.N] + mu)) ** 2 + 0.05, (rate, errs)
    # the lifted orbitals are M-orthonormal eigenvectors of the fine pencil
    assert np.abs(U.T @ M @ U - np.eye(p.N)).max() < 1e-8
    assert np.abs(H @ U - (M @ U) * lam).max() < 1e-6 * np.abs(H).max()
