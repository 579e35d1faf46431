"""NEXT-1 on the GPU: the pencil eigensolver, the lift and the Algorithm-3 outer loop
through the C ABI, against the oracle (tests/test_oracle_next1.py pins it) on the same inputs.
Tolerances: eigenvalues |d lambda| <= 1e-9 max|lambda| (north_star's projected-eigenvalue bound);
eigenvectors compared through the residual and F_B-orthonormality (signs are arbitrary, Q23); lift
|d u| <= 1e-12 (|P||Y| + |U~||Y|) elementwise."""
import numpy as np
import pytest
import scipy.linalg as sl

import gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
DEV = "cuda"


def dt(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _ctx(p, mu):
    import paper_2404_19249_b200 as ks
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
    ctx.assemble_veff(dt(p.V), mu)
    ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
    return ctx


@pytest.mark.parametrize("c", [2, 3, pytest.param(4, marks=pytest.mark.slow)])
def test_pencil_eig_matches_oracle(c):
    """C4 (D = 745) is the pencil bench.py times after the step (next1_ms); C5 (D = 1363) is checked in
    tests/test_gpu_fullsize.py."""
    p = gen.make_problem(c)
    ctx = _ctx(p, p.mu)
    Ut, _, _ = ctx.block_solve(dt(p.lam), dt(p.U))
    FA, FB = ctx.project_augmented(Ut)
    ev, Y = ctx.pencil_eig(FA, FB, p.N)
    assert ctx.sync() == 0
    FAh, FBh = FA.cpu().numpy(), FB.cpu().numpy()
    evo, Yo = oracle.pencil_eig(FAh, FBh, p.N)
    ev, Y = ev.cpu().numpy(), Y.cpu().numpy()
    assert np.all(np.abs(ev - evo) <= 1e-9 * np.abs(evo).max())
    scale = np.abs(FAh).max() + np.abs(ev).max() * np.abs(FBh).max()
    assert np.abs(FAh @ Y - (FBh @ Y) * ev).max() <= 1e-9 * scale
    assert np.abs(Y.T @ FBh @ Y - np.eye(p.N)).max() <= 1e-9


def test_pencil_eig_rank_deficient_is_reported():
    import paper_2404_19249_b200 as ks
    p = gen.make_problem(1)
    ctx = _ctx(p, p.mu)
    D = p.n_H + 2
    FA = torch.eye(D, dtype=torch.float64, device=DEV)
    FB = torch.eye(D, dtype=torch.float64, device=DEV)
    FB[D - 1, D - 1] = -1.0
    with pytest.raises(ks.KSError) as e:
        ctx.pencil_eig(FA, FB, 2)
    assert e.value.status == ks.KS_E_RANK


@pytest.mark.parametrize("c,k", [(2, 4), (3, 8), (2, 3)])
def test_lift_matches_oracle(c, k):
    p = gen.make_problem(c)
    ctx = _ctx(p, p.mu)
    om = oracle.Mesh.from_problem(p)
    rng = np.random.default_rng(c * 10 + k)
    Ut = rng.standard_normal((p.n_free, p.N))
    Y = rng.standard_normal((p.n_H + p.N, k))
    Un = ctx.lift(dt(Ut), dt(Y)).cpu().numpy()
    ref = om.lift(p.n_H, p.P_rowptr, p.P_col, p.P_val, Ut, Y)
    import scipy.sparse as sp
    P = sp.csr_matrix((p.P_val, p.P_col, p.P_rowptr), shape=(p.n_free, p.n_H))
    bound = abs(P) @ np.abs(Y[:p.n_H]) + np.abs(Ut) @ np.abs(Y[p.n_H:])
    assert np.all(np.abs(Un - ref) <= 1e-12 * bound)


def test_augmented_solve_converges_like_the_oracle():
    """The outer loop of Algorithm 3 on the harmonic oscillator (fixed potential): the GPU's Ritz values
    converge to the brute-force fine eigenvalues, iterate by iterate within 1e-9 of the oracle's loop."""
    p = gen.make_problem(dict(L=5.0, n=10, grading=None, jitter=0.15, nuclei=[((0.0, 0.0, 0.0), 1)],
                              vnoise=0.0, N=4, orbitals="gauss", lam=("const", 2.0), nc=5, seed=9,
                              potential="harmonic"))
    mu = 0.0
    xf = p.xyz[p.free_nodes]
    ctr = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    U0 = np.ascontiguousarray(np.stack([np.exp(-0.5 * ((xf - c) ** 2).sum(1)) for c in ctr], axis=1))
    ctx = _ctx(p, mu)
    lam, U = dt(p.lam), dt(U0)
    outer, hist = ctx.augmented_solve(lam, U, tol_eig=1e-12, max_outer=60, tol_bvp=1e-12)
    assert ctx.sync() == 0
    om = oracle.Mesh.from_problem(p)
    om.assemble_veff(p.V, mu)
    H, M = om.csr("H").toarray(), om.csr("M").toarray()
    w = sl.eigh(H, M, eigvals_only=True)[:p.N]
    lam_h = lam.cpu().numpy()
    assert np.all(np.abs(lam_h - w) <= 1e-9 * np.abs(w).max()), (lam_h, w)
    # the oracle's loop, iterate by iterate (same inputs; the Ritz values of the first iterations agree
    # to the solver tolerance before rounding differences can matter)
    lo, Uo = p.lam.copy(), U0.copy()
    for it in range(min(outer, 8)):
        lo, Uo, _ = oracle.augmented_step(om, p.n_H, p.P_rowptr, p.P_col, p.P_val, lo, Uo, tol=1e-12)
        assert np.all(np.abs(hist[it] - lo) <= 1e-9 * np.abs(lo).max()), (it, hist[it], lo)
    Uh = U.cpu().numpy()
    assert np.abs(Uh.T @ M @ Uh - np.eye(p.N)).max() < 1e-8


@pytest.mark.parametrize("c", [2, 3])
def test_filtered_and_dense_pencil_solvers_agree(c, monkeypatch):
    """ks_pencil_eig's Chebyshev-filtered subspace iteration (default when k + 8 <= D / 2) and the dense
    cuSOLVER path (KS_PENCIL_DENSE=1) give the same eigenvalues and the same eigenvectors up to sign."""
    p = gen.make_problem(c)
    ctx = _ctx(p, p.mu)
    Ut, _, _ = ctx.block_solve(dt(p.lam), dt(p.U))
    FA, FB = ctx.project_augmented(Ut)
    ev_f, Y_f = ctx.pencil_eig(FA, FB, p.N)
    monkeypatch.setenv("KS_PENCIL_DENSE", "1")
    ev_d, Y_d = ctx.pencil_eig(FA, FB, p.N)
    assert ctx.sync() == 0
    ev_f, ev_d = ev_f.cpu().numpy(), ev_d.cpu().numpy()
    assert np.all(np.abs(ev_f - ev_d) <= 1e-10 * np.abs(ev_d).max())
    O = Y_f.cpu().numpy().T @ FB.cpu().numpy() @ Y_d.cpu().numpy()
    gaps = np.diff(ev_d)
    simple = np.ones(p.N, bool)
    simple[1:] &= gaps > 1e-6 * np.abs(ev_d).max()
    simple[:-1] &= gaps > 1e-6 * np.abs(ev_d).max()
    assert np.all(np.abs(np.abs(np.diag(O))[simple] - 1.0) <= 1e-8)


def test_pencil_eig_random_pencil_any_start():
    """A random SPD pencil, where the start block (unit vectors on the last k coordinates) carries no
    information: the filtered iteration still converges (or falls back to the dense path) to scipy's answer."""
    rng = np.random.default_rng(3)
    D, k = 300, 8
    Q = rng.standard_normal((D, D))
    FA = Q @ np.diag(np.linspace(-5.0, 5.0, D)) @ Q.T / D
    Bm = rng.standard_normal((D, D))
    FB = Bm @ Bm.T / D + np.eye(D)
    p = gen.make_problem(1)
    ctx = _ctx(p, p.mu)
    ev, Y = ctx.pencil_eig(dt(FA), dt(FB), k)
    assert ctx.sync() == 0
    ref = sl.eigh(FA, FB, eigvals_only=True)[:k]
    ev, Y = ev.cpu().numpy(), Y.cpu().numpy()
    assert np.all(np.abs(ev - ref) <= 1e-9 * np.abs(ref).max())
    assert np.abs(Y.T @ FB @ Y - np.eye(k)).max() <= 1e-9
    assert np.abs(FA @ Y - (FB @ Y) * ev).max() <= 1e-9 * (np.abs(FA).max() + np.abs(ev).max() * np.abs(FB).max())


def test_pencil_eig_falls_back_to_the_dense_path(monkeypatch):
    """A filtered iteration stopped before convergence (KS_PENCIL_EF_MAXIT=1) falls back to the dense
    cuSOLVER path on fresh copies of F_A, F_B: the same eigenpairs as KS_PENCIL_DENSE=1."""
    p = gen.make_problem(2)
    ctx = _ctx(p, p.mu)
    Ut, _, _ = ctx.block_solve(dt(p.lam), dt(p.U))
    FA, FB = ctx.project_augmented(Ut)
    monkeypatch.setenv("KS_PENCIL_EF_MAXIT", "1")
    ev_f, Y_f = ctx.pencil_eig(FA, FB, p.N)
    monkeypatch.delenv("KS_PENCIL_EF_MAXIT")
    monkeypatch.setenv("KS_PENCIL_DENSE", "1")
    ev_d, Y_d = ctx.pencil_eig(FA, FB, p.N)
    assert ctx.sync() == 0
    assert torch.equal(ev_f, ev_d) and torch.equal(Y_f, Y_d)


@pytest.mark.parametrize("c", [2, 3, 4])
@pytest.mark.parametrize("variant", ["KS_PENCIL_DEVICE=1", "KS_EF_HOSTEIG=jacobi", "KS_EF_GEMM=cublas", "KS_EF_RR=cublas"])
def test_filtered_loop_variants_agree(c, variant, monkeypatch):
    """The filtered iteration's variants give the same eigenvalues (1e-10 relative) and F_B-orthonormal eigenvectors
    that agree up to sign: the default (host Rayleigh-Ritz, cuBLAS filter) and the whole loop as one cooperative
    kernel (KS_PENCIL_DEVICE=1, ks_efdev.cu: Rayleigh-Ritz, convergence test and filter on the device), and the
    default loop with the host's small eigenproblems by cyclic Jacobi instead of Householder + QL
    (KS_EF_HOSTEIG=jacobi) or its D x D by D x m products by cuBLAS instead of k_sym_gemm (KS_EF_GEMM=cublas), or its
    Gram matrices, rotation and residuals by cuBLAS and k_resid instead of k_gram_pair and k_rotate_resid
    (KS_EF_RR=cublas). Each is bitwise reproducible."""
    p = gen.make_problem(c)
    ctx = _ctx(p, p.mu)
    Ut, _, _ = ctx.block_solve(dt(p.lam), dt(p.U))
    FA, FB = ctx.project_augmented(Ut)
    ev_d, Y_d = ctx.pencil_eig(FA, FB, p.N)
    name, val = variant.split("=")
    monkeypatch.setenv(name, val)
    ev_1, Y_1 = ctx.pencil_eig(FA, FB, p.N)
    ev_2, Y_2 = ctx.pencil_eig(FA, FB, p.N)
    assert ctx.sync() == 0
    assert torch.equal(ev_1, ev_2) and torch.equal(Y_1, Y_2)
    ev_1, ev_d = ev_1.cpu().numpy(), ev_d.cpu().numpy()
    assert np.all(np.abs(ev_1 - ev_d) <= 1e-10 * np.abs(ev_d).max())
    B = FB.cpu().numpy()
    Y1, Yd = Y_1.cpu().numpy(), Y_d.cpu().numpy()
    assert np.abs(Y1.T @ B @ Y1 - np.eye(p.N)).max() <= 1e-10
    assert np.abs(Yd.T @ B @ Yd - np.eye(p.N)).max() <= 1e-10
    O = Y1.T @ B @ Yd
    gaps = np.diff(ev_d)
    simple = np.ones(p.N, bool)
    simple[1:] &= gaps > 1e-6 * np.abs(ev_d).max()
    simple[:-1] &= gaps > 1e-6 * np.abs(ev_d).max()
    assert np.all(np.abs(np.abs(np.diag(O))[simple] - 1.0) <= 1e-8)
