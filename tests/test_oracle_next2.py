"""Pins of the NEXT-2 oracle functions: the LDA exchange / Perdew-Zunger correlation
potential and the nodal density (reading R6). Independent checks:
  * the potential is the density derivative of the energy density, v_xc = d(rho eps_xc)/d rho, on both sides
    of the r_s = 1 switch (finite differences of the oracle's own energy against its potential: the two
    formulas are printed separately in the paper);
  * textbook constants: Dirac exchange eps_x = -0.458165 / r_s (Hartree), the PZ (Ceperley-Alder) correlation
    eps_c(r_s = 1) = -0.0596 with the two branches meeting there to ~1e-4, and the Gell-Mann-Brueckner
    high-density limit eps_c -> A ln r_s + B, A = 0.0311 = (1 - ln 2) / pi^2;
  * rho <= 0 gives zero potential; the density of unit orbitals is the occupation."""
import numpy as np
import pytest

import gen
import oracle

def rho_of_rs(rs):
    return 3.0 / (4.0 * np.pi * np.asarray(rs, dtype=float) ** 3)


def test_potential_is_the_derivative_of_the_energy_density():
    rs = np.concatenate([np.linspace(0.05, 0.95, 19), np.linspace(1.05, 20.0, 20)])
    rho = rho_of_rs(rs)
    v, _ = oracle.vxc(rho)
    h = 1e-6 * rho
    _, ep = oracle.vxc(rho + h)
    _, em = oracle.vxc(rho - h)
    dnum = ((rho + h) * ep - (rho - h) * em) / (2 * h)
    assert np.all(np.abs(dnum - v) <= 1e-7 * np.abs(v))


def test_textbook_constants():
    # Dirac exchange energy per electron: -(3/4)(3/pi)^(1/3) rho^(1/3) = -0.458165.../r_s
    cx = 0.75 * (9.0 / (4.0 * np.pi ** 2)) ** (1.0 / 3.0)
    assert abs(cx - 0.4581652932831429) < 1e-15
    # at r_s = 1: eps_xc = -0.458165 + eps_c(1), eps_c(1) = -0.0596 (both PZ branches meet there)
    _, e1 = oracle.vxc(rho_of_rs([1.0]))
    assert abs(e1[0] - (-cx + (-0.05963))) < 2e-4
    _, ea = oracle.vxc(rho_of_rs([1.0 - 1e-12]))
    assert abs(ea[0] - e1[0]) < 1e-4
    # high density: eps_c -> A ln r_s + B with A = (1 - ln 2)/pi^2 (Gell-Mann-Brueckner)
    for rs in (1e-3, 1e-2):
        _, e = oracle.vxc(rho_of_rs([rs]))
        ec = e[0] + cx / rs
        assert abs(ec - ((1 - np.log(2)) / np.pi ** 2 * np.log(rs) - 0.048)) < 2e-3 + 0.0116 * rs


def test_no_electrons_no_potential():
    v, e = oracle.vxc(np.array([0.0, -1e-3]))
    assert np.all(v == 0.0) and np.all(e == 0.0)


def test_density_of_unit_orbitals():
    p = gen.make_problem(dict(L=2.0, n=4, grading=None, jitter=0.1, nuclei=[((0.0, 0.0, 0.0), 1)], vnoise=0.0,
                              N=2, orbitals="gauss", lam=("const", -0.5), nc=2, seed=1))
    m = oracle.Mesh.from_problem(p)
    U = np.zeros((p.n_free, 2))
    U[3, 0] = 1.0
    U[3, 1] = 0.5
    U[7, 1] = -2.0
    rho = m.density(U, f=2.0)
    expect = np.zeros(p.n_nodes)
    expect[p.free_nodes[3]] = 2.0 * (1.0 + 0.25)
    expect[p.free_nodes[7]] = 2.0 * 4.0
    assert np.array_equal(rho, expect)


def _gauss_box(n, L=8.0):
    return gen.make_problem(dict(L=L, n=n, grading=None, jitter=0.0, nuclei=[((0.0, 0.0, 0.0), 1)], vnoise=0.0, N=1,
                                 orbitals="exp", lam=("const", -0.5), nc=2, seed=1))


def _gaussians(xyz, centres, charges, sig=1.0):
    """density of Gaussian charges and their exact potential sum_k Q_k erf(r_k / (sqrt 2 sig)) / r_k"""
    from scipy.special import erf
    rho = np.zeros(xyz.shape[0])
    pot = np.zeros(xyz.shape[0])
    for c, q in zip(centres, charges):
        r = np.sqrt(((xyz - np.asarray(c)) ** 2).sum(1))
        rho += q * (2 * np.pi * sig ** 2) ** -1.5 * np.exp(-r ** 2 / (2 * sig ** 2))
        pot += q * erf(r / (np.sqrt(2) * sig)) / np.maximum(r, 1e-300)
    return rho, pot


def test_hartree_converges_to_the_exact_potential_of_a_gaussian_charge():
    """-Lap V = 4 pi rho for a Gaussian charge Q = 2 about c: V = Q erf(|x-c|/sqrt2)/|x-c| (textbook); the P1
    solution with multipole boundary data converges at O(h^2); moments: Q, centre c, zero dipole."""
    errs = []
    for n in (16, 32):
        p = _gauss_box(n)
        m = oracle.Mesh.from_problem(p)
        rho, exact = _gaussians(p.xyz, [(0.3, -0.2, 0.1)], [2.0])
        vh, mom, it = m.hartree(rho, tol=1e-12)
        assert abs(mom[0] - 2.0) < 1e-3 and np.allclose(mom[1:4], [0.3, -0.2, 0.1], atol=1e-3)
        assert np.abs(mom[4:7]).max() < 1e-12
        bd = p.dirichlet == 1
        assert np.abs(vh[bd] - exact[bd]).max() < 1e-3
        errs.append(np.abs(vh - exact).max())
    assert errs[0] / errs[1] > 3.0, errs      # h halves: O(h^2) -> ~4


def test_hartree_boundary_multipoles_capture_the_quadrupole():
    """Two equal Gaussian charges at (+-1.5, 0, 0): zero dipole about the centre, a strong quadrupole. The
    multipole boundary data (with the 1/2 of the Taylor expansion, reading R5) must match the exact potential
    far better than the size of the quadrupole term itself (a wrong factor would leave an error of that size)."""
    p = _gauss_box(24, L=10.0)
    m = oracle.Mesh.from_problem(p)
    rho, exact = _gaussians(p.xyz, [(1.5, 0.0, 0.0), (-1.5, 0.0, 0.0)], [1.0, 1.0])
    vh, mom, _ = m.hartree(rho, tol=1e-12)
    bd = p.dirichlet == 1
    r = np.sqrt((p.xyz[bd] ** 2).sum(1))
    mono = mom[0] / r
    quad_size = np.abs(exact[bd] - mono).max()
    assert quad_size > 1e-3
    assert np.abs(vh[bd] - exact[bd]).max() < 0.1 * quad_size


def test_anderson_depth_one_is_linear_mixing():
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal(50), rng.standard_normal(50)
    assert np.allclose(oracle.anderson_mix([a], [b], beta=0.7, depth=5), 0.7 * b + (1.0 - 0.7) * a, rtol=0, atol=1e-15)


def test_anderson_solves_a_linear_fixed_point_like_gmres():
    """For a linear map rho_out = G rho_in + c (contractive), Anderson mixing with beta = 1 and enough depth
    reaches the fixed point (I - G)^-1 c in at most dim + 1 steps (its equivalence with GMRES)."""
    rng = np.random.default_rng(1)
    d = 4
    G = 0.5 * rng.standard_normal((d, d)) / np.sqrt(d)
    c = rng.standard_normal(d)
    exact = np.linalg.solve(np.eye(d) - G, c)
    x = np.zeros(d)
    hin, hout = [], []
    for _ in range(d + 1):
        hin.append(x)
        hout.append(G @ x + c)
        x = oracle.anderson_mix(hin, hout, beta=1.0, depth=d + 1)
    assert np.abs(x - exact).max() < 1e-10


def test_scf_converges_to_the_fine_kohn_sham_solution():
    """Algorithm 3 (nonlinear, He-like: Z = 2, one doubly occupied orbital) on a graded fine mesh with a
    nonnested graded coarse mesh: at convergence the Ritz value is the lowest eigenvalue of the fine-mesh
    Kohn-Sham operator H[rho] assembled from the converged density (brute-force dense eigensolve), and the
    outer density change decays linearly."""
    import scipy.linalg as sl
    nuc = [((0.0, 0.0, 0.0), 2)]
    mk = lambda n: gen.make_problem(dict(L=8.0, n=n, grading=("power", 1.8), jitter=0.0, nuclei=nuc, vnoise=0.0,
                                         N=1, orbitals="gauss", lam=("const", -0.9), nc=2, seed=2))
    p, c = mk(12), mk(6)
    rp, col, val, nH = oracle.interpolation(p.xyz, p.free_nodes, c.xyz, c.tets, c.dirichlet)
    m = oracle.Mesh.from_problem(p)
    r = oracle.scf_solve(m, nH, rp, col, val, p.V, p.lam.copy(), p.U.copy(), mu=2.0, tol=1e-9, max_outer=60,
                         inner=30)
    assert r["dres"][-1] <= 1e-9 and r["outer"] < 60
    vh, _, _ = m.hartree(r["rho"], tol=1e-13)
    m.assemble_veff(p.V + vh + oracle.vxc(r["rho"])[0], 2.0)
    w = sl.eigh(m.csr("H").toarray(), m.csr("M").toarray(), eigvals_only=True)[0]
    assert abs(r["lam"][0] - w) < 1e-7 * abs(w), (r["lam"], w)
    tail = r["dres"][-6:]
    assert np.all(tail[1:] < tail[:-1])
