"""NEXT-2 on the GPU: nodal density, LDA/PZ exchange-correlation potential and the Hartree
potential through the C ABI against the oracle (tests/test_oracle_next2.py pins it).
Tolerances: density and V_xc |d| <= 1e-14 relative (the same pointwise formulas; libdevice vs libm
cbrt/log differ by an ulp); Hartree moments 1e-10 x (1 + |m|): the a-priori bound of a sum of ~3e5 element
terms in two different orders (reading R9); potential max |d| <= 1e-9 max |V_H| (both PCGs to
1e-12); the SCF loop Ritz values 1e-9 relative, outer iteration by outer iteration."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
DEV = "cuda"


def dt(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _ctx(p):
    import paper_2404_19249_b200 as ks
    return ks.Context(p.xyz, p.tets, p.dirichlet)


@pytest.mark.parametrize("c", [1, 2])
def test_density_and_vxc_match_oracle(c):
    p = gen.make_problem(c)
    ctx = _ctx(p)
    om = oracle.Mesh.from_problem(p)
    rho = ctx.density(dt(p.U), f=2.0)
    v, e = ctx.vxc(rho)
    rho_o = om.density(p.U, f=2.0)
    assert np.all(np.abs(rho.cpu().numpy() - rho_o) <= 1e-14 * np.abs(rho_o))
    v_o, e_o = oracle.vxc(rho_o)
    assert np.all(np.abs(v.cpu().numpy() - v_o) <= 1e-14 * np.abs(v_o) + 1e-300)
    assert np.all(np.abs(e.cpu().numpy() - e_o) <= 1e-14 * np.abs(e_o) + 1e-300)
    # a density sweep across the r_s = 1 switch and tiny / zero densities
    rs = np.concatenate([np.geomspace(1e-3, 0.999, 40), np.geomspace(1.0, 50.0, 40)])
    r = np.zeros(p.n_nodes)
    r[:rs.size] = 3.0 / (4.0 * np.pi * rs ** 3)
    v, e = ctx.vxc(dt(r))
    v_o, e_o = oracle.vxc(r)
    assert np.all(np.abs(v.cpu().numpy() - v_o) <= 1e-14 * np.abs(v_o) + 1e-300)


@pytest.mark.parametrize("n,centre", [(16, (0.3, -0.2, 0.1)), (24, (1.0, 0.5, -0.7))])
def test_hartree_matches_oracle(n, centre):
    from scipy.special import erf
    p = gen.make_problem(dict(L=8.0, n=n, grading=None, jitter=0.1, nuclei=[((0.0, 0.0, 0.0), 1)], vnoise=0.0, N=1,
                              orbitals="exp", lam=("const", -0.5), nc=2, seed=4))
    r = np.sqrt(((p.xyz - np.asarray(centre)) ** 2).sum(1))
    rho = 2.0 * (2 * np.pi) ** -1.5 * np.exp(-r ** 2 / 2)
    ctx = _ctx(p)
    vh, mom, it = ctx.hartree(dt(rho), tol=1e-12)
    assert ctx.sync() == 0
    om = oracle.Mesh.from_problem(p)
    vh_o, mom_o, it_o = om.hartree(rho, tol=1e-12)
    # sums over ~10^5..10^6 element terms in different orders (block tree vs sequential): the worst-case
    # rounding bound (n_terms - 1) u sum|terms| ~ 3.7e-11 (1 + |m|) at n = 24 (reading R9)
    assert np.all(np.abs(mom[:4] - mom_o[:4]) <= 1e-10 * (1 + np.abs(mom_o[:4])))
    assert np.all(np.abs(mom[4:] - mom_o[4:]) <= 1e-10 * (1 + np.abs(mom_o[7:]).max()))
    vg = vh.cpu().numpy()
    assert np.abs(vg - vh_o).max() <= 1e-9 * np.abs(vh_o).max()
    assert abs(it - it_o) <= 3
    # and the physics: close to the exact potential of the Gaussian charge
    exact = 2.0 * erf(r / np.sqrt(2)) / np.maximum(r, 1e-300)
    assert np.abs(vg - exact).max() < 0.2


@pytest.mark.parametrize("c", [1, 2])
def test_hartree_two_level_matches_oracle(c, monkeypatch):
    """With a coarse space set, ks_hartree runs the two-level preconditioned CG (Jacobi + coarse correction
    P (P^T K P)^-1 P^T, ks_pcg2l.cu): the same potential as the oracle's Jacobi-PCG within the solve
    tolerance, in fewer iterations, bitwise reproducible; KS_HARTREE_2L=0 falls back to Jacobi."""
    p = gen.make_problem(c)
    ctx = _ctx(p)
    ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
    xf = p.xyz
    r = np.sqrt(((xf - np.array([0.3, -0.2, 0.1])) ** 2).sum(1))
    rho = 2.0 * (2 * np.pi) ** -1.5 * np.exp(-r ** 2 / 2)
    vh, mom, it2 = ctx.hartree(dt(rho), tol=1e-12)
    vh_b, _, it2b = ctx.hartree(dt(rho), tol=1e-12)
    assert ctx.sync() == 0
    assert torch.equal(vh, vh_b) and it2 == it2b
    om = oracle.Mesh.from_problem(p)
    vh_o, _, it_o = om.hartree(rho, tol=1e-12)
    assert np.abs(vh.cpu().numpy() - vh_o).max() <= 1e-9 * np.abs(vh_o).max()
    assert it2 < it_o
    monkeypatch.setenv("KS_HARTREE_2L", "0")
    vh_j, _, it_j = ctx.hartree(dt(rho), tol=1e-12)
    assert abs(it_j - it_o) <= 3
    assert np.abs(vh_j.cpu().numpy() - vh_o).max() <= 1e-9 * np.abs(vh_o).max()


def test_hartree_warm_start_reaches_the_same_potential():
    p = gen.make_problem(1)
    ctx = _ctx(p)
    rho = ctx.density(dt(p.U), f=2.0)
    vh, _, it_cold = ctx.hartree(rho, tol=1e-12)
    vh2 = vh.clone()
    vh2, _, it_warm = ctx.hartree(rho, tol=1e-12, vh=vh2, warm=True)
    assert it_warm <= 1
    assert torch.allclose(vh, vh2, rtol=1e-10, atol=0)


def test_scf_solve_matches_the_oracle_loop():
    """Algorithm 3 for a He-like system (Z = 2, one doubly occupied orbital) with a nonnested graded coarse
    mesh: the GPU driver (ks_scf_solve, with P from ks_interpolation) against oracle.scf_solve (P from the
    oracle's point location), outer iteration by outer iteration."""
    nuc = [((0.0, 0.0, 0.0), 2)]
    mk = lambda n: gen.make_problem(dict(L=8.0, n=n, grading=("power", 1.8), jitter=0.0, nuclei=nuc, vnoise=0.0,
                                         N=1, orbitals="gauss", lam=("const", -0.9), nc=2, seed=2))
    p, c = mk(12), mk(6)
    ctx = _ctx(p)
    rp, col, val, nH = ctx.interpolation(c.xyz, c.tets, c.dirichlet)
    ctx.set_coarse(nH, rp, col, val)
    lam, U = dt(p.lam), dt(p.U)
    out = ctx.scf_solve(dt(p.V), lam, U, mu=2.0, tol=1e-9, max_outer=60, inner=30)
    assert ctx.sync() == 0
    om = oracle.Mesh.from_problem(p)
    orp, ocol, oval, onH = oracle.interpolation(p.xyz, p.free_nodes, c.xyz, c.tets, c.dirichlet)
    ref = oracle.scf_solve(om, onH, orp, ocol, oval, p.V, p.lam.copy(), p.U.copy(), mu=2.0, tol=1e-9, max_outer=60,
                           inner=30)
    assert abs(out["outer"] - ref["outer"]) <= 1
    k = min(out["outer"], ref["outer"])
    assert np.all(np.abs(out["lams"][:3] - ref["lams"][:3]) <= 1e-8 * np.abs(ref["lams"][:3]))
    assert abs(lam.cpu().numpy()[0] - ref["lam"][0]) <= 1e-8 * abs(ref["lam"][0])
    assert out["dres"][-1] <= 1e-9


@pytest.mark.slow
def test_scf_solve_four_orbitals_matches_the_oracle_loop():
    """Algorithm 3 with N = 4 doubly occupied orbitals (four Z = 3 centres, no symmetry) on a graded 24^3 fine
    mesh with an independent graded 6^3 coarse mesh: GPU (ks_scf_solve, P from ks_interpolation) against
    oracle.scf_solve, every outer iteration's Ritz values within 1e-9 relative. (The coarse mesh is small so the
    oracle's Jacobi eigensolves of every inner step stay cheap: D = 125 + 4.)"""
    nuc = [((1.1, 0.3, -0.2), 3), ((-1.2, 0.2, 0.4), 3), ((0.2, 1.3, 0.1), 3), ((0.1, -1.0, -0.9), 3)]
    mk = lambda n: gen.make_problem(dict(L=9.0, n=n, grading=("power", 1.5), jitter=0.0, nuclei=nuc, vnoise=0.0,
                                         N=4, orbitals="gauss", lam=("uniform", -2.0, -0.5), nc=2, seed=9))
    p, c = mk(24), mk(6)
    assert p.n_free >= 23 ** 3
    ctx = _ctx(p)
    rp, col, val, nH = ctx.interpolation(c.xyz, c.tets, c.dirichlet)
    ctx.set_coarse(nH, rp, col, val)
    lam, U = dt(p.lam), dt(p.U)
    out = ctx.scf_solve(dt(p.V), lam, U, mu=6.0, tol=1e-10, max_outer=120, inner=30)
    assert ctx.sync() == 0
    om = oracle.Mesh.from_problem(p)
    orp, ocol, oval, onH = oracle.interpolation(p.xyz, p.free_nodes, c.xyz, c.tets, c.dirichlet)
    assert onH == nH
    ref = oracle.scf_solve(om, onH, orp, ocol, oval, p.V, p.lam.copy(), p.U.copy(), mu=6.0, tol=1e-10,
                           max_outer=120, inner=30)
    assert abs(out["outer"] - ref["outer"]) <= 1
    # outer iteration by outer iteration while both took the same inner steps (the same path up to rounding)
    k = 0
    while k < min(out["outer"], ref["outer"]) and out["inner"][k] == ref["inner"][k]:
        k += 1
    assert k >= 3
    scale = np.abs(ref["lams"][:k]).max()
    assert np.all(np.abs(out["lams"][:k] - ref["lams"][:k]) <= 1e-9 * scale)
    # the converged Ritz values
    assert np.all(np.abs(lam.cpu().numpy() - ref["lam"]) <= 1e-9 * np.abs(ref["lam"]).max())
    assert out["dres"][-1] <= 1e-10
