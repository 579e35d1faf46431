"""Edge cases through the C ABI: a mesh whose nodes are all Dirichlet (no unknowns), a mesh with a single
free node, and the NEXT entry points on the smallest meshes. Each call must either do the (trivial) work
or fail with a status code -- never fault."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
DEV = "cuda"


def dt(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def box(n, L=1.0, N=1, nc=1):
    return gen.make_problem(dict(L=L, n=n, grading=None, jitter=0.0, nuclei=[((0.0, 0.0, 0.0), 1)], vnoise=0.0,
                                 N=N, orbitals="gauss", lam=("const", -0.5), nc=nc, seed=1))


def test_no_free_nodes_is_rejected_cleanly():
    import paper_2404_19249_b200 as ks
    p = box(1)                      # 8 nodes, all on the boundary
    assert p.n_free == 0
    try:
        ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
    except ks.KSError as e:
        assert e.status in (ks.KS_E_ARG, ks.KS_E_MESH)
        return
    # if accepted, the operations on an empty system must succeed trivially or report an argument error
    ctx.assemble_veff(dt(p.V), 1.0)
    assert ctx.sync() == 0


def test_single_free_node():
    import paper_2404_19249_b200 as ks
    p = box(2, N=1, nc=2)           # 27 nodes, 1 free (the centre)
    assert p.n_free == 1
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
    ctx.assemble_veff(dt(p.V), 8.0)
    Ut, it, rr = ctx.block_solve(dt(p.lam), dt(p.U), tol=1e-12)
    assert ctx.sync() == 0
    om = oracle.Mesh.from_problem(p)
    om.assemble_veff(p.V, 8.0)
    ref = om.block_pcg(p.lam, p.U, tol=1e-12)
    assert np.allclose(Ut.cpu().numpy(), ref["Ut"], rtol=1e-12, atol=0)
    # one unknown: the exact solve is b / A_11 and the projection pencil is 1 + 1 (coarse free node + orbital)
    if p.n_H >= 1:
        ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
        FA, FB = ctx.project_augmented(Ut)
        assert ctx.sync() == 0
        FAo, FBo = om.project(p.n_H, p.P_rowptr, p.P_col, p.P_val, ref["Ut"])
        assert np.allclose(FA.cpu().numpy(), FAo, rtol=1e-12, atol=1e-300)


def test_next_entry_points_on_a_small_mesh():
    """density / V_xc / Hartree / interpolation / pencil eig / lift on a 3^3-cell box."""
    import paper_2404_19249_b200 as ks
    p = box(3, L=2.0, N=2, nc=2)
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
    rho = ctx.density(dt(p.U), f=2.0)
    v, e = ctx.vxc(rho)
    vh, mom, it = ctx.hartree(rho, tol=1e-12)
    assert ctx.sync() == 0
    om = oracle.Mesh.from_problem(p)
    vh_o, mom_o, _ = om.hartree(om.density(p.U, 2.0), tol=1e-12)
    assert np.abs(vh.cpu().numpy() - vh_o).max() <= 1e-9 * np.abs(vh_o).max()
    c = box(2, L=2.0)
    rp, col, val, nH = ctx.interpolation(c.xyz, c.tets, c.dirichlet)
    orp, ocol, oval, onH = oracle.interpolation(p.xyz, p.free_nodes, c.xyz, c.tets, c.dirichlet)
    assert nH == onH and np.array_equal(rp.cpu().numpy(), orp)
    ctx.assemble_veff(dt(p.V), 8.0)
    ctx.set_coarse(nH, rp, col, val)
    Ut, _, _ = ctx.block_solve(dt(p.lam), dt(p.U), tol=1e-12)
    FA, FB = ctx.project_augmented(Ut)
    ev, Y = ctx.pencil_eig(FA, FB, p.N)
    Un = ctx.lift(Ut, Y)
    assert ctx.sync() == 0
    evo, _ = oracle.pencil_eig(FA.cpu().numpy(), FB.cpu().numpy(), p.N)
    assert np.allclose(ev.cpu().numpy(), evo, rtol=1e-9, atol=1e-12)
    assert np.all(np.isfinite(Un.cpu().numpy()))


def test_zero_inputs_stop_before_the_first_iteration(monkeypatch):
    """U = 0 (b = 0 in every column) and rho = 0 (no charge): the solvers stop at the initial check with exact
    zeros and no 0/0 -- the block PCG, and both Hartree paths (two-level with a coarse space, and Jacobi)."""
    import paper_2404_19249_b200 as ks
    p = box(6, L=2.0, N=3, nc=3)
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
    ctx.assemble_veff(dt(p.V), 5.0)
    U = torch.zeros((p.n_free, 3), dtype=torch.float64, device=DEV)
    Ut, iters, relres = ctx.block_solve(dt(p.lam), U)
    assert ctx.sync() == 0
    assert torch.count_nonzero(Ut) == 0 and torch.all(iters == 0) and torch.all(relres == 0)
    ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
    rho = torch.zeros(p.n_nodes, dtype=torch.float64, device=DEV)
    for env in ("1", "0"):
        monkeypatch.setenv("KS_HARTREE_2L", env)
        vh, mom, it = ctx.hartree(rho)
        assert ctx.sync() == 0
        assert it == 0 and torch.count_nonzero(vh) == 0 and np.all(mom == 0)
