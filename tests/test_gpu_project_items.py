"""GPU parity of the A_H pass on the item-ordered sliced-ELL copy of the pattern (ks_project.cu k_proj_ai,
DESIGN.md §4.4) against the oracle and against k_proj_a (KS_PROJ_AI=0):

  * every entry of F_A, F_B within the per-entry bound of the oracle (reading Q12', tests/fbounds.py), at C2/C3
    and ragged N (NP = 8, 16, 32 tensor-core item passes and the FFMA ones);
  * F_A, F_B bitwise equal between the two A passes: k_proj_ai sums every window row and every k-step of the item
    contraction in k_proj_a's order (A_H = P^T H P, st5);
  * call orders around the coarse space (assemble before / after ks_set_coarse, a second coarse space rebuilding the
    item layout, a new assembly) all give the oracle's projection.
"""
import numpy as np
import pytest

import gen
import oracle
from fbounds import assert_entrywise, projection_bounds

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _ks():
    import paper_2404_19249_b200 as pkg
    return pkg


def dt(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def small(n=8, N=3, nc=3, **kw):
    cfg = dict(L=3.0, n=n, grading=None, jitter=0.2, nuclei=[((0.3, -0.2, 0.1), 2)], vnoise=0.05, N=N,
               orbitals="gauss", lam=("uniform", -2.0, -0.5), nc=nc, seed=77)
    cfg.update(kw)
    return gen.make_problem(cfg)


def check_against_oracle(ctx, om, p, Ut, what=""):
    FA, FB = ctx.project_augmented(dt(Ut))
    assert ctx.sync() == 0, ctx.last_error()
    FA, FB = FA.cpu().numpy(), FB.cpu().numpy()
    FAo, FBo = om.project(p.n_H, p.P_rowptr, p.P_col, p.P_val, Ut)
    bA, bB = projection_bounds(om, p.n_H, p.P_rowptr, p.P_col, p.P_val, Ut)
    assert_entrywise(FA, FAo, bA, what="F_A " + what)
    assert_entrywise(FB, FBo, bB, what="F_B " + what)
    return FA, FB


@pytest.mark.parametrize("case", ["c2", "c3", "N3", "N5", "N8", "N16", "N20", "N32"])
def test_item_layout_A_pass_matches_the_oracle_and_k_proj_a(case, monkeypatch):
    p = gen.make_problem(int(case[1])) if case[0] == "c" else small(N=int(case[1:]))
    om = oracle.Mesh.from_problem(p)
    om.assemble_veff(p.V, p.mu)
    ctx = _ks().Context(p.xyz, p.tets, p.dirichlet)
    ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
    ctx.assemble_veff(dt(p.V), p.mu)
    Ut = p.U + 0.1 * np.random.default_rng(5).standard_normal(p.U.shape)
    out = []
    for mode in ("1", "0", "1"):
        monkeypatch.setenv("KS_PROJ_AI", mode)
        out.append(check_against_oracle(ctx, om, p, Ut, what=f"KS_PROJ_AI={mode}"))
    for FA, FB in out[1:]:
        assert np.array_equal(FA, out[0][0]) and np.array_equal(FB, out[0][1])


def test_coarse_space_changes(monkeypatch):
    """assemble -> set_coarse, set_coarse with another coarse space (the item layout rebuilt), back, a new
    assembly: the projection is the oracle's after each."""
    monkeypatch.delenv("KS_PROJ_AI", raising=False)
    p2, p3 = small(N=8, nc=2), small(N=8, nc=3)
    assert np.array_equal(p2.xyz, p3.xyz) and np.array_equal(p2.V, p3.V)
    om = oracle.Mesh.from_problem(p2)
    om.assemble_veff(p2.V, p2.mu)
    ctx = _ks().Context(p2.xyz, p2.tets, p2.dirichlet)
    ctx.assemble_veff(dt(p2.V), p2.mu)
    Ut = p2.U + 0.1 * np.random.default_rng(9).standard_normal(p2.U.shape)
    for p in (p2, p3, p2):
        ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
        check_against_oracle(ctx, om, p, Ut, what=f"after set_coarse n_H={p.n_H}")
    V2 = p2.V + 0.3 * np.sin(np.arange(p2.V.size))
    om.assemble_veff(V2, 2.0 * p2.mu)
    ctx.assemble_veff(dt(V2), 2.0 * p2.mu)
    check_against_oracle(ctx, om, p2, Ut, what="after a new assembly")


def test_repeated_projections_reuse_A_H_until_H_or_its_storage_changes(monkeypatch):
    """A_H = P^T H P depends on H only: projections of one assembly reuse its item partials (the outer iterations of
    ks_augmented_solve), bitwise equal to a fresh computation; a two-level Hartree solve (which builds P^T K P in
    the same partial storage) and a new assembly invalidate them."""
    monkeypatch.delenv("KS_PROJ_AI", raising=False)
    p = small(N=8, nc=3)
    om = oracle.Mesh.from_problem(p)
    om.assemble_veff(p.V, p.mu)
    ctx = _ks().Context(p.xyz, p.tets, p.dirichlet)
    ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
    ctx.assemble_veff(dt(p.V), p.mu)
    rng = np.random.default_rng(11)
    U1 = p.U + 0.1 * rng.standard_normal(p.U.shape)
    U2 = p.U + 0.1 * rng.standard_normal(p.U.shape)
    F1 = check_against_oracle(ctx, om, p, U1, what="first")
    F2 = check_against_oracle(ctx, om, p, U2, what="second, reused A_H")
    nH = p.n_H
    assert np.array_equal(F1[0][:nH, :nH], F2[0][:nH, :nH])
    rho = ctx.density(dt(p.U), 2.0)
    ctx.hartree(rho, tol=1e-8)   # P^T K P through the same item partials
    F3 = check_against_oracle(ctx, om, p, U1, what="after a two-level Hartree solve")
    assert np.array_equal(F3[0], F1[0]) and np.array_equal(F3[1], F1[1])
    V2 = p.V + 0.2 * np.cos(np.arange(p.V.size))
    om.assemble_veff(V2, p.mu)
    ctx.assemble_veff(dt(V2), p.mu)
    check_against_oracle(ctx, om, p, U1, what="after a new assembly")
