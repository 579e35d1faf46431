"""NEXT-3 on the GPU: ks_interpolation (Algorithm 1) against the oracle's brute-force
point location and against gen's structured construction, then through the projection.
Tolerances: entries of P |d| <= 1e-12 (barycentric coordinates in [0, 1], computed from the same coordinates
in a different order); the sparsity pattern equal (no entry near the 1e-13 drop threshold in these inputs
is checked separately); projected blocks per entry <= 1e-9 x (|W|^T |Op| |W|)_ij (tests/fbounds.py)."""
import numpy as np
import pytest
import scipy.sparse as sp

import fbounds
import gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
DEV = "cuda"


def dt(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def coarse(nc, L, jitter=0.0, seed=3):
    p = gen.make_problem(dict(L=L, n=nc, grading=None, jitter=jitter, nuclei=[((0.0, 0.0, 0.0), 1)], vnoise=0.0,
                              N=1, orbitals="exp", lam=("const", -0.5), nc=1, seed=seed))
    return p.xyz, p.tets, p.dirichlet


def csr_dense(rp, col, val, n, m):
    return sp.csr_matrix((val, col, rp), shape=(n, m)).toarray()


@pytest.mark.parametrize("c,jitter", [(1, 0.0), (2, 0.0), (1, 0.2), (2, 0.25)])
def test_interpolation_matches_oracle(c, jitter):
    import paper_2404_19249_b200 as ks
    p = gen.make_problem(c)
    xc, tc, dc = coarse(p.nc + (1 if jitter else 0), p.L, jitter=jitter, seed=c + 7)
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
    rp, col, val, nH = ctx.interpolation(xc, tc, dc)
    rp, col, val = rp.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy()
    orp, ocol, oval, onH = oracle.interpolation(p.xyz, p.free_nodes, xc, tc, dc)
    assert nH == onH
    A, B = csr_dense(rp, col, val, p.n_free, nH), csr_dense(orp, ocol, oval, p.n_free, onH)
    assert np.abs(A - B).max() <= 1e-12
    assert np.array_equal(A != 0, B != 0)
    # rows sorted by coarse column
    for i in range(0, p.n_free, 97):
        assert np.all(np.diff(col[rp[i]:rp[i + 1]]) > 0)


def test_interpolation_full_size_equals_structured_construction():
    """C4 (2.05 M fine nodes, 10^3-cell coarse Kuhn mesh): the GPU operator equals gen's construction
    (sorted fractional coordinates, no point location) entry by entry."""
    import paper_2404_19249_b200 as ks
    p = gen.make_problem(4)
    xc, tc, dc = coarse(p.nc, p.L)
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
    rp, col, val, nH = ctx.interpolation(xc, tc, dc)
    assert nH == p.n_H
    assert np.array_equal(rp.cpu().numpy(), p.P_rowptr)
    assert np.array_equal(col.cpu().numpy(), p.P_col)
    assert np.abs(val.cpu().numpy() - p.P_val).max() <= 1e-13


def test_projection_with_unstructured_coarse_mesh():
    """The whole hot path on a nonnested, unstructured coarse mesh: P from ks_interpolation on the GPU,
    F_A, F_B against the oracle's projection with the oracle's P."""
    import paper_2404_19249_b200 as ks
    p = gen.make_problem(2)
    xc, tc, dc = coarse(5, p.L, jitter=0.25, seed=8)
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
    ctx.assemble_veff(dt(p.V), p.mu)
    rp, col, val, nH = ctx.interpolation(xc, tc, dc)
    ctx.set_coarse(nH, rp, col, val)
    rng = np.random.default_rng(2)
    Ut = p.U + 0.1 * rng.standard_normal(p.U.shape)
    FA, FB = ctx.project_augmented(dt(Ut))
    assert ctx.sync() == 0
    om = oracle.Mesh.from_problem(p)
    om.assemble_veff(p.V, p.mu)
    orp, ocol, oval, onH = oracle.interpolation(p.xyz, p.free_nodes, xc, tc, dc)
    FAo, FBo = om.project(onH, orp, ocol, oval, Ut)
    # per entry (Q12'), with the entries of |P| widened by 1e-3 on its pattern: the GPU's P differs from
    # the oracle's by <= 1e-12 per entry (above), i.e. 1e-9 x 1e-3, and that difference propagates linearly
    n = Ut.shape[0]
    Pg = sp.csr_matrix((val.cpu().numpy(), col.cpu().numpy(), rp.cpu().numpy()), shape=(n, nH))
    Po = sp.csr_matrix((oval, ocol, orp), shape=(n, onH))
    assert nH == onH and abs(Pg - Po).max() <= 1e-12 and ((Pg != 0) != (Po != 0)).nnz == 0
    P_abs = sp.csr_matrix((np.abs(oval) + 1e-3, ocol, orp), shape=(n, nH))
    for F, Fo, op in ((FA.cpu().numpy(), FAo, "H"), (FB.cpu().numpy(), FBo, "M")):
        fbounds.assert_entrywise(F, Fo, fbounds.abs_gram(P_abs, np.abs(Ut), abs(om.csr(op))), 1e-9, "F_" + op)
