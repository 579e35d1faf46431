"""Pins of the NEXT-3 oracle (oracle.interpolation: the nonnested P1 interpolation operator of Algorithm 1,
PAPER.md:499-548, by brute-force point location). Independent constructions: the structured-coarse-mesh
operator of gen (sorted fractional coordinates, no point location), exact reproduction of affine functions
(P1 interpolation is exact on them), the centroid of a single tet, and points outside the coarse mesh."""
import numpy as np
import pytest
import scipy.sparse as sp

import gen
import oracle


def coarse_kuhn(nc, L, jitter=0.0, seed=3):
    """Coarse Kuhn mesh of the box [-L, L]^3 (optionally with interior nodes jittered: unstructured and
    nonnested with respect to the fine mesh). Returns xyz, tets, dirichlet."""
    p = gen.make_problem(dict(L=L, n=nc, grading=None, jitter=jitter, nuclei=[((0.0, 0.0, 0.0), 1)], vnoise=0.0,
                              N=1, orbitals="exp", lam=("const", -0.5), nc=1, seed=seed))
    return p.xyz, p.tets, p.dirichlet


def dense(rp, col, val, nrows, ncols):
    return sp.csr_matrix((val, col, rp), shape=(nrows, ncols)).toarray()


@pytest.mark.parametrize("c", [1, 2])
def test_matches_structured_construction(c):
    p = gen.make_problem(c)
    xc, tc, dc = coarse_kuhn(p.nc, p.L)
    rp, col, val, nH = oracle.interpolation(p.xyz, p.free_nodes, xc, tc, dc)
    assert nH == p.n_H
    A = dense(rp, col, val, p.n_free, nH)
    B = dense(p.P_rowptr, p.P_col, p.P_val, p.n_free, p.n_H)
    assert np.abs(A - B).max() <= 1e-14
    assert np.array_equal(A != 0, B != 0)


def test_reproduces_affine_functions_on_unstructured_coarse_mesh():
    p = gen.make_problem(2)
    xc, tc, _ = coarse_kuhn(5, p.L, jitter=0.25, seed=8)       # jittered: nonnested, unstructured
    nodir = np.zeros(xc.shape[0], np.uint8)                     # keep every coarse vertex
    rp, col, val, nH = oracle.interpolation(p.xyz, p.free_nodes, xc, tc, nodir)
    P = sp.csr_matrix((val, col, rp), shape=(p.n_free, nH))
    xf = p.xyz[p.free_nodes]
    for coef in ([1.0, 0.0, 0.0, 0.0], [0.3, -1.2, 0.7, 2.0]):
        f_c = coef[0] + xc @ np.array(coef[1:])
        f_f = coef[0] + xf @ np.array(coef[1:])
        assert np.abs(P @ f_c - f_f).max() <= 1e-12 * (1 + np.abs(f_f).max())
    assert np.all(val >= -1e-12) and np.all(val <= 1 + 1e-12)
    assert np.all(np.diff(rp) <= 4)


def test_centroid_of_a_single_tet():
    xc = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    tc = np.array([[0, 1, 2, 3]], np.int32)
    q = xc.mean(0)[None, :]
    rp, col, val, nH = oracle.interpolation(q, np.array([0]), xc, tc, np.zeros(4, np.uint8))
    assert nH == 4 and list(col) == [0, 1, 2, 3]
    assert np.allclose(val, 0.25, rtol=0, atol=1e-15)
    # a Dirichlet vertex drops out of the row (zero data on the boundary)
    rp, col, val, nH = oracle.interpolation(q, np.array([0]), xc, tc, np.array([0, 1, 0, 0], np.uint8))
    assert nH == 3 and list(col) == [0, 1, 2] and np.allclose(val, 0.25)


def test_point_outside_is_an_error():
    xc = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    tc = np.array([[0, 1, 2, 3]], np.int32)
    with pytest.raises(oracle.OracleError):
        oracle.interpolation(np.array([[1.0, 1.0, 1.0]]), np.array([0]), xc, tc, np.zeros(4, np.uint8))
