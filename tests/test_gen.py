"""Input generator checks (counts, orientation, interpolation operator, shift formula)."""
import os

import numpy as np
import pytest

import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


@pytest.mark.parametrize("row", _rows("kuhn_counts.txt")[:3])
def test_counts_against_appendix(row):
    n, nodes, tets, free = (int(x) for x in row[:4])
    cfg = {16: 1, 32: 2, 64: 3}[n]
    p = gen.make_problem(cfg)
    assert p.n_nodes == nodes and p.n_tets == tets and p.n_free == free


def test_kuhn_orientation_and_volume():
    for c in (1, 2, 3):
        p = gen.make_problem(c)
        x = p.xyz[p.tets]
        vol = np.einsum("ij,ij->i", np.cross(x[:, 1] - x[:, 0], x[:, 2] - x[:, 0]), x[:, 3] - x[:, 0]) / 6
        assert vol.min() > 0
        assert abs(vol.sum() - (2 * p.L) ** 3) <= 1e-10 * (2 * p.L) ** 3  # SPEC.md:22-25 volume invariant


def test_box_faces_and_dirichlet():
    p = gen.make_problem(2)
    on = np.any(np.isclose(np.abs(p.xyz), p.L, rtol=0, atol=1e-12), axis=1)
    assert np.array_equal(on, p.dirichlet.astype(bool))
    # (0,1)^3 with n=2 leaves exactly one free node
    q = gen.make_problem(dict(L=1.0, n=2, grading=None, jitter=0.0, nuclei=[((0, 0, 0), 1)],
                              vnoise=0.0, N=1, orbitals="exp", lam=("const", -0.5), nc=2))
    assert q.n_free == 1


@pytest.mark.parametrize("row", _rows("mu_shift.txt"))
def test_mu_formula(row):
    name, charges, mu = row
    Z = [float(z) for z in charges.split(",")]
    cfg = dict(L=4.0, n=4, grading=None, jitter=0.0,
               nuclei=[((0.5 * k, 0.0, 0.0), z) for k, z in enumerate(Z)], vnoise=0.0, N=1,
               orbitals="exp", lam=("const", -0.5), nc=2)
    assert gen.make_problem(cfg).mu == float(mu)


def test_rng_counter_based():
    a = gen.uniform01(7, 3, np.arange(1000))
    b = gen.uniform01(7, 3, np.arange(500, 1000))
    assert np.array_equal(a[500:], b)
    assert 0.0 <= a.min() and a.max() < 1.0 and abs(a.mean() - 0.5) < 0.05


@pytest.mark.parametrize("c", [1, 2, 3])
def test_interpolation_reproduces_linears(c):
    """P_H = I_H^h (Alg. 1): for fine nodes whose coarse tet has only free vertices
    the rows are barycentric weights: sum to 1 and reproduce x, y, z exactly."""
    p = gen.make_problem(c)
    nc, L = p.nc, p.L
    Hc = 2 * L / nc
    m = nc - 1
    cf = np.arange(p.n_H)
    cx = np.stack([-L + Hc * (1 + cf % m), -L + Hc * (1 + (cf // m) % m), -L + Hc * (1 + cf // (m * m))], 1)
    rows = np.repeat(np.arange(p.n_free), np.diff(p.P_rowptr))
    s = np.bincount(rows, weights=p.P_val, minlength=p.n_free)
    full = np.isclose(s, 1.0, atol=1e-12)
    assert full.mean() > 0.1
    xf = p.xyz[p.free_nodes]
    for a in range(3):
        rec = np.bincount(rows, weights=p.P_val * cx[p.P_col, a], minlength=p.n_free)
        assert np.max(np.abs(rec[full] - xf[full, a])) < 1e-12 * L
    assert np.all(p.P_val > 0) and np.all(p.P_val <= 1 + 1e-15)
    assert np.all(np.diff(p.P_rowptr) <= 4)
