"""GPU parity at BASELINE.json's largest size (config C5: 7.19 M nodes, 103.6 M nnz, N = 32 orbitals,
~12 GB on the device) in the launch configuration bench.py times, on outputs the oracle can afford:
  - assembled operator (all 103.6 M entries of A) against the oracle, bound of DESIGN.md §2 Q12;
  - the block solve of all 32 columns on the GPU; the TRUE relative residual of every column
    (a property that holds at any size) and two sampled columns solved by the oracle one by one
    (M-norm difference <= 1e-8, iterations within +-2);
  - the projection of the GPU's U~ by both sides, every entry within 1e-9 (|W|^T |Op| |W|)_ij
    (tests/fbounds.py), and the lowest N pencil eigenvalues (GPU eigensolver on the GPU's F against
    LAPACK on the oracle's F) within 1e-9 max|lambda|.
The oracle's share is ~3 minutes of one CPU core; the test is marked slow."""
import numpy as np
import pytest

import scipy.linalg as sl

import gen
import oracle
from fbounds import assert_entrywise, projection_bounds

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")


def test_config5_sampled_parity():
    import paper_2404_19249_b200 as ks
    p = gen.make_problem(5)
    dev = torch.device("cuda", 0)
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet, max_N=p.N)
    ctx.assemble_veff(torch.from_numpy(p.V).to(dev), p.mu)
    ctx.set_coarse(p.n_H, torch.from_numpy(p.P_rowptr).to(dev), torch.from_numpy(p.P_col).to(dev),
                   torch.from_numpy(p.P_val).to(dev))
    lam = torch.from_numpy(p.lam).to(dev)
    U = torch.from_numpy(p.U).to(dev)
    Ut, iters, relres = ctx.block_solve(lam, U, tol=1e-10, max_iter=2000)
    true_rel = ctx.true_residual(lam, U, Ut)
    FA, FB = ctx.project_augmented(Ut)
    ev, _ = ctx.pencil_eig(FA, FB, p.N)
    assert ctx.sync() == 0, ctx.last_error()
    ev = ev.cpu().numpy()
    A_gpu = ctx.values()["A"].cpu().numpy()
    ut = Ut.cpu().numpy()
    it = iters.cpu().numpy()
    tr = true_rel.cpu().numpy()
    FA, FB = FA.cpu().numpy(), FB.cpu().numpy()
    del ctx, U, Ut
    torch.cuda.empty_cache()

    # every column converged to the tolerance (recursive residual), true residual at the same level
    assert np.all(relres.cpu().numpy() <= 1e-10)
    assert np.all(tr <= 1e-9), tr

    om = oracle.Mesh.from_problem(p)
    om.assemble_veff(p.V, p.mu)
    v = om.values()
    # |A_e| bound per entry: 0.5 |K| + |MV| + mu M with |K| <= (K_ii + K_jj)/2 and |MV| <= 2 M max|V|
    rp, col, _, _ = om.pattern()
    rows = np.repeat(np.arange(om.n_free), np.diff(rp))
    isdiag = rows == col
    Kd = np.zeros(om.n_free)
    Kd[rows[isdiag]] = v["K"][isdiag]
    bA = 0.5 * 0.5 * (Kd[rows] + Kd[col]) + v["M"] * (2.0 * np.abs(p.V).max() + p.mu)
    assert np.all(np.abs(A_gpu - v["A"]) <= 1e-12 * bA)
    del rows, isdiag, Kd, bA, A_gpu

    # two sampled columns solved by the oracle one by one
    M = om.csr("M")
    for c in (0, p.N - 1):
        ref = om.block_pcg(p.lam[c:c + 1], np.ascontiguousarray(p.U[:, c:c + 1]), tol=1e-10, max_iter=2000)
        d = ut[:, c] - ref["Ut"][:, 0]
        rel = np.sqrt(d @ (M @ d)) / np.sqrt(ref["Ut"][:, 0] @ (M @ ref["Ut"][:, 0]))
        assert rel <= 1e-8, (c, rel)
        assert abs(int(it[c]) - int(ref["iters"][0])) <= 2, (c, it[c], ref["iters"])

    # projection of the same U~ by both sides
    FAo, FBo = om.project(p.n_H, p.P_rowptr, p.P_col, p.P_val, ut)
    bA, bB = projection_bounds(om, p.n_H, p.P_rowptr, p.P_col, p.P_val, ut)
    assert_entrywise(FA, FAo, bA, what="F_A")
    assert_entrywise(FB, FBo, bB, what="F_B")
    wo = sl.eigh(FAo, FBo, eigvals_only=True, subset_by_index=[0, p.N - 1])
    assert np.all(np.abs(ev - wo) <= 1e-9 * np.abs(wo).max()), (ev, wo)
