"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element, on the same
seeded inputs. Tolerances (reading Q12, BASELINE.json north_star):
  pattern, emap, inverse map, free numbering: bit-exact
  K, M, M_V, H, A, diag: |delta| <= 1e-12 * (sum of |element contributions| bound) per entry
  SpMM: |delta_ij| <= 1e-12 * (|Op| |X|)_ij
  block solve: ||u~_gpu - u~_oracle||_M / ||u~_oracle||_M <= 1e-8 per column at tol 1e-10,
               iteration counts within +-2
  projection: every entry |dF_ij| <= 1e-9 (|W|^T |Op| |W|)_ij, W = [P | U~] (tests/fbounds.py, Q12');
              pencil eigenvalues within 1e-9 max|lambda|.
"""
import numpy as np
import pytest
import scipy.linalg as sl
import scipy.sparse as sp

import gen
import oracle
from fbounds import assert_entrywise, projection_bounds

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _ks():
    import paper_2404_19249_b200 as pkg
    return pkg


DEV = "cuda"


def dt(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


class Case:
    def __init__(self, p, assemble=True, coarse=True):
        self.p = p
        self.om = oracle.Mesh.from_problem(p)
        self.ctx = _ks().Context(p.xyz, p.tets, p.dirichlet)
        if assemble:
            self.om.assemble_veff(p.V, p.mu)
            self.ctx.assemble_veff(dt(p.V), p.mu)
        if coarse:
            self.ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))


_cache = {}


def case(c):
    if c not in _cache:
        _cache[c] = Case(gen.make_problem(c))
    return _cache[c]


def small(n=5, N=3, **kw):
    cfg = dict(L=3.0, n=n, grading=None, jitter=0.2, nuclei=[((0.3, -0.2, 0.1), 2)], vnoise=0.05, N=N,
               orbitals="gauss", lam=("uniform", -2.0, -0.5), nc=2, seed=77)
    cfg.update(kw)
    return gen.make_problem(cfg)


# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("c", [1, 2, 3])
def test_pattern_and_maps_bit_exact(c):
    k = case(c)
    rp, col, emap, fon = k.om.pattern()
    g_rp, g_col, g_emap, g_fon, g_iptr, g_iidx = (t.cpu().numpy() for t in k.ctx.pattern())
    assert np.array_equal(g_rp, rp.astype(np.int32))
    assert np.array_equal(g_col, col)
    assert np.array_equal(g_emap, emap)
    assert np.array_equal(g_fon, fon)
    # inverse map: emap indices grouped by target, ascending
    valid = np.nonzero(emap >= 0)[0]
    order = valid[np.argsort(emap[valid], kind="stable")]
    assert np.array_equal(g_iidx, order.astype(np.int32))
    assert np.array_equal(g_iptr, np.searchsorted(emap[order], np.arange(k.om.nnz + 1)).astype(np.int32))


def _value_bounds(k):
    """Per-entry bounds on sum_T |element contribution| (so 1e-12 x bound is a relative tolerance that
    survives cancellation): |K_T(a,b)| <= (K_T(a,a) + K_T(b,b))/2, M_T > 0, |MV_T| <= 2 M_T max|V|."""
    v = k.om.values()
    rp, col, _, _ = k.om.pattern()
    rows = np.repeat(np.arange(k.om.n_free), np.diff(rp))
    isdiag = rows == col
    Kd = np.zeros(k.om.n_free)
    Kd[rows[isdiag]] = v["K"][isdiag]
    bK = 0.5 * (Kd[rows] + Kd[col])
    vmax = np.abs(k.p.V).max()
    bM = v["M"]
    bMV = 2.0 * v["M"] * vmax
    return v, bK, bM, bMV


@pytest.mark.parametrize("c", [1, 2, 3])
def test_assembled_values(c):
    k = case(c)
    v, bK, bM, bMV = _value_bounds(k)
    g = {kk: t.cpu().numpy() for kk, t in k.ctx.values().items()}
    tol = 1e-12
    assert np.all(np.abs(g["K"] - v["K"]) <= tol * bK)
    assert np.all(np.abs(g["M"] - v["M"]) <= tol * bM)
    assert np.all(np.abs(g["MV"] - v["MV"]) <= tol * bMV)
    bH = 0.5 * bK + bMV
    assert np.all(np.abs(g["H"] - v["H"]) <= tol * bH)
    bA = bH + k.p.mu * bM
    assert np.all(np.abs(g["A"] - v["A"]) <= tol * bA)
    rp, col, _, _ = k.om.pattern()
    rows = np.repeat(np.arange(k.om.n_free), np.diff(rp))
    dA = np.zeros(k.om.n_free)
    dA[rows[rows == col]] = bA[rows == col]
    assert np.all(np.abs(g["diag"] - v["diag"]) <= tol * dA)


@pytest.mark.parametrize("c,N", [(1, 1), (2, 4), (2, 3), (2, 16), (3, 8), (2, 32), (2, 64), (2, 2), (2, 5)])
def test_spmm(c, N):
    k = case(c)
    rng = np.random.default_rng(N)
    X = rng.standard_normal((k.om.n_free, N))
    Xd = dt(X)
    for op in ("K", "M", "MV", "H", "A"):
        Y = k.ctx.spmm(op, Xd).cpu().numpy()
        ref = k.om.spmm(op, X)
        Aabs = abs(k.om.csr(op))
        bound = Aabs @ np.abs(X)
        assert np.all(np.abs(Y - ref) <= 1e-12 * bound + 1e-300), op


@pytest.mark.parametrize("N", [3, 16])
def test_spmm_A_fresh_after_each_assembly(N):
    """spmm('A') right after assemble_veff (no earlier MV/H call) and after a re-assembly with another mu:
    the generic CSR path (ragged N) reads the CSR view of A, which must follow the last assembly."""
    p = small(n=6, N=N)
    k = Case(p, assemble=False, coarse=False)
    rng = np.random.default_rng(11)
    X = rng.standard_normal((p.n_free, N))
    for mu in (p.mu, 3.0 * p.mu + 1.0):
        k.ctx.assemble_veff(dt(p.V), mu)
        k.om.assemble_veff(p.V, mu)
        Y = k.ctx.spmm("A", dt(X)).cpu().numpy()
        ref = k.om.spmm("A", X)
        assert np.all(np.abs(Y - ref) <= 1e-12 * (abs(k.om.csr("A")) @ np.abs(X)) + 1e-300), mu


def _mnorm_rel(M, a, b):
    d = a - b
    return np.sqrt(np.einsum("ij,ij->j", d, M @ d)) / np.sqrt(np.einsum("ij,ij->j", b, M @ b))


def _solve_both(k, lam, U, tol=1e-10, max_iter=2000):
    ref = k.om.block_pcg(lam, U, tol=tol, max_iter=max_iter)
    Ut, iters, relres = k.ctx.block_solve(dt(lam), dt(U), tol=tol, max_iter=max_iter)
    st = k.ctx.sync()
    return ref, Ut.cpu().numpy(), iters.cpu().numpy(), relres.cpu().numpy(), st


@pytest.mark.parametrize("c", [1, 2, 3])
def test_block_solve_matches_oracle(c):
    k = case(c)
    p = k.p
    ref, ut, it, rr, st = _solve_both(k, p.lam, p.U)
    assert st == 0 and ref["status"] == 0
    assert np.all(_mnorm_rel(k.om.csr("M"), ut, ref["Ut"]) <= 1e-8)
    assert np.all(np.abs(it - ref["iters"]) <= 2)
    assert np.all(rr <= 1e-10)
    tr = k.ctx.true_residual(dt(p.lam), dt(p.U), dt(ut)).cpu().numpy()
    assert np.all(tr <= 1e-9)


@pytest.mark.parametrize("N", [1, 2, 3, 5, 7, 13, 20, 33, 64])
def test_block_solve_ragged_N(N):
    """Non-power-of-two N (padded internally), ragged tail tiles, N = 1 with odd n."""
    p = small(n=7, N=N)
    k = Case(p)
    ref, ut, it, rr, st = _solve_both(k, p.lam, p.U)
    assert st == 0
    assert np.all(_mnorm_rel(k.om.csr("M"), ut, ref["Ut"]) <= 1e-8)
    assert np.all(np.abs(it - ref["iters"]) <= 2)


def test_block_solve_degenerate_tiny_mesh():
    """One free node (box with 2 cells per axis) and a fully Dirichlet-dominated problem."""
    p = small(n=2, N=2, nc=2)
    assert p.n_free == 1
    k = Case(p, coarse=False)
    ref, ut, it, rr, st = _solve_both(k, p.lam, p.U)
    assert st == 0
    assert np.allclose(ut, ref["Ut"], rtol=1e-12, atol=0)


def test_not_spd_and_not_converged_and_nonfinite():
    ks = _ks()
    p = small(n=6, N=2, potential="harmonic")
    k = Case(p, assemble=False, coarse=False)
    # mu = 0 with a strongly negative potential shift -> indefinite A
    k.ctx.assemble_veff(dt(p.V - 50.0), 0.0)
    k.ctx.block_solve(dt(np.zeros(2)), dt(p.U), tol=1e-10, max_iter=500)
    assert k.ctx.sync() == ks.KS_E_NOT_SPD
    # max_iter = 1 -> NOT_CONVERGED, one iteration per column, last iterate written
    k.ctx.assemble_veff(dt(p.V), 10.0)
    k.om.assemble_veff(p.V, 10.0)
    Ut, iters, _ = k.ctx.block_solve(dt(p.lam), dt(p.U), tol=1e-10, max_iter=1)
    assert k.ctx.sync() == ks.KS_E_NOT_CONVERGED
    ref = k.om.block_pcg(p.lam, p.U, tol=1e-10, max_iter=1)
    assert np.all(iters.cpu().numpy() == 1)
    assert np.allclose(Ut.cpu().numpy(), ref["Ut"], rtol=1e-10, atol=1e-14)
    # NaN in V -> NONFINITE
    V = p.V.copy()
    V[5] = np.nan
    k.ctx.assemble_veff(dt(V), 10.0)
    assert k.ctx.sync() == ks.KS_E_NONFINITE


def test_mesh_errors():
    ks = _ks()
    xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    with pytest.raises(ks.KSError) as e:
        ks.Context(xyz, np.array([[0, 2, 1, 3]], np.int32), np.zeros(4, np.uint8))
    assert e.value.status == ks.KS_E_MESH
    with pytest.raises(ks.KSError) as e:
        ks.Context(xyz, np.array([[0, 1, 2, 9]], np.int32), np.zeros(4, np.uint8))
    assert e.value.status == ks.KS_E_MESH


def test_argument_errors():
    ks = _ks()
    k = case(1)
    U = dt(k.p.U)
    with pytest.raises(ks.KSError):
        k.ctx.block_solve(dt(k.p.lam), U, Ut=U)          # aliasing
    with pytest.raises(ks.KSError):
        k.ctx.block_solve(dt(k.p.lam), U, tol=0.0)
    with pytest.raises(ks.KSError):
        k.ctx.block_solve(dt(k.p.lam), U, max_iter=0)


@pytest.mark.parametrize("c", [1, 2, 3])
def test_projection_matches_oracle(c):
    k = case(c)
    p = k.p
    rng = np.random.default_rng(c)
    Ut = p.U + 0.1 * rng.standard_normal(p.U.shape)
    FA, FB = k.ctx.project_augmented(dt(Ut))
    assert k.ctx.sync() == 0
    FA, FB = FA.cpu().numpy(), FB.cpu().numpy()
    FAo, FBo = k.om.project(p.n_H, p.P_rowptr, p.P_col, p.P_val, Ut)
    bA, bB = projection_bounds(k.om, p.n_H, p.P_rowptr, p.P_col, p.P_val, Ut)
    assert_entrywise(FA, FAo, bA, what="F_A")
    assert_entrywise(FB, FBo, bB, what="F_B")
    w = sl.eigh(FA, FB, eigvals_only=True)[:p.N]
    wo = sl.eigh(FAo, FBo, eigvals_only=True)[:p.N]
    assert np.all(np.abs(w - wo) <= 1e-9 * np.abs(wo).max())


@pytest.mark.parametrize("N", [1, 3, 5, 8, 16, 20, 32, 33, 64])
def test_projection_ragged_N(N):
    """Every item-pass variant: NP = 2, 4 (FFMA), 8, 16, 32 (FP64 tensor cores), 64 (row-block Gram), with
    ragged N and small items (many item boundaries inside a 4-row k-step)."""
    p = small(n=8, N=N, nc=3)
    k = Case(p)
    rng = np.random.default_rng(N)
    Ut = rng.standard_normal((p.n_free, N))
    FA, FB = k.ctx.project_augmented(dt(Ut))
    FAo, FBo = k.om.project(p.n_H, p.P_rowptr, p.P_col, p.P_val, Ut)
    bA, bB = projection_bounds(k.om, p.n_H, p.P_rowptr, p.P_col, p.P_val, Ut)
    assert_entrywise(FA.cpu().numpy(), FAo, bA, what="F_A")
    assert_entrywise(FB.cpu().numpy(), FBo, bB, what="F_B")


def test_whole_step_deterministic():
    """Two runs of assemble + solve + project are bitwise identical."""
    k = case(2)
    p = k.p
    outs = []
    for _ in range(2):
        k.ctx.assemble_veff(dt(p.V), p.mu)
        Ut, it, rr = k.ctx.block_solve(dt(p.lam), dt(p.U))
        FA, FB = k.ctx.project_augmented(Ut)
        assert k.ctx.sync() == 0
        outs.append([x.cpu().numpy().copy() for x in (k.ctx.values()["A"], Ut, it, rr, FA, FB)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_solve_then_pencil_eigenvalues_end_to_end():
    """Whole path on C2 against the oracle's whole path: lowest N pencil eigenvalues within 1e-9."""
    k = case(2)
    p = k.p
    ref = k.om.block_pcg(p.lam, p.U)
    FAo, FBo = k.om.project(p.n_H, p.P_rowptr, p.P_col, p.P_val, ref["Ut"])
    Ut, _, _ = k.ctx.block_solve(dt(p.lam), dt(p.U))
    FA, FB = k.ctx.project_augmented(Ut)
    assert k.ctx.sync() == 0
    w = sl.eigh(FA.cpu().numpy(), FB.cpu().numpy(), eigvals_only=True)[:p.N]
    wo = sl.eigh(FAo, FBo, eigvals_only=True)[:p.N]
    assert np.all(np.abs(w - wo) <= 1e-9 * np.abs(wo).max())


@pytest.mark.slow
def test_config4_full_parity():
    """C4 at full size (the bench workload): pattern bit-exact, values, block solve and projection
    against the oracle (the oracle's C4 solve takes ~1 min on one core)."""
    k = Case(gen.make_problem(4))
    p = k.p
    rp, col, emap, fon = k.om.pattern()
    g_rp, g_col, g_emap, g_fon, _, _ = (t.cpu().numpy() for t in k.ctx.pattern())
    assert np.array_equal(g_rp, rp.astype(np.int32)) and np.array_equal(g_col, col)
    assert np.array_equal(g_emap, emap) and np.array_equal(g_fon, fon)
    v, bK, bM, bMV = _value_bounds(k)
    g = {kk: t.cpu().numpy() for kk, t in k.ctx.values().items()}
    assert np.all(np.abs(g["A"] - v["A"]) <= 1e-12 * (0.5 * bK + bMV + p.mu * bM))
    ref, ut, it, rr, st = _solve_both(k, p.lam, p.U)
    assert st == 0 and ref["status"] == 0
    assert np.all(_mnorm_rel(k.om.csr("M"), ut, ref["Ut"]) <= 1e-8)
    assert np.all(np.abs(it - ref["iters"]) <= 2)
    FA, FB = k.ctx.project_augmented(dt(ut))
    FAo, FBo = k.om.project(p.n_H, p.P_rowptr, p.P_col, p.P_val, ut)
    bA, bB = projection_bounds(k.om, p.n_H, p.P_rowptr, p.P_col, p.P_val, ut)
    assert_entrywise(FA.cpu().numpy(), FAo, bA, what="F_A")
    assert_entrywise(FB.cpu().numpy(), FBo, bB, what="F_B")
    # the pencil's lowest N eigenvalues: the GPU eigensolver on the GPU's F against LAPACK on the oracle's F
    ev, _ = k.ctx.pencil_eig(FA, FB, p.N)
    assert k.ctx.sync() == 0
    wo = sl.eigh(FAo, FBo, eigvals_only=True, subset_by_index=[0, p.N - 1])
    assert np.all(np.abs(ev.cpu().numpy() - wo) <= 1e-9 * np.abs(wo).max())


@pytest.mark.parametrize("c", [2, 3])
def test_block_solve_three_phase_kernel(c, monkeypatch):
    """The three-phase kernel (KS_PCG_FUSED=0: q = A p, then r, then x and p; the Poisson mode of the Hartree
    solve always runs it) reaches the oracle's solutions like the default fused two-phase kernel."""
    monkeypatch.setenv("KS_PCG_FUSED", "0")
    k = case(c)
    p = k.p
    ref, ut, it, rr, st = _solve_both(k, p.lam, p.U)
    assert st == 0 and ref["status"] == 0
    assert np.all(_mnorm_rel(k.om.csr("M"), ut, ref["Ut"]) <= 1e-8)
    assert np.all(np.abs(it - ref["iters"]) <= 2)


def test_pipelined_host_steps_equal_the_device_path():
    """ks_step_submit / ks_step_wait (two device slots, copy streams) give bitwise the same F_A, F_B as the
    device-resident calls on the same inputs, for several pipelined steps with alternating inputs."""
    import paper_2404_19249_b200 as ks
    k = case(2)
    p = k.p
    rng = np.random.default_rng(5)
    Us = [p.U, p.U + 1e-3 * rng.standard_normal(p.U.shape), p.U]
    ref = []
    for U in Us:
        Ut, _, _ = k.ctx.block_solve(dt(p.lam), dt(U))
        FA, FB = k.ctx.project_augmented(Ut)
        ref.append((FA.cpu().numpy(), FB.cpu().numpy()))
    Vh = torch.from_numpy(p.V).pin_memory()
    lamh = torch.from_numpy(p.lam).pin_memory()
    Uhs = [torch.from_numpy(np.ascontiguousarray(U)).pin_memory() for U in Us]
    outs = []
    for Uh in Uhs:
        outs.append(ks.solve_step_host(k.ctx, Vh, p.mu, lamh, Uh, None, wait=False))
    k.ctx.step_wait()
    assert k.ctx.sync() == 0
    for (FA, FB), (FAr, FBr) in zip(outs, ref):
        assert np.array_equal(FA.numpy(), FAr) and np.array_equal(FB.numpy(), FBr)


@pytest.mark.parametrize("c", [2, 3])
def test_assembly_variants_are_bitwise_equal(c, monkeypatch):
    """The star-mask assembly (32-bit masks: every star here has 24 tets; KS_ASM_MASK=64: 64-bit masks) and the
    per-entry inverse-map walk (KS_ASM_MASK=0, the kernel for stars > 64 tets) sum every entry's element
    contributions in the same ascending order: the sliced-ELL A, H, diag(A) they write, seen through a whole
    solve + projection, are bitwise equal."""
    p = case(c).p
    outs = []
    for mode in (None, "64", "0"):
        if mode is None:
            monkeypatch.delenv("KS_ASM_MASK", raising=False)
        else:
            monkeypatch.setenv("KS_ASM_MASK", mode)
        ctx = _ks().Context(p.xyz, p.tets, p.dirichlet)   # the mode is fixed at ks_create
        ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
        ctx.assemble_veff(dt(p.V), p.mu)
        Ut, it, rr = ctx.block_solve(dt(p.lam), dt(p.U))
        FA, FB = ctx.project_augmented(Ut)
        assert ctx.sync() == 0
        outs.append([x.cpu().numpy() for x in (Ut, it, rr, FA, FB)])
        del ctx
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)
