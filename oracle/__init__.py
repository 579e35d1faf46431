"""ctypes wrapper of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs. The product package (paper_2404_19249_b200) never imports
this module and shares no code with it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_E_ARG, OR_E_MESH, OR_E_NONFINITE, OR_E_NOT_SPD, OR_E_NOT_CONVERGED, OR_E_NOMEM = range(7)
WHICH = {"K": 0, "M": 1, "MV": 2, "H": 3, "A": 4}


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc (-O2, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int, C.c_double
        L.or_create.restype = vp
        L.or_create.argtypes = [i64, vp, i64, vp, vp, C.POINTER(C.c_int)]
        L.or_destroy.argtypes = [vp]
        L.or_last_error.restype = C.c_char_p
        L.or_last_error.argtypes = [vp]
        L.or_sizes.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.or_get_pattern.argtypes = [vp, vp, vp, vp, vp]
        L.or_get_values.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
        L.or_assemble_veff.restype = i32
        L.or_assemble_veff.argtypes = [vp, vp, dbl]
        L.or_spmm.restype = i32
        L.or_spmm.argtypes = [vp, i32, i32, vp, vp]
        L.or_block_pcg.restype = i32
        L.or_block_pcg.argtypes = [vp, i32, vp, vp, vp, dbl, i32, vp, vp, vp]
        L.or_project.restype = i32
        L.or_project.argtypes = [vp, i64, vp, vp, vp, i32, vp, vp, vp]
        L.or_pencil_eig.restype = i32
        L.or_pencil_eig.argtypes = [i64, vp, vp, i32, vp, vp]
        L.or_interpolation.restype = i32
        L.or_interpolation.argtypes = [vp, i64, vp, i64, vp, i64, vp, vp, dbl, vp, vp, vp, C.POINTER(i64)]
        L.or_density.restype = i32
        L.or_density.argtypes = [vp, i32, vp, dbl, vp]
        L.or_vxc.restype = i32
        L.or_vxc.argtypes = [i64, vp, vp, vp]
        L.or_hartree.restype = i32
        L.or_hartree.argtypes = [vp, vp, vp, dbl, i32, vp, vp, C.POINTER(C.c_int)]
        L.or_lift.restype = i32
        L.or_lift.argtypes = [vp, i64, vp, vp, vp, i32, vp, i32, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


def pencil_eig(FA, FB, k):
    """Lowest k eigenpairs of F_A y = lambda F_B y (NEXT-1, oracle.c or_pencil_eig: Cholesky + cyclic
    Jacobi). Returns (evals [k], evecs [D][k]); raises OracleError(OR_E_NOT_SPD) if F_B is not SPD."""
    FA = np.ascontiguousarray(FA, dtype=np.float64)
    FB = np.ascontiguousarray(FB, dtype=np.float64)
    D = FA.shape[0]
    ev = np.empty(k)
    Y = np.empty((D, k))
    st = lib().or_pencil_eig(D, _p(FA), _p(FB), int(k), _p(ev), _p(Y))
    if st != OR_OK:
        raise OracleError(st, "pencil_eig")
    return ev, Y


def vxc(rho):
    """NEXT-2: LDA exchange + Perdew-Zunger correlation potential and energy per electron at nodal densities
    (oracle.c or_vxc). Returns (v_xc, eps_xc)."""
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    v = np.empty_like(rho)
    e = np.empty_like(rho)
    lib().or_vxc(rho.size, _p(rho), _p(v), _p(e))
    return v, e


def anderson_mix(rho_in_hist, rho_out_hist, beta=0.7, depth=5):
    """NEXT-2: Anderson mixing (Eqs. mix2-mix6) with the histories of input and output
    densities (oldest first, newest last; only the last `depth` are used). With m the newest index and
    F^(j) = rho_out^(j) - rho_in^(j), the coefficients alpha_j (j = m0..m-1) solve
        sum_k (F^m - F^j, F^m - F^k) alpha_k = (F^m - F^j, F^m)                               (mix6)
    (discrete l2 inner product of the nodal vectors, reading R7), then
        rho~ = rho^m + sum_j alpha_j (rho^j - rho^m)   for in and out                        (mix4)
        rho_in^(m+1) = beta rho~_out + (1 - beta) rho~_in.                                    (mix1)"""
    hin = [np.asarray(x, dtype=np.float64) for x in rho_in_hist[-depth:]]
    hout = [np.asarray(x, dtype=np.float64) for x in rho_out_hist[-depth:]]
    F = [o - i for i, o in zip(hin, hout)]
    m = len(F) - 1
    alpha = np.zeros(m)
    if m > 0:
        G = np.empty((m, m))
        r = np.empty(m)
        for j in range(m):
            dj = F[m] - F[j]
            r[j] = dj @ F[m]
            for k in range(m):
                G[j, k] = dj @ (F[m] - F[k])
        alpha = np.linalg.solve(G, r)
    t_in = hin[m] + sum(alpha[j] * (hin[j] - hin[m]) for j in range(m))
    t_out = hout[m] + sum(alpha[j] * (hout[j] - hout[m]) for j in range(m))
    return beta * t_out + (1.0 - beta) * t_in


def scf_solve(mesh, n_H, P_rowptr, P_col, P_val, V_ext, lam, U, mu, f=2.0, tol=1e-8, max_outer=60, inner=20,
              inner_tol=None, beta=0.7, depth=5, bvp_tol=1e-12, hartree_tol=1e-12):
    """NEXT-2: Algorithm 3 for the Kohn-Sham equation, in the paper's order (DESIGN.md
    reading R8 for the inner loop):
      outer: V_eff = V_ext + V_Har[rho] + V_xc[rho] -> assemble (st4) -> the N
             BVPs from (lambda, Psi) (Aux_Linear_Problem) -> Psi~;
      inner (the small KS equation Nonlinear_Eig_Hh on S_H + span{Psi~}, solved self-consistently with Psi~
             fixed, at most `inner` steps): project (st1-st7) -> small eigenproblem ->
             lift -> rho_out = f sum psi^2 -> stop when ||rho_out - rho_in||_M <= inner_tol ||rho_out||_M, else
             Anderson-mix (depth, beta) and reassemble st4 with the mixed density;
      stop when the outer density change ||rho^(l) - rho^(l-1)||_M <= tol ||rho^(l)||_M.
    Returns dict(lam, U, rho, outer, inner steps per outer, outer density changes, lam history)."""
    inner_tol = tol if inner_tol is None else inner_tol
    fr = mesh.free_of_node()
    order = np.argsort(fr[fr >= 0])
    Mf = mesh.csr("M")

    def mnorm(x):
        xf = x[fr >= 0][order]
        return np.sqrt(xf @ (Mf @ xf))

    def veff(rho):
        vh, _, _ = mesh.hartree(rho, tol=hartree_tol)
        return V_ext + vh + vxc(rho)[0]

    rho = mesh.density(U, f)
    steps, dres, lams = [], [], []
    for it in range(max_outer):
        mesh.assemble_veff(veff(rho), mu)
        r = mesh.block_pcg(lam, U, tol=bvp_tol)
        if r["status"] != OR_OK:
            raise OracleError(r["status"], "scf_solve: block_pcg")
        Ut = r["Ut"]
        rho_in, hin, hout = rho, [], []
        for k in range(inner):
            FA, FB = mesh.project(n_H, P_rowptr, P_col, P_val, Ut)
            lam, Y = pencil_eig(FA, FB, U.shape[1])
            U = mesh.lift(n_H, P_rowptr, P_col, P_val, Ut, Y)
            rho_out = mesh.density(U, f)
            res = mnorm(rho_out - rho_in) / mnorm(rho_out)
            if res <= inner_tol or k == inner - 1:
                break
            hin.append(rho_in)
            hout.append(rho_out)
            rho_in = anderson_mix(hin, hout, beta, depth)
            mesh.assemble_veff(veff(rho_in), mu)
        steps.append(k + 1)
        change = mnorm(rho_out - rho) / mnorm(rho_out)
        dres.append(change)
        lams.append(lam.copy())
        rho = rho_out
        if change <= tol:
            break
    return dict(lam=lam, U=U, rho=rho, outer=len(dres), inner=np.array(steps), dres=np.array(dres),
                lams=np.array(lams))


INTERP_DROP = 1e-13  # |lambda| <= this is dropped from a P row (reading R4)


def interpolation(xyz_f, free_nodes, xyz_c, tets_c, dirichlet_c, drop=INTERP_DROP):
    """NEXT-3: the nonnested P1 interpolation operator of Algorithm 1 (oracle.c or_interpolation, brute-force
    point location). Returns (rowptr [n_free+1] i32, col i32, val f64, n_H)."""
    xyz_f = np.ascontiguousarray(xyz_f, dtype=np.float64)
    fn = np.ascontiguousarray(free_nodes, dtype=np.int64)
    xyz_c = np.ascontiguousarray(xyz_c, dtype=np.float64)
    tets_c = np.ascontiguousarray(tets_c, dtype=np.int32)
    dir_c = np.ascontiguousarray(dirichlet_c, dtype=np.uint8)
    nf = fn.shape[0]
    rp = np.zeros(nf + 1, np.int32)
    col = np.zeros(4 * nf, np.int32)
    val = np.zeros(4 * nf)
    nH = C.c_int64()
    st = lib().or_interpolation(_p(xyz_f), nf, _p(fn), xyz_c.shape[0], _p(xyz_c), tets_c.shape[0], _p(tets_c),
                                _p(dir_c), float(drop), _p(rp), _p(col), _p(val), C.byref(nH))
    if st != OR_OK:
        raise OracleError(st, "interpolation")
    return rp, col[:rp[-1]].copy(), val[:rp[-1]].copy(), nH.value


def augmented_step(mesh, n_H, P_rowptr, P_col, P_val, lam, U, tol=1e-10, max_iter=2000):
    """One outer iteration of Algorithm 3 with a fixed potential, in the paper's order:
    the N shifted BVPs (Aux_Linear_Problem) with the shift mu of the mesh's last
    assemble_veff, the projection onto W = [P_H | U~] (st1-st7), the small eigenproblem
    on W (Nonlinear_Eig_Hh) and the lift of its lowest N eigenvectors. Returns
    (lambda_new [N], U_new [n_free][N], info)."""
    N = U.shape[1]
    r = mesh.block_pcg(lam, U, tol=tol, max_iter=max_iter)
    if r["status"] != OR_OK:
        raise OracleError(r["status"], "augmented_step: block_pcg")
    FA, FB = mesh.project(n_H, P_rowptr, P_col, P_val, r["Ut"])
    ev, Y = pencil_eig(FA, FB, N)
    Unew = mesh.lift(n_H, P_rowptr, P_col, P_val, r["Ut"], Y)
    return ev, Unew, dict(iters=r["iters"], FA=FA, FB=FB, Y=Y)


class Mesh:
    """Oracle view of one fine mesh (P1, Dirichlet-eliminated)."""

    def __init__(self, xyz, tets, dirichlet):
        L = lib()
        self._keep = (np.ascontiguousarray(xyz, dtype=np.float64),
                      np.ascontiguousarray(tets, dtype=np.int32),
                      np.ascontiguousarray(dirichlet, dtype=np.uint8))
        xyz, tets, dirichlet = self._keep
        self.n_nodes, self.n_tets = xyz.shape[0], tets.shape[0]
        st = C.c_int(0)
        self._h = L.or_create(self.n_nodes, _p(xyz), self.n_tets, _p(tets), _p(dirichlet), C.byref(st))
        if not self._h:
            raise MemoryError("or_create")
        if st.value != OR_OK:
            msg = L.or_last_error(self._h).decode()
            L.or_destroy(self._h)
            self._h = None
            raise OracleError(st.value, msg)
        nf, nnz = C.c_int64(), C.c_int64()
        L.or_sizes(self._h, C.byref(nf), C.byref(nnz))
        self.n_free, self.nnz = nf.value, nnz.value
        self.mu = None

    @classmethod
    def from_problem(cls, p):
        return cls(p.xyz, p.tets, p.dirichlet)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_destroy(self._h)
            self._h = None

    def pattern(self):
        row_ptr = np.empty(self.n_free + 1, np.int64)
        col = np.empty(self.nnz, np.int32)
        emap = np.empty(16 * self.n_tets, np.int32)
        fon = np.empty(self.n_nodes, np.int32)
        lib().or_get_pattern(self._h, _p(row_ptr), _p(col), _p(emap), _p(fon))
        return row_ptr, col, emap, fon

    def values(self):
        out = {k: np.empty(self.nnz) for k in ("K", "M", "MV", "H", "A")}
        out["diag"] = np.empty(self.n_free)
        out["vol"] = np.empty(self.n_tets)
        lib().or_get_values(self._h, *[_p(out[k]) for k in ("K", "M", "MV", "H", "A", "diag", "vol")])
        return out

    def assemble_veff(self, V, mu):
        V = np.ascontiguousarray(V, dtype=np.float64)
        assert V.shape == (self.n_nodes,)
        st = lib().or_assemble_veff(self._h, _p(V), float(mu))
        self.mu = float(mu)
        return st

    def spmm(self, which, X):
        X = np.ascontiguousarray(X, dtype=np.float64)
        if X.ndim == 1:
            X = X[:, None]
        N = X.shape[1]
        Y = np.empty_like(X)
        st = lib().or_spmm(self._h, WHICH[which], N, _p(X), _p(Y))
        if st != OR_OK:
            raise OracleError(st, "spmm")
        return Y

    def block_pcg(self, lam, U, tol=1e-10, max_iter=2000):
        U = np.ascontiguousarray(U, dtype=np.float64)
        N = U.shape[1]
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        Ut = np.empty_like(U)
        iters = np.empty(N, np.int32)
        rr = np.empty(N)
        rt = np.empty(N)
        st = lib().or_block_pcg(self._h, N, _p(lam), _p(U), _p(Ut), float(tol), int(max_iter),
                                _p(iters), _p(rr), _p(rt))
        return dict(Ut=Ut, iters=iters, relres=rr, relres_true=rt, status=st)

    def project(self, n_H, P_rowptr, P_col, P_val, Ut):
        Ut = np.ascontiguousarray(Ut, dtype=np.float64)
        N = Ut.shape[1]
        D = n_H + N
        FA = np.empty((D, D))
        FB = np.empty((D, D))
        pr = np.ascontiguousarray(P_rowptr, dtype=np.int32)
        pc = np.ascontiguousarray(P_col, dtype=np.int32)
        pv = np.ascontiguousarray(P_val, dtype=np.float64)
        st = lib().or_project(self._h, int(n_H), _p(pr), _p(pc), _p(pv), N, _p(Ut), _p(FA), _p(FB))
        if st != OR_OK:
            raise OracleError(st, "project")
        return FA, FB

    def lift(self, n_H, P_rowptr, P_col, P_val, Ut, Y):
        """U_new = P Y[:n_H] + U~ Y[n_H:] (NEXT-1 lift, oracle.c or_lift)."""
        Ut = np.ascontiguousarray(Ut, dtype=np.float64)
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        N, k = Ut.shape[1], Y.shape[1]
        Unew = np.empty((self.n_free, k))
        pr = np.ascontiguousarray(P_rowptr, dtype=np.int32)
        pc = np.ascontiguousarray(P_col, dtype=np.int32)
        pv = np.ascontiguousarray(P_val, dtype=np.float64)
        st = lib().or_lift(self._h, int(n_H), _p(pr), _p(pc), _p(pv), N, _p(Ut), k, _p(Y), _p(Unew))
        if st != OR_OK:
            raise OracleError(st, "lift")
        return Unew

    def density(self, U, f=2.0):
        """NEXT-2: nodal density f sum_i psi_i^2 on all nodes (oracle.c or_density)."""
        U = np.ascontiguousarray(U, dtype=np.float64)
        rho = np.empty(self.n_nodes)
        lib().or_density(self._h, U.shape[1], _p(U), float(f), _p(rho))
        return rho

    def hartree(self, rho, tol=1e-12, max_iter=100000):
        """NEXT-2: Hartree potential on all nodes (oracle.c or_hartree). Returns (vh [n_nodes], moments [10],
        iterations)."""
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        vh = np.empty(self.n_nodes)
        mom = np.empty(10)
        it = C.c_int()
        st = lib().or_hartree(self._h, _p(self._keep[0]), _p(rho), float(tol), int(max_iter), _p(vh), _p(mom),
                              C.byref(it))
        if st != OR_OK:
            raise OracleError(st, "hartree")
        return vh, mom, it.value

    def free_of_node(self):
        return self.pattern()[3]

    def csr(self, which):
        """scipy CSR of one operator (for brute-force pins in tests)."""
        import scipy.sparse as sp
        row_ptr, col, _, _ = self.pattern()
        return sp.csr_matrix((self.values()[which], col, row_ptr), shape=(self.n_free, self.n_free))
