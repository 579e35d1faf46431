"""Thin Python binding of libks (include/ks.h): argument marshalling only.

Every compute step runs in the CUDA kernels of libks.so (sm_100a). PyTorch provides device memory and
streams. There is no CPU fallback: if libks.so is missing or no CUDA device is present, calls raise.
Function names follow the C ABI (ks_create -> Context(...), ks_assemble_veff -> ctx.assemble_veff, ...).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# KS_LIB overrides the library path (A/B builds of the same sources with other compile-time options)
LIB_PATH = os.environ.get("KS_LIB") or os.path.join(_PKG, "libks.so")

KS_OK, KS_E_ARG, KS_E_MESH, KS_E_NONFINITE, KS_E_NOT_SPD, KS_E_NOT_CONVERGED, KS_E_CUDA, KS_E_NOMEM, \
    KS_E_STATE, KS_E_RANK, KS_E_WORKSPACE = range(11)
STATUS_NAMES = {0: "KS_OK", 1: "KS_E_ARG", 2: "KS_E_MESH", 3: "KS_E_NONFINITE", 4: "KS_E_NOT_SPD",
                5: "KS_E_NOT_CONVERGED", 6: "KS_E_CUDA", 7: "KS_E_NOMEM", 8: "KS_E_STATE", 9: "KS_E_RANK",
                10: "KS_E_WORKSPACE"}
KS_EXT_EIG, KS_EXT_SCF, KS_EXT_STEP = 1, 2, 4
KS_EXT_ALL = KS_EXT_EIG | KS_EXT_SCF | KS_EXT_STEP
REGIONS = {"persistent": 0, "workspace": 1, "coarse": 3, "ext": 4}
OPS = {"K": 0, "M": 1, "MV": 2, "H": 3, "A": 4}

# every symbol declared in include/ks.h (checked by tests/test_abi.py)
EXPORTS = ["ks_abi_version", "ks_build_info", "ks_plan", "ks_create", "ks_destroy", "ks_set_stream", "ks_pattern",
           "ks_values", "ks_assemble_veff", "ks_spmm", "ks_block_solve", "ks_last_iterations", "ks_solve_trace",
           "ks_true_residual", "ks_coarse_plan", "ks_set_coarse", "ks_ext_plan", "ks_attach_ext",
           "ks_project_augmented", "ks_pencil_eig", "ks_host_sym_eig", "ks_lift", "ks_augmented_solve", "ks_interpolation_plan",
           "ks_interpolation", "ks_density", "ks_vxc", "ks_hartree", "ks_scf_solve", "ks_step_submit",
           "ks_step_wait", "ks_memory_bytes", "ks_memory_usage", "ks_launch_count", "ks_sync", "ks_last_error",
           "ks_slab_init", "ks_slab_spmm", "ks_slab_update", "ks_slab_finish"]


class KSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libks.so (no build, no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libks.so not found at {path}; run __graft_entry__.build() "
                          "(python -c 'import __graft_entry__ as g; g.build()')")
    L = C.CDLL(path)
    vp, i64, i32, dbl, st = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_int
    sig = {
        "ks_abi_version": (C.c_int, []),
        "ks_build_info": (C.c_char_p, []),
        "ks_plan": (st, [i64, vp, i64, vp, vp, i32, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                         C.POINTER(C.c_size_t)]),
        "ks_create": (st, [i64, vp, i64, vp, vp, i32, vp, C.c_size_t, vp, C.c_size_t, vp, C.c_size_t, vp,
                           C.POINTER(vp)]),
        "ks_destroy": (None, [vp]),
        "ks_set_stream": (st, [vp, vp]),
        "ks_pattern": (st, [vp, C.POINTER(i64), C.POINTER(i64)] + [C.POINTER(vp)] * 6),
        "ks_values": (st, [vp] + [C.POINTER(vp)] * 6),
        "ks_assemble_veff": (st, [vp, vp, dbl]),
        "ks_spmm": (st, [vp, C.c_int, i32, vp, vp]),
        "ks_block_solve": (st, [vp, i32, vp, vp, vp, dbl, i32, vp, vp]),
        "ks_last_iterations": (st, [vp, C.POINTER(i32)]),
        "ks_solve_trace": (st, [vp, i32, vp, C.POINTER(i32)]),
        "ks_true_residual": (st, [vp, i32, vp, vp, vp, vp]),
        "ks_coarse_plan": (st, [vp, i64, vp, vp, vp, C.POINTER(C.c_size_t)]),
        "ks_set_coarse": (st, [vp, i64, vp, vp, vp, vp, C.c_size_t]),
        "ks_ext_plan": (st, [vp, C.c_uint32, i64, C.POINTER(C.c_size_t)]),
        "ks_attach_ext": (st, [vp, C.c_uint32, i64, vp, C.c_size_t]),
        "ks_project_augmented": (st, [vp, i32, vp, vp, vp]),
        "ks_pencil_eig": (st, [vp, i64, i32, vp, vp, vp, vp]),
        "ks_host_sym_eig": (st, [i32, vp, vp, vp, i32]),
        "ks_lift": (st, [vp, i32, vp, i32, vp, vp]),
        "ks_augmented_solve": (st, [vp, i32, vp, vp, dbl, i32, dbl, i32, C.POINTER(i32), vp]),
        "ks_interpolation_plan": (st, [vp, i64, vp, i64, C.POINTER(C.c_size_t)]),
        "ks_interpolation": (st, [vp, i64, vp, i64, vp, vp, vp, C.c_size_t, vp, vp, vp, C.POINTER(i64),
                                  C.POINTER(i64)]),
        "ks_density": (st, [vp, i32, vp, dbl, vp]),
        "ks_vxc": (st, [vp, vp, vp, vp]),
        "ks_hartree": (st, [vp, vp, dbl, i32, vp, i32, vp, C.POINTER(i32)]),
        "ks_scf_solve": (st, [vp, i32, vp, dbl, dbl, vp, vp, dbl, i32, i32, dbl, dbl, i32, dbl, dbl,
                              C.POINTER(i32), vp, vp, vp]),
        "ks_step_submit": (st, [vp, i32, vp, dbl, vp, vp, dbl, i32, vp, vp]),
        "ks_step_wait": (st, [vp]),
        "ks_memory_bytes": (st, [vp, C.POINTER(C.c_size_t)]),
        "ks_memory_usage": (st, [vp, i32, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
        "ks_slab_init": (st, [vp, i32, i64, i64, vp, vp, vp, vp, vp]),
        "ks_slab_spmm": (st, [vp, i32, i64, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp]),
        "ks_slab_update": (st, [vp, i32, i64, i64, vp, vp, vp, vp]),
        "ks_slab_finish": (st, [vp, i32, i64, i64, vp, vp, vp, vp]),
        "ks_launch_count": (st, [vp, C.POINTER(i64)]),
        "ks_sync": (st, [vp]),
        "ks_last_error": (C.c_char_p, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _ptr(t) -> int:
    return t.data_ptr()


def _check_cuda_tensor(t, dtype, shape=None, name="tensor"):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must have dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def _n_cols(t) -> int:
    if t.dim() != 2:
        raise ValueError(f"expected a 2-D [rows][N] block, got shape {tuple(t.shape)}")
    return int(t.shape[1])


def _check_host_tensor(t, dtype, shape, name):
    import torch
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise TypeError(f"{name} must be a host (CPU) torch.Tensor")
    if t.dtype != dtype or not t.is_contiguous() or tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must be a contiguous {dtype} tensor of shape {tuple(shape)}, "
                         f"got {t.dtype} {tuple(t.shape)}")
    return t


class Context:
    """ks_plan + ks_create .. ks_destroy. Host mesh arrays are numpy; everything else lives in torch CUDA tensors.

    Every device byte the library uses is a torch uint8 tensor owned here (include/ks.h, "Memory"): the
    persistent and workspace regions from ks_plan (the setup region is released after ks_create), the coarse
    region from ks_coarse_plan, and the extension region (NEXT rows, host steps) from ks_ext_plan, attached on
    the first call that needs it. `max_N` is the largest block of orbitals any call will use."""

    def __init__(self, xyz, tets, dirichlet, stream=None, max_N: int = 64):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libks needs a CUDA device (no CPU fallback)")
        L = load_library()
        self._L = L
        self._h = None
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        tets = np.ascontiguousarray(tets, dtype=np.int32)
        dirichlet = np.ascontiguousarray(dirichlet, dtype=np.uint8)
        self.n_nodes, self.n_tets = xyz.shape[0], tets.shape[0]
        self.max_N = int(max_N)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        sz = [C.c_size_t() for _ in range(3)]
        s = L.ks_plan(self.n_nodes, xyz.ctypes.data, self.n_tets, tets.ctypes.data, dirichlet.ctypes.data,
                      self.max_N, *[C.byref(x) for x in sz])
        if s != KS_OK:
            raise KSError(s, L.ks_last_error(None).decode())
        self.plan = {"persistent": sz[0].value, "workspace": sz[1].value, "setup": sz[2].value}
        self._mem = {"persistent": self._region(sz[0].value), "workspace": self._region(sz[1].value)}
        setup = self._region(sz[2].value)
        h = C.c_void_p()
        s = L.ks_create(self.n_nodes, xyz.ctypes.data, self.n_tets, tets.ctypes.data, dirichlet.ctypes.data,
                        self.max_N, self._mem["persistent"].data_ptr(), sz[0].value,
                        self._mem["workspace"].data_ptr(), sz[1].value, setup.data_ptr(), sz[2].value,
                        C.c_void_p(self.stream.cuda_stream), C.byref(h))
        del setup   # only used during ks_create (which synchronised the stream)
        if s != KS_OK:
            raise KSError(s, L.ks_last_error(None).decode())
        self._h = h
        nf, nnz = C.c_int64(), C.c_int64()
        self._call(L.ks_pattern(self._h, C.byref(nf), C.byref(nnz), *([None] * 6)))
        self.n_free, self.nnz = nf.value, nnz.value
        self.n_H = None
        self.mu = None
        self._ext = (0, 0)   # (features, max_D) of the attached extension region

    def _region(self, nbytes: int):
        """A caller-owned device region for libks (torch's caching allocator; 512-byte aligned)."""
        import torch
        with torch.cuda.stream(self.stream):
            return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=self.device)

    def _need_ext(self, features: int, max_D: int = 0):
        """Attach an extension region covering `features` and pencils up to max_D (re-planned when it grows)."""
        have_f, have_D = self._ext
        f = have_f | features
        D = max(have_D, int(max_D))
        if f == have_f and D == have_D:
            return
        n = C.c_size_t()
        self._call(self._L.ks_ext_plan(self._h, f, D, C.byref(n)))
        self._mem.pop("ext", None)
        self._ext = (0, 0)
        region = self._region(n.value)
        self._call(self._L.ks_attach_ext(self._h, f, D, region.data_ptr(), n.value))
        self._mem["ext"] = region
        self._ext = (f, D)

    def memory_usage(self, region: str):
        """(capacity, used, peak) bytes of one region of the context (ks_memory_usage)."""
        cap, used, peak = C.c_size_t(), C.c_size_t(), C.c_size_t()
        self._call(self._L.ks_memory_usage(self._h, REGIONS[region], C.byref(cap), C.byref(used), C.byref(peak)))
        return cap.value, used.value, peak.value

    # -- plumbing --------------------------------------------------------------------------------
    def _call(self, status):
        if status != KS_OK:
            raise KSError(status, self._L.ks_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.ks_destroy(self._h)
            self._h = None
        self._mem = {}

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream):
        self.stream = stream
        self._call(self._L.ks_set_stream(self._h, C.c_void_p(stream.cuda_stream)))

    def _view(self, dptr, count, dtype):
        """Copy a library-owned device array into a new torch tensor (on the ctx stream)."""
        import torch
        out = torch.empty(count, dtype=dtype, device=self.device)
        if count:
            with torch.cuda.stream(self.stream):
                # device-to-device copy through a torch view of the raw pointer
                src = _raw_tensor(dptr, count, dtype, self.device)
                out.copy_(src)
        return out

    # -- ABI calls ---------------------------------------------------------------------------------
    def pattern(self):
        """(row_ptr, col, emap, free_of_node, inv_ptr, inv_idx) as new int32 CUDA tensors."""
        import torch
        ptrs = [C.c_void_p() for _ in range(6)]
        self._call(self._L.ks_pattern(self._h, None, None, *[C.byref(p) for p in ptrs]))
        inv_ptr = self._view(ptrs[4].value, self.nnz + 1, torch.int32)
        n_contrib = int(inv_ptr[-1].item())
        sizes = [self.n_free + 1, self.nnz, 16 * self.n_tets, self.n_nodes, self.nnz + 1, n_contrib]
        out = [self._view(p.value, s, torch.int32) for p, s in zip(ptrs, sizes)]
        return tuple(out)

    def values(self):
        """dict K, M, MV, H, A, diag of new float64 CUDA tensors (copies)."""
        import torch
        ptrs = [C.c_void_p() for _ in range(6)]
        self._call(self._L.ks_values(self._h, *[C.byref(p) for p in ptrs]))
        names = ["K", "M", "MV", "H", "A", "diag"]
        return {k: self._view(p.value, self.n_free if k == "diag" else self.nnz, torch.float64)
                for k, p in zip(names, ptrs)}

    def assemble_veff(self, veff, mu: float):
        import torch
        _check_cuda_tensor(veff, torch.float64, (self.n_nodes,), "veff")
        self._call(self._L.ks_assemble_veff(self._h, _ptr(veff), float(mu)))
        self.mu = float(mu)

    def spmm(self, op: str, X, Y=None):
        import torch
        N = X.shape[1] if X.dim() == 2 else 1
        shape = (self.n_free, N) if X.dim() == 2 else (self.n_free,)
        _check_cuda_tensor(X, torch.float64, shape, "X")
        if Y is None:
            Y = torch.empty_like(X)
        _check_cuda_tensor(Y, torch.float64, shape, "Y")
        self._call(self._L.ks_spmm(self._h, OPS[op], N, _ptr(X), _ptr(Y)))
        return Y

    def block_solve(self, lam, U, Ut=None, tol=1e-10, max_iter=2000, iters=None, relres=None):
        import torch
        N = _n_cols(U)
        _check_cuda_tensor(U, torch.float64, (self.n_free, N), "U")
        _check_cuda_tensor(lam, torch.float64, (N,), "lambda")
        if Ut is None:
            Ut = torch.empty_like(U)
        if iters is None:
            iters = torch.zeros(N, dtype=torch.int32, device=U.device)
        if relres is None:
            relres = torch.zeros(N, dtype=torch.float64, device=U.device)
        _check_cuda_tensor(Ut, torch.float64, (self.n_free, N), "Ut")
        _check_cuda_tensor(iters, torch.int32, (N,), "iters")
        _check_cuda_tensor(relres, torch.float64, (N,), "relres")
        self._call(self._L.ks_block_solve(self._h, N, _ptr(lam), _ptr(U), _ptr(Ut), float(tol), int(max_iter),
                                          _ptr(iters), _ptr(relres)))
        return Ut, iters, relres

    def last_iterations(self) -> int:
        v = C.c_int32()
        self._call(self._L.ks_last_iterations(self._h, C.byref(v)))
        return v.value

    def solve_trace(self, cap: int = 8192) -> np.ndarray:
        """Phase-end timestamps (ns) of the last block solve (KS_PCG_TRACE=1 at solve time), see ks.h."""
        buf = np.zeros(cap, dtype=np.uint64)
        cnt = C.c_int32()
        self._call(self._L.ks_solve_trace(self._h, cap, buf.ctypes.data, C.byref(cnt)))
        return buf[:cnt.value].copy()

    def true_residual(self, lam, U, Ut):
        import torch
        N = _n_cols(U)
        _check_cuda_tensor(lam, torch.float64, (N,), "lambda")
        _check_cuda_tensor(U, torch.float64, (self.n_free, N), "U")
        _check_cuda_tensor(Ut, torch.float64, (self.n_free, N), "Ut")
        out = torch.empty(N, dtype=torch.float64, device=U.device)
        self._call(self._L.ks_true_residual(self._h, N, _ptr(lam), _ptr(U), _ptr(Ut), _ptr(out)))
        return out

    def set_coarse(self, n_H: int, P_rowptr, P_col, P_val):
        import torch
        _check_cuda_tensor(P_rowptr, torch.int32, (self.n_free + 1,), "P_rowptr")
        _check_cuda_tensor(P_col, torch.int32, None, "P_col")
        _check_cuda_tensor(P_val, torch.float64, tuple(P_col.shape), "P_val")
        if P_col.dim() != 1:
            raise ValueError("P_col must be 1-D")
        n = C.c_size_t()
        self._call(self._L.ks_coarse_plan(self._h, int(n_H), _ptr(P_rowptr), _ptr(P_col), _ptr(P_val), C.byref(n)))
        self.n_H = None
        self._mem.pop("coarse", None)
        self._mem.pop("ext", None)   # ks_set_coarse detaches the extension region
        self._ext = (0, 0)
        region = self._region(n.value)
        self._call(self._L.ks_set_coarse(self._h, int(n_H), _ptr(P_rowptr), _ptr(P_col), _ptr(P_val),
                                         region.data_ptr(), n.value))
        self._mem["coarse"] = region
        self.n_H = int(n_H)

    def project_augmented(self, Ut, FA=None, FB=None):
        import torch
        if self.n_H is None:
            raise KSError(KS_E_STATE, "project_augmented: call set_coarse first")
        N = _n_cols(Ut)
        _check_cuda_tensor(Ut, torch.float64, (self.n_free, N), "Ut")
        D = self.n_H + N
        if FA is None:
            FA = torch.empty((D, D), dtype=torch.float64, device=Ut.device)
        if FB is None:
            FB = torch.empty((D, D), dtype=torch.float64, device=Ut.device)
        _check_cuda_tensor(FA, torch.float64, (D, D), "FA")
        _check_cuda_tensor(FB, torch.float64, (D, D), "FB")
        self._call(self._L.ks_project_augmented(self._h, N, _ptr(Ut), _ptr(FA), _ptr(FB)))
        return FA, FB

    def pencil_eig(self, FA, FB, k: int):
        """ks_pencil_eig: lowest k eigenpairs of F_A y = lambda F_B y -> (evals [k], evecs [D][k]), evecs
        F_B-orthonormal. Chebyshev-filtered subspace iteration after the Cholesky reduction when k + 8 <= D / 2,
        dense cuSOLVER otherwise or with KS_PENCIL_DENSE=1 (include/ks.h)."""
        import torch
        D = FA.shape[0]
        _check_cuda_tensor(FA, torch.float64, (D, D), "FA")
        _check_cuda_tensor(FB, torch.float64, (D, D), "FB")
        self._need_ext(KS_EXT_EIG, D)
        ev = torch.empty(k, dtype=torch.float64, device=FA.device)
        Y = torch.empty((D, k), dtype=torch.float64, device=FA.device)
        self._call(self._L.ks_pencil_eig(self._h, D, int(k), _ptr(FA), _ptr(FB), _ptr(ev), _ptr(Y)))
        return ev, Y

    def lift(self, Ut, Y, Unew=None):
        """ks_lift: U_new = P Y[:n_H] + U~ Y[n_H:]."""
        import torch
        if self.n_H is None:
            raise KSError(KS_E_STATE, "lift: call set_coarse first")
        N, k = _n_cols(Ut), _n_cols(Y)
        _check_cuda_tensor(Ut, torch.float64, (self.n_free, N), "Ut")
        _check_cuda_tensor(Y, torch.float64, (self.n_H + N, k), "Y")
        if Unew is None:
            Unew = torch.empty((self.n_free, k), dtype=torch.float64, device=Ut.device)
        _check_cuda_tensor(Unew, torch.float64, (self.n_free, k), "Unew")
        self._call(self._L.ks_lift(self._h, N, _ptr(Ut), int(k), _ptr(Y), _ptr(Unew)))
        return Unew

    def augmented_solve(self, lam, U, tol_eig=1e-10, max_outer=50, tol_bvp=1e-10, max_iter_bvp=2000):
        """ks_augmented_solve: outer iterations of Algorithm 3 with the current operators; lam and U are
        updated in place. Returns (outer iterations, Ritz-value history [outer][N] as numpy)."""
        import torch
        N = _n_cols(U)
        _check_cuda_tensor(U, torch.float64, (self.n_free, N), "U")
        _check_cuda_tensor(lam, torch.float64, (N,), "lam")
        self._need_ext(KS_EXT_EIG)
        hist = np.zeros((max_outer, N))
        outer = C.c_int32()
        self._call(self._L.ks_augmented_solve(self._h, N, _ptr(lam), _ptr(U), float(tol_eig), int(max_outer),
                                              float(tol_bvp), int(max_iter_bvp), C.byref(outer),
                                              hist.ctypes.data))
        return outer.value, hist[:outer.value].copy()

    def interpolation(self, xyz_c, tets_c, dirichlet_c):
        """ks_interpolation: P = I_H^h from an independent coarse mesh (host arrays) -> (row_ptr, col, val)
        as CUDA tensors and n_H."""
        import torch
        xyz_c = np.ascontiguousarray(xyz_c, dtype=np.float64)
        tets_c = np.ascontiguousarray(tets_c, dtype=np.int32)
        dir_c = np.ascontiguousarray(dirichlet_c, dtype=np.uint8)
        rp = torch.empty(self.n_free + 1, dtype=torch.int32, device=self.device)
        col = torch.empty(4 * self.n_free, dtype=torch.int32, device=self.device)
        val = torch.empty(4 * self.n_free, dtype=torch.float64, device=self.device)
        wb = C.c_size_t()
        self._call(self._L.ks_interpolation_plan(self._h, xyz_c.shape[0], xyz_c.ctypes.data, tets_c.shape[0],
                                                 C.byref(wb)))
        work = self._region(wb.value)   # call scratch (the call synchronises before returning)
        nH, pn = C.c_int64(), C.c_int64()
        self._call(self._L.ks_interpolation(self._h, xyz_c.shape[0], xyz_c.ctypes.data, tets_c.shape[0],
                                            tets_c.ctypes.data, dir_c.ctypes.data, work.data_ptr(), wb.value,
                                            _ptr(rp), _ptr(col), _ptr(val), C.byref(nH), C.byref(pn)))
        del work
        return rp, col[:pn.value], val[:pn.value], nH.value

    def density(self, U, f=2.0, rho=None):
        """ks_density: nodal density on all nodes."""
        import torch
        _check_cuda_tensor(U, torch.float64, (self.n_free, _n_cols(U)), "U")
        if rho is None:
            rho = torch.empty(self.n_nodes, dtype=torch.float64, device=U.device)
        _check_cuda_tensor(rho, torch.float64, (self.n_nodes,), "rho")
        self._call(self._L.ks_density(self._h, U.shape[1], _ptr(U), float(f), _ptr(rho)))
        return rho

    def vxc(self, rho, vxc=None, eps=None):
        """ks_vxc: LDA/PZ exchange-correlation potential (and energy per electron) on all nodes."""
        import torch
        _check_cuda_tensor(rho, torch.float64, (self.n_nodes,), "rho")
        if vxc is None:
            vxc = torch.empty_like(rho)
        if eps is None:
            eps = torch.empty_like(rho)
        _check_cuda_tensor(vxc, torch.float64, (self.n_nodes,), "vxc")
        _check_cuda_tensor(eps, torch.float64, (self.n_nodes,), "eps")
        self._call(self._L.ks_vxc(self._h, _ptr(rho), _ptr(vxc), _ptr(eps)))
        return vxc, eps

    def hartree(self, rho, tol=1e-12, max_iter=100000, vh=None, warm=False):
        """ks_hartree: Hartree potential on all nodes -> (vh, moments [10] numpy, PCG iterations). With a coarse
        space set (set_coarse) the solve is the two-level preconditioned CG (Jacobi + P (P^T K P)^-1 P^T),
        else (or with KS_HARTREE_2L=0) Jacobi-PCG (include/ks.h)."""
        import torch
        _check_cuda_tensor(rho, torch.float64, (self.n_nodes,), "rho")
        if vh is None:
            vh = torch.zeros_like(rho)
        _check_cuda_tensor(vh, torch.float64, (self.n_nodes,), "vh")
        self._need_ext(KS_EXT_SCF)
        mom = np.zeros(10)
        it = C.c_int32()
        self._call(self._L.ks_hartree(self._h, _ptr(rho), float(tol), int(max_iter), _ptr(vh), int(bool(warm)),
                                      mom.ctypes.data, C.byref(it)))
        return vh, mom, it.value

    def scf_solve(self, vext, lam, U, mu, f=2.0, tol=1e-8, max_outer=60, inner=20, inner_tol=None, beta=0.7,
                  depth=5, bvp_tol=1e-12, hartree_tol=1e-12, allow_unconverged=False):
        """ks_scf_solve: Algorithm 3 for the Kohn-Sham equation; lam and U updated in place. Returns dict(outer,
        inner steps, outer density changes, Ritz-value history, converged) as numpy; KS_E_NOT_CONVERGED raises
        unless allow_unconverged."""
        import torch
        _check_cuda_tensor(vext, torch.float64, (self.n_nodes,), "vext")
        N = _n_cols(U)
        _check_cuda_tensor(U, torch.float64, (self.n_free, N), "U")
        _check_cuda_tensor(lam, torch.float64, (N,), "lam")
        self._need_ext(KS_EXT_SCF)
        outer = C.c_int32()
        inner_steps = np.zeros(max_outer, np.int32)
        dres = np.zeros(max_outer)
        lams = np.zeros((max_outer, N))
        st = self._L.ks_scf_solve(self._h, N, _ptr(vext), float(f), float(mu), _ptr(lam), _ptr(U), float(tol),
                                  int(max_outer), int(inner), float(tol if inner_tol is None else inner_tol),
                                  float(beta), int(depth), float(bvp_tol), float(hartree_tol), C.byref(outer),
                                  inner_steps.ctypes.data, dres.ctypes.data, lams.ctypes.data)
        if st not in (KS_OK, KS_E_NOT_CONVERGED) or (st == KS_E_NOT_CONVERGED and not allow_unconverged):
            self._call(st)
        k = outer.value
        return dict(outer=k, inner=inner_steps[:k], dres=dres[:k], lams=lams[:k], converged=st == KS_OK)

    def step_submit(self, V_host, mu, lam_host, U_host, FA_host, FB_host, tol=1e-10, max_iter=2000):
        """ks_step_submit: one pipelined hot-path step from host buffers (pinned torch CPU tensors)."""
        import torch
        N = _n_cols(U_host)
        D = (self.n_H or 0) + N
        for t, shape, name in ((V_host, (self.n_nodes,), "V_host"), (lam_host, (N,), "lam_host"),
                               (U_host, (self.n_free, N), "U_host"), (FA_host, (D, D), "FA_host"),
                               (FB_host, (D, D), "FB_host")):
            _check_host_tensor(t, torch.float64, shape, name)
        self._need_ext(KS_EXT_STEP)
        self._call(self._L.ks_step_submit(self._h, N, V_host.data_ptr(), float(mu), lam_host.data_ptr(),
                                          U_host.data_ptr(), float(tol), int(max_iter), FA_host.data_ptr(),
                                          FB_host.data_ptr()))

    def step_wait(self):
        self._call(self._L.ks_step_wait(self._h))

    def memory_bytes(self) -> int:
        v = C.c_size_t()
        self._call(self._L.ks_memory_bytes(self._h, C.byref(v)))
        return v.value

    def launch_count(self) -> int:
        v = C.c_int64()
        self._call(self._L.ks_launch_count(self._h, C.byref(v)))
        return v.value

    def sync(self) -> int:
        """ks_sync: returns the latched status (0 = OK) without raising."""
        return self._L.ks_sync(self._h)

    def last_error(self) -> str:
        return self._L.ks_last_error(self._h).decode()


def _raw_tensor(dptr: int, count: int, dtype, device):
    """A torch tensor aliasing `count` elements at device address dptr (no copy, no ownership)."""
    import torch

    class _CAI:
        pass

    typestr = {torch.int32: "<i4", torch.float64: "<f8"}[dtype]
    obj = _CAI()
    obj.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (dptr, False), "version": 3,
                                   "strides": None}
    return torch.as_tensor(obj, device=device)


def host_sym_eig(A, method: int = 0):
    """ks_host_sym_eig: all eigenpairs of a small symmetric matrix with the host routine behind ks_pencil_eig's
    Rayleigh-Ritz steps (method 0: Householder + implicit QL, 1: cyclic Jacobi). A: numpy float64 [n][n].
    Returns (w [n] ascending, V [n][n] with V[:, j] the eigenvector j). Runs without a GPU."""
    import numpy as np
    A = np.ascontiguousarray(A, dtype=np.float64)
    if A.ndim != 2 or A.shape[0] != A.shape[1] or A.shape[0] < 1:
        raise KSError(KS_E_ARG, "host_sym_eig: A must be a square matrix")
    n = A.shape[0]
    w, Vt = np.empty(n), np.empty((n, n))
    st = load_library().ks_host_sym_eig(n, A.ctypes.data, w.ctypes.data, Vt.ctypes.data, int(method))
    if st != KS_OK:
        raise KSError(st, "ks_host_sym_eig failed")
    return w, Vt.T.copy()


def solve_step_host(ctx: Context, V_host, mu, lam_host, U_host, out=None, tol=1e-10, max_iter=2000, wait=True):
    """One hot-path step from HOST buffers (pinned torch CPU tensors) through ks_step_submit: H2D of V, lambda,
    U; assemble, block solve, project on the device; D2H of F_A, F_B into `out` (a pair of pinned host
    tensors, allocated when None). With wait=False consecutive calls pipeline (ks_step_wait completes them)."""
    import torch
    N = U_host.shape[1]
    D = ctx.n_H + N
    if out is None:
        out = (torch.empty((D, D), dtype=torch.float64).pin_memory(), torch.empty((D, D), dtype=torch.float64).pin_memory())
    ctx.step_submit(V_host, mu, lam_host, U_host, out[0], out[1], tol=tol, max_iter=max_iter)
    if wait:
        ctx.step_wait()
    return out
