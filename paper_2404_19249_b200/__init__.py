"""B200 (sm_100a, fp64) hot path of the nonnested augmented subspace method for the Kohn-Sham
equation (arXiv 2404.19249): V_eff mass reassembly, batched Jacobi-PCG for the N shifted boundary
value problems, projection onto W = [P_H | U~]. The compute lives in libks.so (csrc/, C ABI in
include/ks.h); this package is the thin ctypes binding (ks.py) and the build script (_build.py)."""
from .ks import (Context, KSError, load_library, solve_step_host, host_sym_eig, LIB_PATH, EXPORTS, STATUS_NAMES,  # noqa: F401
                 KS_OK, KS_E_ARG, KS_E_MESH, KS_E_NONFINITE, KS_E_NOT_SPD, KS_E_NOT_CONVERGED, KS_E_CUDA,
                 KS_E_NOMEM, KS_E_STATE, KS_E_RANK, KS_E_WORKSPACE, KS_EXT_EIG, KS_EXT_SCF, KS_EXT_STEP)

__all__ = ["Context", "KSError", "load_library", "solve_step_host", "host_sym_eig"]
