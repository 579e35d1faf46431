"""The C-ABI library loads and exports every symbol include/ks.h declares (no compute without a GPU),
and the product package refuses to run without CUDA (no CPU fallback)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2404_19249_b200 import _build
    _build.build()
    import paper_2404_19249_b200 as pkg
    return pkg.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ks.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ks_[a-z_]+)\s*\(", src)))


def test_header_declares_the_binding_list():
    import paper_2404_19249_b200 as pkg
    assert declared_symbols() == sorted(pkg.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2404_19249_b200", "libks.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (ks_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert lib.ks_abi_version() == 2
    assert b"sm_100a" in lib.ks_build_info()


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2404_19249_b200", "libks.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_null_context_arguments_rejected(lib):
    import ctypes as C
    h = C.c_void_p()
    assert lib.ks_create(0, None, 0, None, None, 1, None, 0, None, 0, None, 0, None, C.byref(h)) == 1  # KS_E_ARG
    assert b"KS_E_ARG" in lib.ks_last_error(None)
    sz = [C.c_size_t() for _ in range(3)]
    assert lib.ks_plan(0, None, 0, None, None, 1, *[C.byref(x) for x in sz]) == 1   # KS_E_ARG before any device call
    assert lib.ks_sync(None) == 1


def test_no_cpu_fallback():
    import torch
    import paper_2404_19249_b200 as pkg
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    with pytest.raises(RuntimeError):
        pkg.Context(np.zeros((4, 3)), np.zeros((1, 4), np.int32), np.zeros(4, np.uint8))


def test_product_does_not_import_oracle():
    pkg_dir = os.path.join(ROOT, "paper_2404_19249_b200")
    for dirpath, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f


def c_consumer_build(out):
    """Compile tests/c_abi/c_consumer.c (strict C99, -Werror) against include/ks.h and link it with libks.so
    and the CUDA runtime: the ABI is usable from plain C, without Python or torch."""
    lib_dir = os.path.join(ROOT, "paper_2404_19249_b200")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(cuda, "include"), os.path.join(ROOT, "tests", "c_abi", "c_consumer.c"), "-o", out,
           "-L" + lib_dir, "-lks", "-L" + os.path.join(cuda, "lib64"), "-lcudart", "-Wl,-rpath," + lib_dir,
           "-Wl,-rpath," + os.path.join(cuda, "lib64"), "-lm"]
    return subprocess.run(cmd, capture_output=True, text=True)


def test_c_consumer_compiles_and_links(lib, tmp_path):
    r = c_consumer_build(str(tmp_path / "c_consumer"))
    assert r.returncode == 0, r.stderr


@pytest.mark.parametrize("method", [0, 1])
def test_host_sym_eig_matches_lapack(method):
    """ks_host_sym_eig (the host routine of the filtered pencil eigensolver's Rayleigh-Ritz steps; host only, so it
    runs without a GPU): eigenvalues against numpy's LAPACK eigh, residual and orthonormality, for random,
    nearly diagonal (a converged Rayleigh-Ritz step), exactly diagonal, repeated-eigenvalue, decoupled and
    tiny matrices, by Householder + QL (0) and by cyclic Jacobi (1)."""
    import numpy as np
    import paper_2404_19249_b200 as ks
    rng = np.random.default_rng(7)
    cases = []
    for n in (1, 2, 3, 5, 24, 40, 72):
        R = rng.standard_normal((n, n))
        cases.append(0.5 * (R + R.T) + np.diag(np.arange(n, dtype=float)))
        cases.append(np.diag(np.linspace(-18.0, 30.0, n)) + 1e-7 * 0.5 * (R + R.T))
        cases.append(np.diag(np.linspace(-3.0, 4.0, n)[::-1]))
        Q, _ = np.linalg.qr(R)
        cases.append(Q @ np.diag(np.repeat(np.arange((n + 2) // 3, dtype=float), 3)[:n]) @ Q.T)
        B = np.zeros((n, n))                      # two decoupled blocks: a zero sub-diagonal entry mid-matrix
        h = n // 2
        B[:h, :h] = cases[-4][:h, :h]
        B[h:, h:] = cases[-4][h:, h:]
        cases.append(B)
    cases.append(np.zeros((6, 6)))
    for A in cases:
        A = 0.5 * (A + A.T)
        n = A.shape[0]
        w, V = ks.host_sym_eig(A, method)
        ref = np.linalg.eigvalsh(A)
        scale = max(np.abs(ref).max(), 1e-300)
        assert np.all(np.diff(w) >= 0)
        assert np.abs(w - ref).max() <= 1e-13 * n * scale
        assert np.abs(A @ V - V * w).max() <= 1e-13 * n * scale
        assert np.abs(V.T @ V - np.eye(n)).max() <= 1e-13 * n


def test_host_sym_eig_rejects_bad_arguments():
    import numpy as np
    import paper_2404_19249_b200 as ks
    with pytest.raises(ks.KSError):
        ks.host_sym_eig(np.zeros((2, 3)))
    with pytest.raises(ks.KSError):
        ks.host_sym_eig(np.eye(3), method=2)
