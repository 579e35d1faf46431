"""The C ABI from a plain C99 program on the GPU (tests/c_abi/c_consumer.c): ks_create, ks_assemble_veff,
ks_block_solve and ks_sync on a 4^3-cell Kuhn mesh with two orbitals, device memory from the CUDA runtime's
C API. Both columns converge to 1e-10."""
import subprocess

import pytest

from test_abi import c_consumer_build

pytestmark = pytest.mark.gpu


def test_c_consumer_runs(tmp_path):
    exe = str(tmp_path / "c_consumer")
    r = c_consumer_build(exe)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stdout + run.stderr
    fields = run.stdout.split()
    assert fields[0] == "ok" and int(fields[1]) == 27 and int(fields[2]) > 0
    assert float(fields[3]) <= 1e-10 and float(fields[4]) <= 1e-10
