"""NEXT-4 / SURVEY.md §8(e) on CPU: the row-slab partition of ONE block solve (paper_2404_19249_b200/slab.py)
over 2 and 3 gloo processes, against the same driver on one rank and against the oracle's PCG
(tests/slab_cpu.py executes the phases on the host). Checks the partition (balanced, halo from neighbours
only), the halo exchange and the rank-ordered dot reductions: the partitioned solve equals the 1-rank solve to
1e-12 (M-norm, per column) with the same iteration counts, and the oracle's solution to 1e-8."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    import gen
    return gen.make_problem(dict(L=4.0, n=12, grading=None, jitter=0.15, nuclei=[((0.2, -0.3, 0.1), 2)], vnoise=0.05,
                                 N=5, orbitals="gauss", lam=("uniform", -2.0, -0.5), nc=3, seed=31))


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import oracle
    from paper_2404_19249_b200 import slab
    from slab_cpu import CpuSlab
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = _problem()
        om = oracle.Mesh.from_problem(p)
        om.assemble_veff(p.V, p.mu)
        rp, col, _, _ = om.pattern()
        bounds = slab.slab_bounds(rp, col, world)
        ex = CpuSlab(om.csr("A"), om.csr("M"), p.lam, p.mu, p.U, bounds, rank)
        out = slab.slab_block_solve(ex, p.lam, tol=1e-10, max_iter=500)
        q.put((rank, bounds, out, ex.result().copy()))
    finally:
        dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    bounds = res[0][1]
    x = np.concatenate([r[3] for r in res])
    return bounds, [r[2] for r in res], x


def test_slab_bounds_partition_and_halo():
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2404_19249_b200 import slab
    p = _problem()
    om = oracle.Mesh.from_problem(p)
    rp, col, _, _ = om.pattern()
    for world in (1, 2, 3, 4):
        b = slab.slab_bounds(rp, col, world)
        assert b[0][0] == 0 and b[-1][1] == p.n_free
        assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
        nnz = [rp[r1] - rp[r0] for r0, r1, _, _ in b]
        assert max(nnz) - min(nnz) <= 2 * np.diff(rp).max()       # balanced by nonzeros
        for r, (r0, r1, lo, hi) in enumerate(b):                   # the halo covers every referenced row
            cols = col[rp[r0]:rp[r1]]
            assert lo == min(r0, cols.min()) and hi == max(r1, cols.max() + 1)
            sends, recvs = slab.halo_schedule(b, r)
            got = sorted(x for _, a, c in recvs for x in range(a, c))
            assert got == sorted(set(range(lo, hi)) - set(range(r0, r1)))
    with pytest.raises(ValueError):
        slab.slab_bounds(rp, col, p.n_free // 4)                   # halo beyond the neighbour


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_solve_equals_one_rank_and_oracle(world):
    sys.path.insert(0, ROOT)
    import oracle
    p = _problem()
    _, one, x1 = _run(1)
    bounds, outs, xw = _run(world)
    assert len(bounds) == world
    M = None
    om = oracle.Mesh.from_problem(p)
    om.assemble_veff(p.V, p.mu)
    M = om.csr("M")

    def mrel(a, b):
        d = a - b
        return np.sqrt(np.einsum("ij,ij->j", d, M @ d)) / np.sqrt(np.einsum("ij,ij->j", b, M @ b))

    for o in outs:   # every rank took the same decisions
        assert o["status"] == "ok" and o["block_iters"] == outs[0]["block_iters"]
        assert np.array_equal(o["iters"], one[0]["iters"]) and np.array_equal(o["relres"], outs[0]["relres"])
    assert np.all(mrel(xw, x1) <= 1e-12)
    ref = om.block_pcg(p.lam, p.U, tol=1e-10)
    assert np.all(mrel(xw, ref["Ut"]) <= 1e-8)
    assert np.all(np.abs(outs[0]["iters"] - ref["iters"]) <= 2)
    assert np.all(outs[0]["relres"] <= 1e-10)
