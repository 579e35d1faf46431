"""NEXT-4 / SURVEY.md §8(e) on the GPU: the row-slab partition of one block solve through libks's ks_slab_*
kernels (paper_2404_19249_b200/slab.py, GpuSlab). One rank, and two processes sharing the one GPU of this pool
(gloo; the ranks' kernels never wait on one another: the driver exchanges halos and dots on the host between
launches), against ks_block_solve on the whole problem: per column M-norm difference <= 1e-12, the same
iteration counts, and the oracle's solution to 1e-8."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, config, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import gen
    import paper_2404_19249_b200 as ks
    from paper_2404_19249_b200 import slab
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        p = gen.make_problem(config)
        dev = torch.device("cuda", 0)
        ctx = ks.Context(p.xyz, p.tets, p.dirichlet, max_N=p.N)
        ctx.assemble_veff(torch.from_numpy(p.V).to(dev), p.mu)
        bounds = slab.gpu_slab_bounds(ctx, world)
        ex = slab.GpuSlab(ctx, p.lam, torch.from_numpy(p.U).to(dev), bounds, rank)
        out = slab.slab_block_solve(ex, p.lam, tol=1e-10, max_iter=2000)
        assert ctx.sync() == 0
        q.put((rank, out, ex.result().cpu().numpy()))
    finally:
        dist.destroy_process_group()


def _run(world, config):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, config, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    return [r[1] for r in res], np.concatenate([r[2] for r in res])


@pytest.mark.parametrize("config,world", [(2, 1), (2, 2), (3, 2)])
def test_slab_solve_matches_block_solve(config, world):
    import gen
    import oracle
    import paper_2404_19249_b200 as ks
    p = gen.make_problem(config)
    dev = torch.device("cuda", 0)
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet, max_N=p.N)
    ctx.assemble_veff(torch.from_numpy(p.V).to(dev), p.mu)
    Ut, iters, _ = ctx.block_solve(torch.from_numpy(p.lam).to(dev), torch.from_numpy(p.U).to(dev))
    assert ctx.sync() == 0
    ut, it = Ut.cpu().numpy(), iters.cpu().numpy()
    del ctx
    outs, xs = _run(world, config)
    om = oracle.Mesh.from_problem(p)
    om.assemble_veff(p.V, p.mu)
    M = om.csr("M")

    def mrel(a, b):
        d = a - b
        return np.sqrt(np.einsum("ij,ij->j", d, M @ d)) / np.sqrt(np.einsum("ij,ij->j", b, M @ b))

    for o in outs:
        assert o["status"] == "ok" and np.array_equal(o["iters"], it)
    assert np.all(mrel(xs, ut) <= 1e-12)
    ref = om.block_pcg(p.lam, p.U, tol=1e-10)
    assert np.all(mrel(xs, ref["Ut"]) <= 1e-8)
