"""N>1 host logic of bench.py on CPU (gloo, world size 2): each rank gets its own seeded problem (weak
scaling) and the timing combine is max-over-ranks of the device time and sum of the work
units. No data of the method crosses ranks."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist

    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, loc = bench.dist_env()
    ms = 10.0 + 5.0 * rank
    units = 1000 * (rank + 1)
    tmax, usum = bench.combine_ranks(ms, units, w, torch.device("cpu"))
    seed = bench.rank_seed(4, r)
    dist.barrier()
    dist.destroy_process_group()
    q.put((r, w, loc, tmax, usum, seed))


def test_two_rank_combine_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, w0, l0, t0, u0, s0), (r1, w1, l1, t1, u1, s1) = out
    assert (r0, r1, w0, w1, l0, l1) == (0, 1, 2, 2, 0, 1)
    assert t0 == t1 == 15.0            # max over ranks
    assert u0 == u1 == 3000.0          # sum over ranks
    assert s0 != s1                    # independent problems per rank


def test_single_rank_combine_is_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.combine_ranks(7.5, 42, 1, None) == (7.5, 42.0)
