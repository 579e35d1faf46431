#!/usr/bin/env python
"""Standalone multi-RHS SpMM timing (ks_spmm, Y = A X on the sliced-ELL copy) on config C for N in a list:
GB/s of algorithmic bytes 12 nnz + 4 (n+1) + 16 N n (matrix, read X once, write Y)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2404_19249_b200 as ks  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
Ns = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16]
p = gen.make_problem(c)
dev = torch.device("cuda", 0)
ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
ctx.assemble_veff(torch.from_numpy(p.V).to(dev), p.mu)
n, nnz = p.n_free, ctx.nnz
for N in Ns:
    X = torch.randn(n, N, dtype=torch.float64, device=dev)
    Y = torch.empty_like(X)
    for _ in range(3):
        ctx.spmm("A", X, Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 20
    e0.record()
    for _ in range(R):
        ctx.spmm("A", X, Y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    b = 12 * nnz + 4 * (n + 1) + 16 * N * n
    print(json.dumps({"N": N, "ms": ms, "alg_GBs": b / ms / 1e6}),
          flush=True)
