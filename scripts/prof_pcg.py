"""Profiling driver: one fine mesh of config C (default 4), assemble + `reps` block solves (+ projection), for
ncu captures of the PCG / projection kernels (profiles/). Not a benchmark: bench.py is."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--project", action="store_true")
a = ap.parse_args()

import torch  # noqa: E402

import paper_2404_19249_b200 as ks  # noqa: E402

p = gen.make_problem(a.config)
dev = torch.device("cuda", 0)
ctx = ks.Context(p.xyz, p.tets, p.dirichlet, max_N=p.N)
t = lambda x: torch.from_numpy(x).to(dev)
ctx.assemble_veff(t(p.V), p.mu)
ctx.set_coarse(p.n_H, t(p.P_rowptr), t(p.P_col), t(p.P_val))
lam, U = t(p.lam), t(p.U)
for _ in range(a.reps):
    Ut, it, rr = ctx.block_solve(lam, U)
    if a.project:
        ctx.project_augmented(Ut)
assert ctx.sync() == 0, ctx.last_error()
print("ok", p.n_free, p.N, ctx.last_iterations())
