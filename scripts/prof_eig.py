"""Profiling driver of ks_pencil_eig at config C (default 4): solve + project once, then `reps` pencil
eigensolves of the step's F_A, F_B; prints the event-timed and wall-clock time per call (host share)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

import torch  # noqa: E402

import paper_2404_19249_b200 as ks  # noqa: E402

p = gen.make_problem(a.config)
dev = torch.device("cuda", 0)
ctx = ks.Context(p.xyz, p.tets, p.dirichlet, max_N=p.N)
t = lambda x: torch.from_numpy(x).to(dev)
ctx.assemble_veff(t(p.V), p.mu)
ctx.set_coarse(p.n_H, t(p.P_rowptr), t(p.P_col), t(p.P_val))
Ut, _, _ = ctx.block_solve(t(p.lam), t(p.U))
FA, FB = ctx.project_augmented(Ut)
ev, Y = ctx.pencil_eig(FA, FB, p.N)
torch.cuda.synchronize()
s = torch.cuda.current_stream()
for r in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(s)
    ev, Y = ctx.pencil_eig(FA, FB, p.N)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"pencil_eig D={FA.shape[0]} k={p.N}: events {e0.elapsed_time(e1):.3f} ms, wall {1e3*(time.perf_counter()-w0):.3f} ms")
assert ctx.sync() == 0
