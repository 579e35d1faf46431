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
ap.add_argument("--env", default="", help="NAME=VALUE set before the timed calls (A/B knob)")
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
if a.env:
    k_, v_ = a.env.split("=", 1)
    os.environ[k_] = v_
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
if os.environ.get("KS_EF_TRACE") == "1":   # phase times of the device-resident loop (ks_efdev.cu stamps, CTA 0)
    import numpy as np
    t = ctx.solve_trace().astype(np.int64).reshape(-1, 2)
    names = {1: "gemm", 2: "gram", 3: "chol", 4: "reduce", 5: "jacobi", 6: "update", 7: "resid", 8: "filter"}
    tot = {}
    sweeps = []
    for (tag0, t0), (tag1, t1) in zip(t[:-1], t[1:]):
        if tag1 % 100 == 5 and tag1 >= 100:
            sweeps.append(int(tag1 // 100))
            tag1 = 5
        if tag1 in names:
            tot[names[tag1]] = tot.get(names[tag1], 0.0) + (t1 - t0) / 1e3
    print("jacobi sweeps per Rayleigh-Ritz step:", sweeps)
    rounds = int((t[:, 0] == 0).sum())
    print("device loop rounds", rounds, "phase totals us:", {k: round(v, 1) for k, v in tot.items()},
          "total", round(float((t[-1, 1] - t[0, 1]) / 1e3), 1))
