"""Projection driver: one fine mesh of config C (default 4), assemble, then `reps` projections of U with an A/B knob
(--env, default KS_PROJ_AI) set to each of --modes, CUDA-event timed; also the target of ncu captures of the
projection kernels (profiles/). Not a benchmark: bench.py is."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--modes", default="1,0")
ap.add_argument("--env", default="KS_PROJ_AI", help="A/B environment knob the modes set")
a = ap.parse_args()

import torch  # noqa: E402

import paper_2404_19249_b200 as ks  # noqa: E402

p = gen.make_problem(a.config)
dev = torch.device("cuda", 0)
ctx = ks.Context(p.xyz, p.tets, p.dirichlet, max_N=p.N)
t = lambda x: torch.from_numpy(x).to(dev)
ctx.set_coarse(p.n_H, t(p.P_rowptr), t(p.P_col), t(p.P_val))
ctx.assemble_veff(t(p.V), p.mu)
U = t(p.U)
res = {"config": a.config, "n_free": p.n_free, "N": p.N}
for mode in a.modes.split(","):
    os.environ[a.env] = mode
    FA, FB = ctx.project_augmented(U)
    torch.cuda.synchronize()
    ms = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.project_augmented(U)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    res[f"{a.env}={mode}"] = {"median_ms": ms[len(ms) // 2], "min_ms": ms[0]}
assert ctx.sync() == 0, ctx.last_error()
print(json.dumps(res))
