"""Assembly driver: one fine mesh of config C (default 4), `reps` CUDA-event-timed ks_assemble_veff calls (median,
min); also the target of ncu captures of the assembly kernels. Not a benchmark: bench.py is."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()

import torch  # noqa: E402

import paper_2404_19249_b200 as ks  # noqa: E402

p = gen.make_problem(a.config)
dev = torch.device("cuda", 0)
ctx = ks.Context(p.xyz, p.tets, p.dirichlet, max_N=p.N)
V = torch.from_numpy(p.V).to(dev)
ctx.assemble_veff(V, p.mu)
torch.cuda.synchronize()
ms = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.assemble_veff(V, p.mu)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
assert ctx.sync() == 0, ctx.last_error()
ms.sort()
print(json.dumps({"config": a.config, "lib": os.environ.get("KS_LIB", "libks.so"), "median_ms": ms[len(ms) // 2],
                  "min_ms": ms[0]}))
