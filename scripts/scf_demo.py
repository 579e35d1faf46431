#!/usr/bin/env python
"""End-to-end demonstration of the nonnested augmented subspace method on one B200 (NEXT-1..3 on top of the
hot path): a CH4-like molecule (config C3 geometry: C Z=6 at the origin, 4 H at 1.09 bohr; 10 electrons in
N = 5 doubly occupied orbitals, smoothed Coulomb V_ext), graded fine mesh, an independent graded coarse mesh
(nonnested) interpolated by ks_interpolation (Algorithm 1), and ks_scf_solve (Algorithm 3 with Anderson
mixing). Prints one JSON line: sizes, timings, outer/inner iterations, density-change history, Ritz values.
usage: python scripts/scf_demo.py [fine_cells] [coarse_cells] [mu] [max_outer]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2404_19249_b200 as ks  # noqa: E402


def main():
    nf = int(sys.argv[1]) if len(sys.argv) > 1 else 48
    ncs = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    mu = float(sys.argv[3]) if len(sys.argv) > 3 else 20.0
    max_outer = int(sys.argv[4]) if len(sys.argv) > 4 else 150
    base = gen.make_config(3)
    nuc = base["nuclei"]

    def mesh(n):
        return gen.make_problem(dict(base, n=n, N=5, vnoise=0.0, nc=2, grading=("equi", 1.5)))

    t0 = time.time()
    p, c = mesh(nf), mesh(ncs)
    dev = torch.device("cuda", 0)
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
    torch.cuda.synchronize()
    t1 = time.time()
    rp, col, val, nH = ctx.interpolation(c.xyz, c.tets, c.dirichlet)
    ctx.set_coarse(nH, rp, col, val)
    torch.cuda.synchronize()
    t2 = time.time()
    lam = torch.full((p.N,), -1.0, dtype=torch.float64, device=dev)
    U = torch.from_numpy(p.U).to(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = ctx.scf_solve(torch.from_numpy(p.V).to(dev), lam, U, mu=mu, f=2.0, tol=1e-7, max_outer=max_outer, inner=30,
                        inner_tol=1e-7, allow_unconverged=True)
    status = "converged" if out["converged"] else "not converged (max_outer)"
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    rho = ctx.density(U, f=2.0)
    vh, mom, _ = ctx.hartree(rho, tol=1e-12)
    print(json.dumps({
        "system": "CH4-like (C Z=6 + 4 H Z=1 at 1.09 bohr), 10 electrons, N=5, smoothed Coulomb",
        "fine": {"cells": nf, "nodes": int(p.n_nodes), "n_free": int(p.n_free), "tets": int(p.n_tets)},
        "coarse": {"cells": ncs, "n_H": int(nH), "nonnested": "graded coarse Kuhn mesh, P by ks_interpolation"},
        "mu": mu, "status": status, "outer": int(out["outer"]), "inner_steps": out["inner"].tolist(),
        "density_change": [float("%.3e" % x) for x in out["dres"]],
        "lowest_ritz_history": [float("%.8f" % x) for x in out["lams"][:, 0]],
        "ritz_values": lam.cpu().numpy().tolist(), "electrons": float(mom[0]),
        "time_ms": {"scf_total": ms, "per_outer": ms / max(1, out["outer"])},
        "hartree_preconditioner": "Jacobi" if os.environ.get("KS_HARTREE_2L", "1") == "0" else "two-level",
        "setup_s": {"gen": t1 - t0, "interpolation_and_coarse": t2 - t1},
    }), flush=True)


if __name__ == "__main__":
    main()
