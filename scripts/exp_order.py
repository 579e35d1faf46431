#!/usr/bin/env python
"""Experiment: effect of the node numbering on the block solve (gather locality of the SpMM phase).
Builds config C (default 4), renumbers its nodes (lexicographic / Morton / blocked), and times
ks_block_solve with the kernel's phase trace for each. Prints one JSON line per ordering."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2404_19249_b200 as ks  # noqa: E402


def morton3(i, j, k, bits=10):
    code = np.zeros_like(i, dtype=np.int64)
    for b in range(bits):
        code |= ((i >> b) & 1) << (3 * b)
        code |= ((j >> b) & 1) << (3 * b + 1)
        code |= ((k >> b) & 1) << (3 * b + 2)
    return code


def renumber(p, order):
    n1 = p.n_cells + 1
    node = np.arange(p.n_nodes)
    i, j, k = node % n1, (node // n1) % n1, node // (n1 * n1)
    if order == "lex":
        key = node
    elif order == "morton":
        key = morton3(i, j, k)
    elif order.startswith("block"):
        b = int(order[5:])  # bricks of b^3 nodes, bricks lexicographic, lexicographic inside
        nb = (n1 + b - 1) // b
        key = (((k // b) * nb + (j // b)) * nb + (i // b)) * b ** 3 + ((k % b) * b + (j % b)) * b + (i % b)
    else:
        raise ValueError(order)
    perm = np.argsort(key, kind="stable")        # new id -> old id
    inv = np.empty_like(perm)
    inv[perm] = np.arange(p.n_nodes)             # old id -> new id
    xyz = p.xyz[perm]
    tets = inv[p.tets].astype(np.int32)
    dirichlet = p.dirichlet[perm]
    V = p.V[perm]
    # free rows: U rows follow the new free numbering
    old_free = np.cumsum(p.dirichlet == 0) - 1   # old node -> old free index
    new_free_nodes = np.nonzero(dirichlet == 0)[0]
    U = p.U[old_free[perm[new_free_nodes]]]
    return xyz, tets, dirichlet, V, np.ascontiguousarray(U)


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    orders = sys.argv[2].split(",") if len(sys.argv) > 2 else ["lex", "morton", "block4", "block8"]
    p = gen.make_problem(c)
    dev = torch.device("cuda", 0)
    for order in orders:
        xyz, tets, dirichlet, V, U = renumber(p, order)
        ctx = ks.Context(xyz, tets, dirichlet)
        Vd = torch.from_numpy(V).to(dev)
        Ud = torch.from_numpy(U).to(dev)
        lam = torch.from_numpy(p.lam).to(dev)
        Ut = torch.empty_like(Ud)
        ctx.assemble_veff(Vd, p.mu)
        for _ in range(3):
            ctx.block_solve(lam, Ud, Ut, tol=1e-10, max_iter=2000)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            ctx.block_solve(lam, Ud, Ut, tol=1e-10, max_iter=2000)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        os.environ["KS_PCG_TRACE"] = "1"
        ctx.block_solve(lam, Ud, Ut, tol=1e-10, max_iter=2000)
        ts = ctx.solve_trace()
        os.environ.pop("KS_PCG_TRACE")
        d = np.diff(ts.astype(np.int64)) * 1e-3
        k = (len(d) - 1) // 3
        print(json.dumps({"order": order, "stage": os.environ.get("KS_PCG_STAGE", "1"), "solve_ms": ms,
                          "iters": ctx.last_iterations(), "init_us": d[0],
                          "S_us": float(np.mean(d[1::3][:k])), "U_us": float(np.mean(d[2::3][:k])),
                          "P_us": float(np.mean(d[3::3][:k]))}), flush=True)
        del ctx


if __name__ == "__main__":
    main()
