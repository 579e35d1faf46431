"""Seeded synthetic input generator shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no assembly, no solve, no
projection). It only builds the inputs of the hot path, following the recipe in
DESIGN.md §3 (SURVEY.md §8c readings Q13-Q22, §8d config table):

  * a P1 tetrahedral Kuhn mesh of a box (6 tets per cell, positive orientation),
    optionally jittered and/or graded ("shape regular
    decomposition T_h ... linear finite element space S_h in H^1_0");
  * Dirichlet flags for the box surface (psi = 0 on dOmega);
  * a nodal effective potential V_eff (smoothed Coulomb sum + seeded noise), a
    stand-in for V_ext + V_Har + V_xc of PAPER.md:553-561 / st3-st4;
  * N seeded initial orbitals U (free-node rows), their lambda_i, and the shift
    mu = 8 M sum_k Z_k^2 of PAPER.md:1069-1071;
  * a uniform coarse Kuhn mesh and the nonnested interpolation operator
    P_H = I_H^h (Alg. 1, 747-753 st5), rows = fine free nodes,
    cols = coarse free nodes, barycentric weights of the coarse tet containing
    each fine node.

Random numbers come from a counter-based generator (splitmix64 of
seed ^ (stream << 40) ^ index), so every value is reproducible element by
element and independent of array chunking.

Layout conventions (the interface both sides agree on; see include/ks.h):
  node id      = i + (n+1) * (j + (n+1) * k)
  tet id       = 6 * cell + sigma_index, cell = ci + n * (cj + n * ck)
  free index   = rank of a non-Dirichlet node among non-Dirichlet nodes (ascending node id)
  U            = [n_free][N] row-major, orbital index fastest
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = ["Problem", "CONFIGS", "make_problem", "make_config", "kuhn_mesh", "uniform01",
           "SEED_BASE", "config_summary"]

SEED_BASE = 2404192490  # seed_c = 2404192490 + c

# streams (Q22)
_S_JITTER, _S_VNOISE, _S_UNOISE, _S_LAMBDA, _S_NUCLEI, _S_CENTRES = 1, 2, 3, 4, 5, 6

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform01(seed: int, stream: int, index) -> np.ndarray:
    """Counter-based U[0,1): (splitmix64(seed ^ stream<<40 ^ index) >> 11) * 2^-53."""
    idx = np.asarray(index, dtype=np.uint64)
    key = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(stream) << np.uint64(40))
    u = _splitmix64(idx ^ key)
    return (u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _uniform(seed, stream, index, lo, hi):
    return lo + (hi - lo) * uniform01(seed, stream, index)


# ---------------------------------------------------------------------------------------------
# configs (BASELINE.json "configs")
# ---------------------------------------------------------------------------------------------
_CONFIG_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs")


def _load_config(c: int) -> dict:
    """configs/c<c>.json (the single source of the five workloads; JSON lists back to the tuples gen uses)."""
    with open(os.path.join(_CONFIG_DIR, f"c{c}.json")) as f:
        d = json.load(f)
    for k in ("description", "readings", "seed"):
        d.pop(k, None)
    if d.get("grading") is not None:
        d["grading"] = tuple(d["grading"])
    d["lam"] = tuple(d["lam"])
    nuc = d["nuclei"]
    d["nuclei"] = tuple(nuc) if nuc and nuc[0] == "ball" else [(tuple(x), z) for x, z in nuc]
    return d


CONFIGS = {c: _load_config(c) for c in (1, 2, 3, 4, 5)}


def make_config(c: int, **overrides) -> dict:
    cfg = dict(CONFIGS[c])
    cfg["seed"] = SEED_BASE + c
    cfg.update(overrides)
    return cfg


# ---------------------------------------------------------------------------------------------
# mesh
# ---------------------------------------------------------------------------------------------
# Kuhn / Freudenthal split (Q13): permutations in lexicographic order, odd ones get v2<->v3.
_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
_ODD = [False, True, True, False, False, True]


def kuhn_mesh(n: int) -> np.ndarray:
    """Tets (6 n^3, 4) int32 of the Kuhn split of an n^3-cell grid with (n+1)^3 nodes."""
    n1 = n + 1
    cell = np.arange(n ** 3, dtype=np.int64)
    ci, cj, ck = cell % n, (cell // n) % n, cell // (n * n)
    base = ci + n1 * (cj + n1 * ck)
    e = [1, n1, n1 * n1]
    tets = np.empty((n ** 3, 6, 4), dtype=np.int64)
    for s, (a, b, c) in enumerate(_PERMS):
        v0 = base
        v1 = base + e[a]
        v2 = v1 + e[b]
        v3 = base + e[0] + e[1] + e[2]
        if _ODD[s]:
            v2, v3 = v3, v2
        tets[:, s, 0], tets[:, s, 1], tets[:, s, 2], tets[:, s, 3] = v0, v1, v2, v3
    return tets.reshape(-1, 4).astype(np.int32)


def _equidistribution_nodes(n: int, L: float, centres: np.ndarray, p: float) -> np.ndarray:
    """1-D node positions s_0=-L < ... < s_n=L equidistributing
    w(s) = (1/K) sum_k (|s - R_k| + eps)^(1/p - 1), eps = 1e-3 L.
    The cumulative W has the closed form used below; it is inverted by bisection."""
    a = 1.0 / p - 1.0
    eps = 1e-3 * L
    R = np.asarray(centres, dtype=np.float64).reshape(-1)

    def F(s):  # antiderivative of (|s-R|+eps)^a, summed over centres, s: (m,)
        d = s[:, None] - R[None, :]
        return (np.sign(d) * ((np.abs(d) + eps) ** (a + 1.0) - eps ** (a + 1.0)) / (a + 1.0)).sum(1)

    W0, W1 = F(np.array([-L]))[0], F(np.array([L]))[0]
    target = W0 + (W1 - W0) * (np.arange(n + 1) / n)
    lo = np.full(n + 1, -L)
    hi = np.full(n + 1, L)
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        f = F(mid)
        lo = np.where(f < target, mid, lo)
        hi = np.where(f < target, hi, mid)
    s = 0.5 * (lo + hi)
    s[0], s[-1] = -L, L
    return s


@dataclass
class Problem:
    cfg: dict
    n_cells: int
    L: float
    xyz: np.ndarray          # (n_nodes, 3) f64
    tets: np.ndarray         # (n_tets, 4) i32
    dirichlet: np.ndarray    # (n_nodes,) u8
    V: np.ndarray            # (n_nodes,) f64
    nuclei: np.ndarray       # (K, 3)
    Z: np.ndarray            # (K,)
    mu: float
    N: int
    U: np.ndarray            # (n_free, N) f64
    lam: np.ndarray          # (N,) f64
    nc: int
    n_H: int
    P_rowptr: np.ndarray     # (n_free+1,) i32
    P_col: np.ndarray        # (nnzP,) i32
    P_val: np.ndarray        # (nnzP,) f64
    free_nodes: np.ndarray   # (n_free,) node ids of free nodes, ascending
    extra: dict = field(default_factory=dict)

    @property
    def n_nodes(self):
        return self.xyz.shape[0]

    @property
    def n_tets(self):
        return self.tets.shape[0]

    @property
    def n_free(self):
        return self.free_nodes.shape[0]


def _grid_coords(cfg, n, L, seed):
    """Node coordinates (n_nodes,3) of the (optionally graded / jittered) box grid."""
    n1 = n + 1
    n_nodes = n1 ** 3
    node = np.arange(n_nodes, dtype=np.int64)
    ijk = np.stack([node % n1, (node // n1) % n1, node // (n1 * n1)], axis=1)
    interior = np.all((ijk > 0) & (ijk < n), axis=1)
    grading = cfg.get("grading")
    if grading is not None and grading[0] == "equi":
        p = grading[1]
        nuc = cfg["_nuclei_xyz"]
        axes = [_equidistribution_nodes(n, L, nuc[:, a], p) for a in range(3)]
        xyz = np.stack([axes[a][ijk[:, a]] for a in range(3)], axis=1)
    else:
        # reference coordinates in [-L, L], uniform cells of width h = 2L/n
        h = 2.0 * L / n
        ref = -L + h * ijk.astype(np.float64)
        jit = cfg.get("jitter", 0.0)
        if jit:
            # Q14: jitter U(-delta, delta) per axis in reference cell units, interior nodes only
            idx = (3 * node[:, None] + np.arange(3)[None, :]).reshape(-1)
            d = _uniform(seed, _S_JITTER, idx, -jit, jit).reshape(-1, 3) * h
            ref = ref + d * interior[:, None]
        if grading is not None and grading[0] == "power":
            p = grading[1]
            ref = np.sign(ref) * L * (np.abs(ref) / L) ** p
        xyz = ref
    # exact box faces for boundary nodes
    for a in range(3):
        xyz[ijk[:, a] == 0, a] = -L
        xyz[ijk[:, a] == n, a] = L
    dirichlet = (~interior).astype(np.uint8)
    return xyz, dirichlet


def _nuclei(cfg, seed):
    spec = cfg["nuclei"]
    if isinstance(spec, tuple) and spec[0] == "ball":
        # Q20: uniform in the ball by rejection, min pair distance 1.0 bohr, Z ~ U{1..8}
        _, K, r = spec
        pos, Z = [], []
        ctr = 0
        while len(pos) < K:
            u = _uniform(seed, _S_NUCLEI, 4 * ctr + np.arange(4), 0.0, 1.0)
            ctr += 1
            x = (2.0 * u[:3] - 1.0) * r
            if np.dot(x, x) > r * r:
                continue
            if any(np.linalg.norm(x - q) < 1.0 for q in pos):
                continue
            pos.append(x)
            Z.append(1 + min(7, int(u[3] * 8.0)))
        return np.array(pos), np.array(Z, dtype=np.float64)
    pos = np.array([p for p, _ in spec], dtype=np.float64)
    Z = np.array([z for _, z in spec], dtype=np.float64)
    return pos, Z


def _coarse_interpolation(xyz_free, L, nc):
    """P_H (Q21): locate each fine free node in the uniform unperturbed coarse Kuhn mesh on the
    same box; weights are its barycentric coordinates; coarse Dirichlet vertices and exact zeros
    are dropped. Returns CSR (rowptr, col, val) over coarse FREE nodes and n_H."""
    H = 2.0 * L / nc
    n1 = nc + 1
    f = (xyz_free + L) / H
    cell = np.clip(np.floor(f), 0, nc - 1).astype(np.int64)
    fr = np.clip(f - cell, 0.0, 1.0)
    order = np.argsort(-fr, axis=1, kind="stable")          # sigma: descending fractions
    fs = np.take_along_axis(fr, order, axis=1)
    lam = np.stack([1.0 - fs[:, 0], fs[:, 0] - fs[:, 1], fs[:, 1] - fs[:, 2], fs[:, 2]], axis=1)
    e = np.array([1, n1, n1 * n1], dtype=np.int64)
    base = cell[:, 0] + n1 * (cell[:, 1] + n1 * cell[:, 2])
    v0 = base
    v1 = v0 + e[order[:, 0]]
    v2 = v1 + e[order[:, 1]]
    v3 = base + e.sum()
    verts = np.stack([v0, v1, v2, v3], axis=1)
    # coarse free numbering: interior coarse nodes, lexicographic rank
    cn = verts
    ci, cj, ck = cn % n1, (cn // n1) % n1, cn // (n1 * n1)
    inter = (ci > 0) & (ci < nc) & (cj > 0) & (cj < nc) & (ck > 0) & (ck < nc)
    m = nc - 1
    cfree = (ci - 1) + m * ((cj - 1) + m * (ck - 1))
    keep = inter & (lam != 0.0)
    cols = np.where(keep, cfree, np.iinfo(np.int64).max)
    srt = np.argsort(cols, axis=1, kind="stable")
    cols = np.take_along_axis(cols, srt, axis=1)
    vals = np.take_along_axis(lam, srt, axis=1)
    keep = cols != np.iinfo(np.int64).max
    counts = keep.sum(1)
    rowptr = np.zeros(xyz_free.shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    return (rowptr.astype(np.int32), cols[keep].astype(np.int32), vals[keep].astype(np.float64),
            m ** 3)


def make_problem(cfg: dict | int, **overrides) -> Problem:
    """Build the inputs of one config. `cfg` is a config number or a dict with
    keys L, n, grading, jitter, nuclei, vnoise, N, orbitals, lam, nc, seed and optional
    'potential' ('coulomb' (default) or 'harmonic': V = |x|^2/2)."""
    if isinstance(cfg, int):
        cfg = make_config(cfg, **overrides)
    else:
        cfg = dict(cfg)
        cfg.update(overrides)
        cfg.setdefault("seed", SEED_BASE)
    seed = int(cfg["seed"])
    n, L = int(cfg["n"]), float(cfg["L"])
    nuc, Z = _nuclei(cfg, seed)
    cfg["_nuclei_xyz"] = nuc
    xyz, dirichlet = _grid_coords(cfg, n, L, seed)
    del cfg["_nuclei_xyz"]
    tets = kuhn_mesh(n)
    n_nodes = xyz.shape[0]

    # V_eff on ALL nodes (Q16): -sum Z/sqrt(|x-R|^2+0.01) + vnoise*U(-1,1)
    if cfg.get("potential", "coulomb") == "harmonic":
        V = 0.5 * (xyz * xyz).sum(1)
    else:
        V = np.zeros(n_nodes)
        for r, z in zip(nuc, Z):
            d = xyz - r[None, :]
            V -= z / np.sqrt((d * d).sum(1) + 0.01)
    if cfg.get("vnoise", 0.0):
        V = V + cfg["vnoise"] * _uniform(seed, _S_VNOISE, np.arange(n_nodes), -1.0, 1.0)

    free_nodes = np.nonzero(dirichlet == 0)[0].astype(np.int64)
    xf = xyz[free_nodes]
    n_free = free_nodes.shape[0]
    N = int(cfg["N"])

    # initial orbitals (Q18)
    if cfg.get("orbitals", "gauss") == "exp":
        U = np.exp(-np.sqrt((xf * xf).sum(1)))[:, None] * np.ones((1, N))
    elif cfg["orbitals"] == "gauss":
        U = np.empty((n_free, N))
        K = len(Z)
        for i in range(N):
            c = nuc[i % K] + _uniform(seed, _S_CENTRES, 3 * i + np.arange(3), -0.5, 0.5)
            d = xf - c[None, :]
            U[:, i] = np.exp(-0.5 * (d * d).sum(1))
    elif cfg["orbitals"] == "given":
        U = np.asarray(cfg["U"], dtype=np.float64).reshape(n_free, N).copy()
    else:
        raise ValueError(cfg["orbitals"])
    if cfg.get("unoise", 1e-3) and cfg.get("orbitals") != "given":
        U = U + cfg.get("unoise", 1e-3) * _uniform(
            seed, _S_UNOISE, np.arange(n_free * N), -1.0, 1.0).reshape(n_free, N)
    U = np.ascontiguousarray(U)

    lam_spec = cfg["lam"]
    if lam_spec[0] == "const":
        lam = np.full(N, float(lam_spec[1]))
    elif lam_spec[0] == "uniform":
        lam = _uniform(seed, _S_LAMBDA, np.arange(N), lam_spec[1], lam_spec[2])
    else:
        lam = np.asarray(lam_spec[1], dtype=np.float64).copy()

    # mu = 8 M sum Z^2, M = number of nuclei; overridable
    mu = float(cfg["mu"]) if "mu" in cfg else 8.0 * len(Z) * float((Z * Z).sum())

    nc = int(cfg["nc"])
    prow, pcol, pval, n_H = _coarse_interpolation(xf, L, nc)
    return Problem(cfg=cfg, n_cells=n, L=L, xyz=xyz, tets=tets, dirichlet=dirichlet, V=V,
                   nuclei=nuc, Z=Z, mu=mu, N=N, U=U, lam=lam, nc=nc, n_H=n_H,
                   P_rowptr=prow, P_col=pcol, P_val=pval, free_nodes=free_nodes)


def config_summary(p: Problem) -> dict:
    return dict(name=p.cfg.get("name", "custom"), cells=p.n_cells, nodes=p.n_nodes,
                n_free=p.n_free, tets=p.n_tets, N=p.N, mu=p.mu, n_H=p.n_H, nc=p.nc,
                seed=int(p.cfg["seed"]))
