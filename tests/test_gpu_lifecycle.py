"""Lifecycle of the C-ABI context on the GPU: repeated steps, repeated coarse spaces and the two-level Hartree
setup keep the device footprint flat (no leaks, `ks_memory_bytes`), and two contexts driven on two streams
in an interleaved order give bitwise the results each gives alone (no shared mutable state between
contexts, every launch on the context's stream)."""
import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
DEV = "cuda"


def dt(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _step(ctx, p, U):
    ctx.assemble_veff(dt(p.V), p.mu)
    Ut, _, _ = ctx.block_solve(dt(p.lam), U)
    FA, FB = ctx.project_augmented(Ut)
    return Ut, FA, FB


def test_memory_stays_flat_across_repeated_calls():
    import paper_2404_19249_b200 as ks
    p = gen.make_problem(2)
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet)
    U = dt(p.U)
    rho = None
    sizes = []
    for it in range(4):
        ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
        _step(ctx, p, U)
        rho = ctx.density(U, 2.0)
        ctx.hartree(rho, tol=1e-10)   # builds the two-level coarse operator for this coarse space
        assert ctx.sync() == 0
        sizes.append((ctx.memory_bytes(), torch.cuda.memory_allocated()))
    assert sizes[1] == sizes[2] == sizes[3], sizes


def test_every_device_byte_is_caller_owned():
    """include/ks.h "Memory": the library allocates no device memory of its own. Over a whole step with the
    NEXT rows (create, coarse space, assemble, solve, project, pencil eig, Hartree, host-buffer steps) the
    device's used memory grows only by what torch's allocator holds (plus the CUDA context, the module image and
    the cuSOLVER / cuBLAS handles' fixed state), and every region is used up to its planned size."""
    import paper_2404_19249_b200 as ks
    p = gen.make_problem(3)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free0, total = torch.cuda.mem_get_info()
    reserved0 = torch.cuda.memory_reserved()
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet, max_N=p.N)
    ctx.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
    Ut, FA, FB = _step(ctx, p, dt(p.U))
    ctx.pencil_eig(FA, FB, p.N)
    ctx.hartree(ctx.density(dt(p.U), 2.0), tol=1e-8)
    Vh = torch.from_numpy(p.V).pin_memory()
    lamh = torch.from_numpy(p.lam).pin_memory()
    Uh = torch.from_numpy(p.U).pin_memory()
    ks.solve_step_host(ctx, Vh, p.mu, lamh, Uh)
    assert ctx.sync() == 0
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    grown = (free0 - free1) - (torch.cuda.memory_reserved() - reserved0)
    regions = sum(ctx.memory_usage(r)[0] for r in ("persistent", "workspace", "coarse", "ext"))
    assert ctx.memory_bytes() == regions
    assert torch.cuda.memory_allocated() >= regions
    # what is not torch's: the lazily loaded module image, library handles, copy streams (a few hundred MB at
    # most), never the regions (C3: ~1.5 GB)
    assert grown < 0.25 * regions + (512 << 20), (grown, regions)
    for r in ("persistent", "coarse", "ext"):
        cap, used, peak = ctx.memory_usage(r)
        assert used == cap and peak == cap, (r, cap, used, peak)   # the plan is exact for the fixed layouts
    cap, used, peak = ctx.memory_usage("workspace")
    assert peak <= cap and used < cap


def test_two_contexts_on_two_streams_are_independent():
    import paper_2404_19249_b200 as ks
    pa, pb = gen.make_problem(1), gen.make_problem(2)
    ref = []
    for p in (pa, pb):
        c = ks.Context(p.xyz, p.tets, p.dirichlet)
        c.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
        Ut, FA, FB = _step(c, p, dt(p.U))
        assert c.sync() == 0
        ref.append((Ut.cpu(), FA.cpu(), FB.cpu()))
        del c
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    ca = ks.Context(pa.xyz, pa.tets, pa.dirichlet, stream=sa)
    cb = ks.Context(pb.xyz, pb.tets, pb.dirichlet, stream=sb)
    for c, p, s in ((ca, pa, sa), (cb, pb, sb)):
        with torch.cuda.stream(s):
            c.set_coarse(p.n_H, dt(p.P_rowptr), dt(p.P_col), dt(p.P_val))
    torch.cuda.synchronize()
    outs = {}
    Ua, Ub = dt(pa.U), dt(pb.U)
    torch.cuda.synchronize()
    # interleave the calls of the two contexts
    with torch.cuda.stream(sa):
        ca.assemble_veff(dt(pa.V), pa.mu)
    with torch.cuda.stream(sb):
        cb.assemble_veff(dt(pb.V), pb.mu)
    with torch.cuda.stream(sa):
        Uta, _, _ = ca.block_solve(dt(pa.lam), Ua)
    with torch.cuda.stream(sb):
        Utb, _, _ = cb.block_solve(dt(pb.lam), Ub)
    with torch.cuda.stream(sb):
        outs["b"] = (Utb,) + tuple(cb.project_augmented(Utb))
    with torch.cuda.stream(sa):
        outs["a"] = (Uta,) + tuple(ca.project_augmented(Uta))
    assert ca.sync() == 0 and cb.sync() == 0
    for key, r in (("a", ref[0]), ("b", ref[1])):
        for x, y in zip(outs[key], r):
            assert torch.equal(x.cpu(), y)
