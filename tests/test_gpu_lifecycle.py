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
    # most), never the regions (C4: ~12 GB)
    assert grown < (1 << 30), (grown, regions)
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


def test_regions_smaller_than_their_plan_are_refused():
    """include/ks.h "Memory": a region smaller than its plan returns KS_E_WORKSPACE before any kernel writes past
    it; a block wider than max_N returns KS_E_ARG; the setup region may be the workspace; the plan is exact
    (the carved persistent layout uses every planned byte)."""
    import ctypes as C

    import paper_2404_19249_b200 as ks
    L = ks.load_library()
    p = gen.make_problem(1)
    xyz = np.ascontiguousarray(p.xyz)
    tets = np.ascontiguousarray(p.tets, dtype=np.int32)
    dirn = np.ascontiguousarray(p.dirichlet, dtype=np.uint8)
    sz = [C.c_size_t() for _ in range(3)]
    assert L.ks_plan(p.n_nodes, xyz.ctypes.data, p.n_tets, tets.ctypes.data, dirn.ctypes.data, 2,
                     *[C.byref(x) for x in sz]) == 0
    persist, work, setup = (x.value for x in sz)
    assert persist > 0 and work > 0 and setup > 0
    stream = torch.cuda.current_stream().cuda_stream

    def create(pb, wb, sb, shared_setup=False):
        P = torch.empty(max(pb, 1), dtype=torch.uint8, device=DEV)
        W = torch.empty(max(wb, 1), dtype=torch.uint8, device=DEV)
        S = torch.empty(max(sb, 1), dtype=torch.uint8, device=DEV)
        h = C.c_void_p()
        st = L.ks_create(p.n_nodes, xyz.ctypes.data, p.n_tets, tets.ctypes.data, dirn.ctypes.data, 2, P.data_ptr(),
                         pb, W.data_ptr(), wb, None if shared_setup else S.data_ptr(), sb, C.c_void_p(stream),
                         C.byref(h))
        return st, h, (P, W, S)

    # persistent and setup are carved whole by ks_create; the workspace's solver part is carved there and its
    # call scratch by later calls (a workspace too small for the solver part fails here)
    for pb, wb, sb in ((persist - 256, work, setup), (persist, 4096, setup), (persist, work, setup - 256)):
        st, h, _ = create(pb, wb, sb)
        assert st == ks.KS_E_WORKSPACE and not h.value, (pb, wb, sb, st)
        assert b"KS_E_WORKSPACE" in L.ks_last_error(None)
    # the workspace doubles as the setup region when it is large enough
    st, h, keep = create(persist, max(work, setup), 0, shared_setup=True)
    assert st == 0
    cap, used, peak = C.c_size_t(), C.c_size_t(), C.c_size_t()
    assert L.ks_memory_usage(h, 0, C.byref(cap), C.byref(used), C.byref(peak)) == 0
    assert cap.value == used.value == persist
    # N above the planned max_N
    U = torch.zeros((p.n_free, 3), dtype=torch.float64, device=DEV)
    Ut = torch.empty_like(U)
    lam = torch.zeros(3, dtype=torch.float64, device=DEV)
    V = torch.from_numpy(p.V).to(DEV)
    assert L.ks_assemble_veff(h, V.data_ptr(), C.c_double(p.mu)) == 0
    assert L.ks_block_solve(h, 3, lam.data_ptr(), U.data_ptr(), Ut.data_ptr(), C.c_double(1e-10), 100, None,
                            None) == ks.KS_E_ARG
    assert L.ks_sync(h) == 0
    L.ks_destroy(h)
    # a coarse region smaller than its plan
    ctx = ks.Context(p.xyz, p.tets, p.dirichlet, max_N=2)
    n = C.c_size_t()
    Pr, Pc, Pv = dt(p.P_rowptr), dt(p.P_col), dt(p.P_val)
    assert L.ks_coarse_plan(ctx._h, p.n_H, Pr.data_ptr(), Pc.data_ptr(), Pv.data_ptr(), C.byref(n)) == 0
    small = torch.empty(n.value - 256, dtype=torch.uint8, device=DEV)
    assert L.ks_set_coarse(ctx._h, p.n_H, Pr.data_ptr(), Pc.data_ptr(), Pv.data_ptr(), small.data_ptr(),
                           n.value - 256) == ks.KS_E_WORKSPACE
    ctx.set_coarse(p.n_H, Pr, Pc, Pv)   # the binding's planned region works
    assert ctx.memory_usage("coarse")[0] == ctx.memory_usage("coarse")[1]
