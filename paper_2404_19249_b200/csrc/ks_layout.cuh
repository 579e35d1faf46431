// ks_layout.cuh -- the allocation lists of every caller-owned memory region (include/ks.h, "Memory").
// Each layout function is called once with a KsSizer (the plan: ks_plan, ks_coarse_plan, ks_ext_plan) and
// once with a KsCarver (the allocation when the region is bound), so the planned and the carved sizes are
// the same list. Not part of the ABI.
#pragma once
#include "ks_internal.cuh"

struct KsMeshSizes {
  int64_t nn = 0, nt = 0, nf = 0, nnz = 0, nc = 0, ns = 0, sell_total = 0;
};

// carves from the context's current region; the first failure is kept
struct KsCarver {
  ks_ctx *ctx;
  ks_status st = KS_OK;
  explicit KsCarver(ks_ctx *c) : ctx(c) {}
  template <typename T>
  void add(T **p, int64_t count, const char *what) {
    if (st == KS_OK) st = ks_alloc(ctx, (void **)p, sizeof(T) * (size_t)(count > 0 ? count : 1), what);
  }
};

int ks_pow2_at_least(int n);
ks_status ks_count_mesh(int64_t nn, const int32_t *tets, int64_t nt, const uint8_t *dir, KsMeshSizes *z,
                        std::string *err);
ks_status ks_setup_cub_bytes(const KsMeshSizes &z, size_t *bytes);
ks_status ks_coarse_cub_bytes(int64_t nf, size_t *bytes);
ks_status ks_plan_sizes(const KsMeshSizes &z, int max_N, int sm_count, size_t *persist, size_t *work,
                        size_t *setup);

// ---- KS_R_PERSIST (ks_create) ----
template <class A>
void ks_layout_persist(A &a, ks_ctx *c, const KsMeshSizes &z) {
  a.add(&c->d_flags, 1, "flags");
  a.add(&c->d_block_iters, 1, "block iters");
  a.add(&c->barrier, 1, "grid barrier");
  a.add(&c->trace, KS_TRACE_CAP, "pcg trace");
  a.add(&c->trace_count, 1, "pcg trace count");
  a.add(&c->xyz, 3 * z.nn, "xyz");
  a.add(&c->tets, 4 * z.nt, "tets");
  a.add(&c->free_of_node, z.nn, "free_of_node");
  a.add(&c->node_of_free, z.nf, "node_of_free");
  a.add(&c->vol, z.nt, "vol");
  a.add(&c->row_ptr, z.nf + 1 + KS_PAD, "row_ptr");
  a.add(&c->col, z.nnz + KS_PAD, "col");
  a.add(&c->diag_pos, z.nf, "diag_pos");
  a.add(&c->emap, 16 * z.nt, "emap");
  a.add(&c->inv_ptr, z.nnz + 1, "inv_ptr");
  a.add(&c->inv_idx, z.nc, "inv_idx");
  a.add(&c->K, z.nnz + KS_PAD, "K");
  a.add(&c->M, z.nnz + KS_PAD, "M");
  a.add(&c->MV, z.nnz + KS_PAD, "MV");
  a.add(&c->H, z.nnz + KS_PAD, "H");
  a.add(&c->A, z.nnz + KS_PAD, "A");
  a.add(&c->diag, z.nf, "diag");
  a.add(&c->dinv, z.nf + 2, "dinv");   // +2: zero pad for the NP = 1 pairwise streams
  a.add(&c->w_tet, z.nt, "w_tet");
  a.add(&c->v_free, z.nf, "v_free");
  a.add(&c->sell_ptr, z.ns + 1, "sell_ptr");
  a.add(&c->sell_col, z.sell_total, "sell col");
  a.add(&c->sell_A, z.sell_total, "sell A");
  a.add(&c->sell_M, z.sell_total, "sell M");
  a.add(&c->sell_H, z.sell_total, "sell H");
  a.add(&c->sell_K, z.sell_total, "sell K");
  a.add(&c->sell_csr, z.sell_total, "sell -> CSR entry");
  a.add(&c->slot_mask, z.sell_total, "sell star masks");
  a.add(&c->star, z.nf, "row stars");
  a.add(&c->dinvK, z.nf + 2, "1/diag K");
}

// ---- KS_R_SETUP (ks_create only) ----
struct KsSetupTemps {
  uint8_t *dir = nullptr, *cub = nullptr;
  int32_t *flag = nullptr, *scan = nullptr, *sell_cnt = nullptr;
  unsigned long long *bad = nullptr;
  double *grad = nullptr;
  uint64_t *keys = nullptr, *keys_sorted = nullptr;
  int *n_sel = nullptr;
  size_t cub_bytes = 0;
};
template <class A>
void ks_layout_setup(A &a, KsSetupTemps &t, const KsMeshSizes &z, size_t cub_bytes) {
  t.cub_bytes = cub_bytes;
  a.add(&t.dir, z.nn, "setup dir");
  a.add(&t.flag, z.nn, "setup flag");
  a.add(&t.scan, z.nn, "setup scan");
  a.add(&t.bad, 1, "setup bad");
  a.add(&t.cub, (int64_t)cub_bytes, "setup cub");
  a.add(&t.grad, 12 * z.nt, "setup grad");
  a.add(&t.keys, 16 * z.nt, "setup keys");
  a.add(&t.keys_sorted, 16 * z.nt, "setup sorted keys");
  a.add(&t.n_sel, 1, "setup n_sel");
  a.add(&t.sell_cnt, z.ns + 1, "setup sell counts");
}

// ---- KS_R_WORK: solver workspace for N <= max_N (ks_pcg.cu); the rest of the region is call scratch ----
#define KS_PCG_GMAX_PER_SM 2   // persistent PCG blocks per SM the partials are sized for
template <class A>
void ks_layout_work(A &a, ks_ctx *c, int64_t nf, int max_N, int sm_count) {
  const int np = ks_pow2_at_least(max_N);
  const int64_t cnt = nf * (int64_t)np;
  a.add(&c->r, cnt, "pcg r");
  a.add(&c->p, cnt, "pcg p");
  a.add(&c->q, cnt, "pcg q");
  a.add(&c->xpad, cnt, "pcg x pad");
  a.add(&c->upad, cnt, "pcg u pad");
  a.add(&c->bpad, cnt, "pcg b pad");
  a.add(&c->partials, (int64_t)KS_PCG_GMAX_PER_SM * sm_count * 4 * np * 2, "pcg partials");
}

// ---- KS_R_COARSE (ks_set_coarse): sizes known after the item grouping ----
struct KsCoarseSizes {
  int64_t nf = 0, nnz = 0, pn = 0, ni = 0, dtot = 0, nH = 0, gram = 0;
  int64_t nis = 0, istot = 0;   // item slices, item-layout slots
  int np = 2;   // projection block width (>= 2)
};
template <class A>
void ks_layout_coarse(A &a, ks_ctx *c, const KsCoarseSizes &s) {
  a.add(&c->P_ptr, s.nf + 1, "P_ptr");
  a.add(&c->P_col, s.pn, "P_col");
  a.add(&c->P_val, s.pn, "P_val");
  a.add(&c->perm, s.nf, "perm");
  a.add(&c->Pv4, 4 * s.nf, "Pv4");
  a.add(&c->pos_of_row, s.nf, "pos_of_row");
  a.add(&c->Pv4p, 4 * s.nf, "Pv4 (item order)");
  a.add(&c->item_ptr, s.ni + 1, "item_ptr");
  a.add(&c->item_S, 4 * s.ni, "item_S");
  a.add(&c->CT_val, 4 * s.ni, "CT_val");
  a.add(&c->item_D_ptr, s.ni + 1, "item_D_ptr");
  a.add(&c->item_D, s.dtot, "item_D");
  a.add(&c->slotmap, 4 * s.nnz, "slotmap");
  a.add(&c->CT_ptr, s.nH + 1, "CT_ptr");
  a.add(&c->AH_part, 4 * s.dtot, "AH_part");
  a.add(&c->B_H, s.nH * s.nH, "B_H");
  a.add(&c->Y_H, s.nf * s.np, "Y_H (item order)");
  a.add(&c->Y_M, s.nf * s.np, "Y_M (item order)");
  a.add(&c->proj_u, s.nf * s.np, "proj U pad");
  a.add(&c->proj_up, s.nf * s.np, "proj U (item order)");
  a.add(&c->bH_part, 4 * s.ni * s.np, "bH_part");
  a.add(&c->cH_part, 4 * s.ni * s.np, "cH_part");
  a.add(&c->gram_part, s.gram, "gram partials");
  a.add(&c->islice0, s.ni + 1, "item first slice");
  a.add(&c->isell_ptr, s.nis + 1, "item sell ptr");
  a.add(&c->inat, s.nf, "item rows: natural sell base");
  a.add(&c->isell_col, s.istot, "item sell col");
  a.add(&c->islot, s.istot, "item sell window slots");
}

// temporaries of ks_set_coarse (call scratch in KS_R_WORK); the grouping arrays first live here too
struct KsCoarseTemps {
  int32_t *P_ptr = nullptr, *P_col = nullptr, *perm = nullptr, *pos_of_row = nullptr;
  double *P_val = nullptr, *Pv4 = nullptr, *Pv4p = nullptr;
  int32_t *item_ptr = nullptr, *item_S = nullptr, *item_D_ptr = nullptr;
  unsigned long long *bad = nullptr;
  uint64_t *key = nullptr, *key_sorted = nullptr;
  int32_t *rows = nullptr, *flag = nullptr, *gincl = nullptr, *gfirst = nullptr, *iflag = nullptr, *iincl = nullptr;
  int32_t *item_of_pos = nullptr, *ct_key = nullptr, *ct_key_sorted = nullptr, *ct_val = nullptr, *dcnt = nullptr;
  int32_t *islice0 = nullptr, *isw = nullptr, *isell_ptr = nullptr;   // item slices (first, widths, slot offsets)
  int *dmax = nullptr;
  uint8_t *cub = nullptr;
  size_t cub_bytes = 0;
};
// the part sized by n_free and p_nnz (before the item count is known)
template <class A>
void ks_layout_coarse_temps_rows(A &a, KsCoarseTemps &t, int64_t nf, int64_t pn, size_t cub_bytes) {
  t.cub_bytes = cub_bytes;
  a.add(&t.P_ptr, nf + 1, "c.P_ptr");
  a.add(&t.P_col, pn, "c.P_col");
  a.add(&t.P_val, pn, "c.P_val");
  a.add(&t.perm, nf, "c.perm");
  a.add(&t.Pv4, 4 * nf, "c.Pv4");
  a.add(&t.pos_of_row, nf, "c.pos_of_row");
  a.add(&t.Pv4p, 4 * nf, "c.Pv4p");
  a.add(&t.bad, 1, "c.bad");
  a.add(&t.key, nf, "c.key");
  a.add(&t.key_sorted, nf, "c.key_sorted");
  a.add(&t.rows, nf, "c.rows");
  a.add(&t.cub, (int64_t)cub_bytes, "c.cub");
  a.add(&t.flag, nf, "c.flag");
  a.add(&t.gincl, nf, "c.gincl");
  a.add(&t.gfirst, nf, "c.gfirst");
  a.add(&t.iflag, nf, "c.iflag");
  a.add(&t.iincl, nf, "c.iincl");
  a.add(&t.item_of_pos, nf, "c.item_of_pos");
  a.add(&t.dmax, 1, "c.dmax");
}
// the part sized by the item count
template <class A>
void ks_layout_coarse_temps_items(A &a, KsCoarseTemps &t, int64_t ni, int64_t nf) {
  a.add(&t.item_ptr, ni + 1, "c.item_ptr");
  a.add(&t.item_S, 4 * ni, "c.item_S");
  a.add(&t.item_D_ptr, ni + 1, "c.item_D_ptr");
  a.add(&t.ct_key, 4 * ni, "c.ct_key");
  a.add(&t.ct_key_sorted, 4 * ni, "c.ct_key_sorted");
  a.add(&t.ct_val, 4 * ni, "c.ct_val");
  a.add(&t.dcnt, ni + 1, "c.dcnt");
  const int64_t nis = ni + (nf + 7) / 8;   // sum of ceil(rows / 8) over items
  a.add(&t.islice0, ni + 1, "c.islice0");
  a.add(&t.isw, nis + 1, "c.isw");
  a.add(&t.isell_ptr, nis + 1, "c.isell_ptr");
}

// call scratch of KS_R_WORK: ks_set_coarse's temporaries (items <= rows, p_nnz <= 4 rows) and the
// true-residual partials
inline size_t ks_scratch_bound(const KsMeshSizes &z, int max_N, int sm_count, size_t coarse_cub) {
  KsSizer s;
  KsCoarseTemps t;
  ks_layout_coarse_temps_rows(s, t, z.nf, 4 * z.nf, coarse_cub);
  ks_layout_coarse_temps_items(s, t, z.nf, z.nf);
  KsSizer r;
  double *part = nullptr;
  r.add(&part, (int64_t)2 * max_N * 4 * sm_count, "true residual partials");
  return s.bytes > r.bytes ? s.bytes : r.bytes;
}

// ---- KS_R_EXT (ks_attach_ext): the NEXT-1/2 rows and the host-buffer step pipeline ----
#define KS_EXT_NSLOT2L 8     // block partial slots of the two-level Hartree kernel (ks_pcg2l.cu NSLOT)
#define KS_EXT_AMAX 8        // Anderson history bound (ks_scf.cu AMAX)
#define KS_EXT_DEPTH_MAX 7   // largest Anderson depth ks_scf_solve accepts
#define KS_EXT_EF_GUARD 24   // most guard vectors of the filtered pencil eigensolver (ks_outer.cu EF_GUARD_MAX)
#define KS_EXT_BLAS_WS (32u << 20)   // cuBLAS workspace handed over with cublasSetWorkspace
struct KsExtSizes {
  unsigned features = 0;
  int64_t nn = 0, nt = 0, nf = 0, nH = 0, ni = 0, D = 0, lwork = 1;
  int N = 1, sm_count = 1;
};
template <class A>
void ks_layout_ext(A &a, ks_ctx *c, const KsExtSizes &e) {
  const int64_t D = e.D, N = e.N, m = e.N + KS_EXT_EF_GUARD;
  if (e.features & (KS_EXT_EIG | KS_EXT_SCF)) {
    a.add(&c->eig_A, D * D, "pencil A");
    a.add(&c->eig_B, D * D, "pencil B");
    a.add(&c->eig_w, D, "pencil eigenvalues");
    a.add(&c->eig_info, 1, "pencil info");
    a.add(&c->eig_work, e.lwork, "cuSOLVER workspace");
    a.add(&c->ef_buf, 4 * D * m, "filtered eig blocks");
    a.add(&c->ef_small, 2 * m * m + m + 1, "filtered eig small");
    a.add(&c->ef_dev, ks_ef_device_scratch(e.sm_count, (int)m, D), "filtered eig device scratch");
    a.add(&c->blas_ws, (int64_t)KS_EXT_BLAS_WS, "cuBLAS workspace");
    if (e.nH > 0) {   // cached coarse factor and the explicit L^-1 of the fast reduction
      a.add(&c->ef_LH, e.nH * e.nH, "L_H");
      a.add(&c->ef_LHinv, e.nH * e.nH, "L_H^-1");
      a.add(&c->ef_Linv, D * D, "L^-1");
      a.add(&c->ef_TD, D * D, "reduction temporary");
      a.add(&c->ef_aux, 2 * e.nH * N + 2 * N * N + 8, "Schur pieces");
    }
    a.add(&c->outer_Ut, e.nf * N, "outer U~");
    a.add(&c->outer_FA, D * D, "outer F_A");
    a.add(&c->outer_FB, D * D, "outer F_B");
    a.add(&c->outer_Y, D * N, "outer Y");
    a.add(&c->outer_lam, N, "outer lambda");
  }
  if (e.features & KS_EXT_SCF) {
    a.add(&c->har_w, e.nn, "hartree w");
    a.add(&c->har_c, 4 * e.nt, "hartree element loads");
    a.add(&c->har_b, e.nf, "hartree rhs");
    a.add(&c->har_x0, e.nf, "hartree x0");
    a.add(&c->har_x, e.nf, "hartree x");
    a.add(&c->har_mom, 16, "hartree moments");
    a.add(&c->har_part, 9 * 8 * (int64_t)e.sm_count, "hartree partials");
    a.add(&c->har_iters, 1, "hartree iterations");
    if (e.nH > 0) {
      a.add(&c->har2l_KHinv, e.nH * e.nH, "K_H^-1");
      a.add(&c->har2l_rpart, 4 * e.ni, "restriction partials");
      a.add(&c->har2l_rH, e.nH, "r_H");
      a.add(&c->har2l_y, e.nH, "y_H");
      a.add(&c->har2l_r, e.nf, "2l r");
      a.add(&c->har2l_r2, e.nf, "2l r'");
      a.add(&c->har2l_p, e.nf, "2l p");
      a.add(&c->har2l_q, e.nf, "2l q");
      a.add(&c->har2l_part, (int64_t)KS_EXT_NSLOT2L * 4 * e.sm_count, "2l partials");
      a.add(&c->har2l_Pc4, 4 * e.nf, "P columns 4-wide");
    }
    a.add(&c->scf_rho, e.nn, "scf rho");
    a.add(&c->scf_in, e.nn, "scf rho_in");
    a.add(&c->scf_out, e.nn, "scf rho_out");
    a.add(&c->scf_vh, e.nn, "scf V_H");
    a.add(&c->scf_vxc, e.nn, "scf V_xc");
    a.add(&c->scf_veff, e.nn, "scf V_eff");
    a.add(&c->scf_Ut, e.nf * N, "scf U~");
    a.add(&c->scf_FA, D * D, "scf F_A");
    a.add(&c->scf_FB, D * D, "scf F_B");
    a.add(&c->scf_Y, D * N, "scf Y");
    a.add(&c->scf_hin, (int64_t)KS_EXT_DEPTH_MAX * e.nn, "anderson in");
    a.add(&c->scf_hout, (int64_t)KS_EXT_DEPTH_MAX * e.nn, "anderson out");
    a.add(&c->scf_part, (int64_t)4 * e.sm_count * (KS_EXT_AMAX * KS_EXT_AMAX + KS_EXT_AMAX), "scf partials");
    a.add(&c->scf_red, KS_EXT_AMAX * KS_EXT_AMAX + KS_EXT_AMAX, "scf reductions");
    a.add(&c->scf_alpha, KS_EXT_AMAX, "anderson alpha");
    a.add(&c->scf_slot, KS_EXT_AMAX + 1, "anderson slots");
  }
  if (e.features & KS_EXT_STEP) {
    for (int s = 0; s < 2; s++) {
      a.add(&c->st_V[s], e.nn, "step V");
      a.add(&c->st_lam[s], N, "step lambda");
      a.add(&c->st_U[s], e.nf * N, "step U");
      a.add(&c->st_Ut[s], e.nf * N, "step U~");
      a.add(&c->st_FA[s], D * D, "step F_A");
      a.add(&c->st_FB[s], D * D, "step F_B");
    }
  }
}
