// ks_stream.cu -- the hot-path step from HOST buffers, pipelined (ks_step_submit / ks_step_wait).
//
// Each submitted step copies its inputs (V_eff, lambda, U) from pinned host memory, runs ks_assemble_veff,
// ks_block_solve and ks_project_augmented on the context's stream, and copies F_A, F_B back to the host.
// Two device slots alternate between consecutive steps; host->device copies run on one copy stream and
// device->host copies on another, ordered against the compute stream by events, so the input copy of step
// s+1 overlaps the compute of step s (B200: separate H2D and D2H copy engines).
#include "ks_internal.cuh"

// the two device slots live in the extension workspace (KS_EXT_STEP, planned for N <= max_N); the copy streams
// and events are created on first use
static ks_status ensure_step_slots(ks_ctx *ctx, int N) {
  if (!(ctx->ext_features & KS_EXT_STEP) || ctx->ext_nH != ctx->n_H)
    return ks_fail(ctx, KS_E_STATE, "ks_step_submit: attach an extension workspace planned with KS_EXT_STEP for this "
                   "coarse space");
  if (N > ctx->max_N) return ks_fail(ctx, KS_E_ARG, "ks_step_submit: N = %d exceeds max_N = %d", N, ctx->max_N);
  if (!ctx->s_h2d) {
    KS_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking));
    KS_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking));
    for (int s = 0; s < 2; s++) {
      KS_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_h2d[s], cudaEventDisableTiming));
      KS_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_comp[s], cudaEventDisableTiming));
      KS_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_d2h[s], cudaEventDisableTiming));
    }
  }
  return KS_OK;
}

void ks_free_stream(ks_ctx *ctx) {
  if (ctx->s_h2d) {
    cudaStreamSynchronize(ctx->s_h2d);
    cudaStreamSynchronize(ctx->s_d2h);
    cudaStreamDestroy(ctx->s_h2d);
    cudaStreamDestroy(ctx->s_d2h);
    for (int s = 0; s < 2; s++) {
      cudaEventDestroy(ctx->ev_h2d[s]);
      cudaEventDestroy(ctx->ev_comp[s]);
      cudaEventDestroy(ctx->ev_d2h[s]);
    }
  }
  ctx->s_h2d = ctx->s_d2h = nullptr;
}

ks_status ks_step_submit_impl(ks_ctx *ctx, int N, const double *h_V, double mu, const double *h_lambda,
                              const double *h_U, double tol, int max_iter, double *h_FA, double *h_FB) {
  KS_TRY(ensure_step_slots(ctx, N));
  const int s = (int)(ctx->step_count & 1);
  const int64_t n = ctx->n_free, nn = ctx->n_nodes, D = ctx->n_H + N;
  const bool reuse = ctx->step_count >= 2;
  // inputs: after the compute that last used this slot (step - 2)
  if (reuse) KS_CUDA(ctx, cudaStreamWaitEvent(ctx->s_h2d, ctx->ev_comp[s], 0));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->st_V[s], h_V, sizeof(double) * nn, cudaMemcpyHostToDevice, ctx->s_h2d));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->st_lam[s], h_lambda, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->s_h2d));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->st_U[s], h_U, sizeof(double) * n * N, cudaMemcpyHostToDevice, ctx->s_h2d));
  KS_CUDA(ctx, cudaEventRecord(ctx->ev_h2d[s], ctx->s_h2d));
  // compute: after the inputs, and after the read-back of this slot's previous results
  KS_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_h2d[s], 0));
  if (reuse) KS_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_d2h[s], 0));
  KS_TRY(ks_assemble_impl(ctx, ctx->st_V[s], mu));
  KS_TRY(ks_solve_impl(ctx, N, ctx->st_lam[s], ctx->st_U[s], ctx->st_Ut[s], tol, max_iter, nullptr, nullptr));
  KS_TRY(ks_project_impl(ctx, N, ctx->st_Ut[s], ctx->st_FA[s], ctx->st_FB[s]));
  KS_CUDA(ctx, cudaEventRecord(ctx->ev_comp[s], ctx->stream));
  // results
  KS_CUDA(ctx, cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_comp[s], 0));
  KS_CUDA(ctx, cudaMemcpyAsync(h_FA, ctx->st_FA[s], sizeof(double) * D * D, cudaMemcpyDeviceToHost, ctx->s_d2h));
  KS_CUDA(ctx, cudaMemcpyAsync(h_FB, ctx->st_FB[s], sizeof(double) * D * D, cudaMemcpyDeviceToHost, ctx->s_d2h));
  KS_CUDA(ctx, cudaEventRecord(ctx->ev_d2h[s], ctx->s_d2h));
  ctx->step_count++;
  return KS_OK;
}

ks_status ks_step_wait_impl(ks_ctx *ctx) {
  if (ctx->s_h2d) {
    KS_CUDA(ctx, cudaStreamSynchronize(ctx->s_h2d));
    KS_CUDA(ctx, cudaStreamSynchronize(ctx->s_d2h));
  }
  return KS_OK;
}
