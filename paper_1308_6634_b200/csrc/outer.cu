// outer.cu -- the lagged-diffusivity fixed-point loop around the hot path
// (solve_nonlinear, outer.cpp:40-100), device-resident: each outer step
// rebuilds the V-cycle hierarchy from the previous iterate on the device
// (K_D + auto shift + Galerkin coarsening; no CSR, no std::map), runs the
// device mlsqr from zero, and evaluates R(f^k) with a canonical reduction.
// With rel_decrease_threshold <= 0 the loop runs a fixed count (BASELINE
// configs "K outer x I inner"); otherwise the stagnation rule of
// outer_stop_check (outer.cpp:31-38) applies and f^{k-1} is returned.
#include <cstring>
#include <memory>

#include "internal.cuh"

namespace mlsqr_b200 {

static bool outer_stop_check(const std::vector<double>& hist, double threshold) {
  const size_t k = hist.size();
  if (k < 2) return false;
  const double prev = hist[k - 2];
  if (prev == 0.0) return true;
  return (hist[k - 1] - prev) / prev > -threshold;
}

OuterSolver::OuterSolver(Op* o, int dims, size_t nx, size_t ny, size_t nz, double h,
                         const mlsqr_outer_cfg& cfg)
    : op(o), dims_(dims), nx_(nx), ny_(ny), nz_(nz), h_(h), cfg_(cfg) {
  // OuterConfig::validate (outer.cpp:10-27)
  require(cfg.pen_kind >= 0 && cfg.pen_kind <= 3, MLSQR_EINVAL, "unknown penalty kind");
  require(cfg.pen_kind == MLSQR_PEN_TIKHONOV || cfg.T > 0.0, MLSQR_EINVAL,
          "penalty threshold T must be positive");
  require(cfg.inner_cap >= 1, MLSQR_EINVAL, "inner_cap must be at least 1");
  require(cfg.rel_decrease_threshold < 1.0, MLSQR_EINVAL,
          "rel_decrease_threshold must lie in (0, 1) (or <= 0: fixed count)");
  require(cfg.max_outer >= 1, MLSQR_EINVAL, "max_outer must be at least 1");
  require(cfg.tau >= 0.0, MLSQR_EINVAL, "tau must be nonnegative");
  validate_stop(cfg.inner_stop);
  require(dims >= 1 && dims <= 3, MLSQR_EINVAL, "grid must be 1D, 2D or 3D");
  const size_t ey = dims >= 2 ? ny : 1, ez = dims >= 3 ? nz : 1;
  require(nx * ey * ez == o->cols, MLSQR_EDIM, "grid does not match operator columns");
  require(o->sol_shape.len == nx, MLSQR_EDIM, "operator solution rows must follow the grid x extent");
  inner_ = cfg.inner_stop;
  if (cfg.inner_cap < inner_.max_iters) inner_.max_iters = cfg.inner_cap;
  require(cfg.spd_mode >= MLSQR_SPD_VCYCLE && cfg.spd_mode <= MLSQR_SPD_INNER_CG, MLSQR_EINVAL,
          "unknown SpdSolver mode");
  require(cfg.spd_mode != MLSQR_SPD_INNER_CG || cfg.k_inner >= 1, MLSQR_EINVAL, "inner-CG mode needs k_inner >= 1");
  if (cfg.spd_mode == MLSQR_SPD_VCYCLE)
    vc_ = make_vcycle(o->ctx, dims, nx, ny, nz, h, cfg.mg_levels, cfg.nu_pre, cfg.nu_post, cfg.omega,
                      cfg.coarse_sweeps);
  else  // a one-level V-cycle is the device holder of M; the SpdSolver is rebuilt from it per step
    vc_ = make_vcycle(o->ctx, dims, nx, ny, nz, h, 1, 1, 1, 1.0, 1);
  ws_ = workspace_new(o->ctx, o->rows, o->cols, o->data_shape, o->sol_shape, inner_.max_iters, op_guard(o));
  RowShape s{nx, ey * ez};
  const size_t J = s.segments(), G = dist_gather_size(o->ctx, J);
  pseg_.alloc(J);
  pscr_.alloc(reduce_scratch_size(G > J ? G : J) + J);
  pgat_.alloc(G > 0 ? G : 1);
  pval_.alloc(1);
  if (o->ctx->sharded()) {
    const size_t plane = nx * ey;
    pfg_.alloc(s.n() + 2 * plane);
    MLSQR_CUDA(cudaMemsetAsync(pfg_.p, 0, sizeof(double) * pfg_.n, o->ctx->stream));
  }
  trace_.resize((size_t)inner_.max_iters);
  al_.resize((size_t)inner_.max_iters + 1);
  be_.resize((size_t)inner_.max_iters + 2);
}

OuterSolver::~OuterSolver() {
  delete vcycle_as_pc(vc_);
  workspace_free(ws_);
}

// one outer step of outer.cpp:59-87 from f_prev (device) into f_out (device)
void OuterSolver::step(const double* g, const double* f_prev, double* f_out, mlsqr_outer_step* st,
                       int k) {
  Ctx* c = op->ctx;
  vcycle_update_async(vc_, f_prev, cfg_.pen_kind, cfg_.T, cfg_.epsilon);
  // outer.cpp:64-70: SpdSolver::factorize / inner_cg of this step's M, or the V-cycle itself
  std::unique_ptr<Pc> solver;
  if (cfg_.spd_mode == MLSQR_SPD_CHOLESKY) solver.reset(make_chol_map(vc_, nullptr));
  if (cfg_.spd_mode == MLSQR_SPD_INNER_CG) solver.reset(make_inner_cg_map(vc_, cfg_.k_inner));
  mlsqr_solve_info info{};
  if (g_ready) MLSQR_CUDA(cudaStreamWaitEvent(c->stream, g_ready, 0));
  solve_mlsqr(op, solver ? solver.get() : vcycle_as_pc(vc_), g, cfg_.tau, inner_, f_out, trace_.data(), al_.data(),
              be_.data(), &info, ws_);
  if (out_host) {  // f_out is final: send it home on the side stream while R(f) is evaluated
    cudaStream_t side = c->side_stream();
    MLSQR_CUDA(cudaEventRecord(c->ev_copy2, c->stream));
    MLSQR_CUDA(cudaStreamWaitEvent(side, c->ev_copy2, 0));
    MLSQR_CUDA(cudaMemcpyAsync(out_host, f_out, sizeof(double) * op->cols, cudaMemcpyDeviceToHost, side));
  }
  penalty_functional_async(c, dims_, nx_, ny_, nz_, h_, f_out, cfg_.pen_kind, cfg_.T, pseg_.p,
                           pscr_.p, pgat_.p, pfg_.p ? pfg_.p + nx_ * (dims_ >= 2 ? ny_ : 1) : nullptr,
                           pval_.p);
  double pv = 0.0, eps = 0.0;
  MLSQR_CUDA(cudaMemcpyAsync(&pv, pval_.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  MLSQR_CUDA(cudaMemcpyAsync(&eps, vcycle_eps_dev(vc_), sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  MLSQR_CUDA(cudaStreamSynchronize(c->stream));
  if (out_host) MLSQR_CUDA(cudaStreamSynchronize(c->side));
  last_info = info;
  if (st) {
    st->k = k;
    st->penalty_value = pv;
    st->inner_iterations = info.iterations;
    st->inner_stop = info.stop_reason;
    st->final_residual = info.iterations == 0 ? be_[0] : trace_[(size_t)info.iterations - 1].res_data;
    st->eps_used = eps;
  }
}

void nonlinear_solve(Op* o, const double* g_dev, int dims, size_t nx, size_t ny, size_t nz,
                     double h, const mlsqr_outer_cfg& cfg, double* f_dev, mlsqr_outer_step* steps,
                     int* n_steps, int* stop_reason, int* triggered_at, double* alphas,
                     double* betas) {
  Ctx* c = o->ctx;
  OuterSolver os(o, dims, nx, ny, nz, h, cfg);
  const size_t n = o->cols;
  DevBuf<double> prev(n), cur(n);
  MLSQR_CUDA(cudaMemsetAsync(prev.p, 0, sizeof(double) * n, c->stream));  // f^0 = 0
  std::vector<double> hist;
  *stop_reason = 1;
  *triggered_at = 0;
  *n_steps = 0;
  const int ab = cfg.inner_cap + 1, bb = cfg.inner_cap + 2;
  for (int k = 1; k <= cfg.max_outer; ++k) {
    mlsqr_outer_step& st = steps[k - 1];
    os.step(g_dev, prev.p, cur.p, &st, k);
    hist.push_back(st.penalty_value);
    if (alphas) std::memcpy(alphas + (size_t)(k - 1) * ab, os.al_.data(), sizeof(double) * (size_t)os.last_info.n_alphas);
    if (betas) std::memcpy(betas + (size_t)(k - 1) * bb, os.be_.data(), sizeof(double) * (size_t)os.last_info.n_betas);
    *n_steps = k;
    if (cfg.rel_decrease_threshold > 0.0 && outer_stop_check(hist, cfg.rel_decrease_threshold)) {
      *stop_reason = 0;  // stagnation: return f^{k-1}
      *triggered_at = k;
      break;
    }
    std::swap(prev.p, cur.p);
  }
  MLSQR_CUDA(cudaMemcpyAsync(f_dev, prev.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  MLSQR_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace mlsqr_b200
