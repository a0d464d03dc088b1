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

void nonlinear_solve(Op* o, const double* g_dev, int dims, size_t nx, size_t ny, size_t nz,
                     double h, const mlsqr_outer_cfg& cfg, double* f_dev, mlsqr_outer_step* steps,
                     int* n_steps, int* stop_reason, int* triggered_at, double* alphas,
                     double* betas) {
  Ctx* c = o->ctx;
  // OuterConfig::validate (outer.cpp:10-27)
  require(cfg.pen_kind >= 0 && cfg.pen_kind <= 3, MLSQR_EINVAL, "unknown penalty kind");
  require(cfg.pen_kind == MLSQR_PEN_TIKHONOV || cfg.T > 0.0, MLSQR_EINVAL, "penalty threshold T must be positive");
  require(cfg.inner_cap >= 1, MLSQR_EINVAL, "inner_cap must be at least 1");
  require(cfg.rel_decrease_threshold < 1.0, MLSQR_EINVAL, "rel_decrease_threshold must lie in (0, 1) (or <= 0: fixed count)");
  require(cfg.max_outer >= 1, MLSQR_EINVAL, "max_outer must be at least 1");
  require(cfg.tau >= 0.0, MLSQR_EINVAL, "tau must be nonnegative");
  validate_stop(cfg.inner_stop);
  const size_t ey = dims >= 2 ? ny : 1, ez = dims >= 3 ? nz : 1;
  require(dims >= 1 && dims <= 3, MLSQR_EINVAL, "grid must be 1D, 2D or 3D");
  require(nx * ey * ez == o->cols, MLSQR_EDIM, "grid does not match operator columns");
  require(o->sol_shape.len == nx, MLSQR_EDIM, "operator solution rows must follow the grid x extent");

  mlsqr_stop inner = cfg.inner_stop;
  if (cfg.inner_cap < inner.max_iters) inner.max_iters = cfg.inner_cap;

  std::unique_ptr<VCycle, void (*)(VCycle*)> vc(
      make_vcycle(c, dims, nx, ny, nz, h, cfg.mg_levels, cfg.nu_pre, cfg.nu_post, cfg.omega,
                  cfg.coarse_sweeps),
      [](VCycle* v) { delete vcycle_as_pc(v); });
  const size_t n = o->cols;
  DevBuf<double> prev(n), cur(n);
  MLSQR_CUDA(cudaMemsetAsync(prev.p, 0, sizeof(double) * n, c->stream));  // f^0 = 0
  std::unique_ptr<Workspace, void (*)(Workspace*)> ws(
      workspace_new(c, o->rows, o->cols, o->data_shape, o->sol_shape, inner.max_iters), workspace_free);
  RowShape s{nx, ey * ez};
  DevBuf<double> pseg(s.segments()), pscr(reduce_scratch_size(s.segments())), pval(1);
  std::vector<mlsqr_iter_rec> trace((size_t)inner.max_iters);
  std::vector<double> al((size_t)inner.max_iters + 1), be((size_t)inner.max_iters + 2);
  std::vector<double> hist;
  *stop_reason = 1;
  *triggered_at = 0;
  *n_steps = 0;
  const int ab = cfg.inner_cap + 1, bb = cfg.inner_cap + 2;
  for (int k = 1; k <= cfg.max_outer; ++k) {
    vcycle_update_async(vc.get(), prev.p, cfg.pen_kind, cfg.T, cfg.epsilon);
    mlsqr_solve_info info{};
    solve_mlsqr(o, vcycle_as_pc(vc.get()), g_dev, cfg.tau, inner, cur.p, trace.data(), al.data(),
                be.data(), &info, ws.get());
    penalty_functional_async(c, dims, nx, ny, nz, h, cur.p, cfg.pen_kind, cfg.T, pseg.p, pscr.p, pval.p);
    double pv = 0.0, eps = 0.0;
    MLSQR_CUDA(cudaMemcpyAsync(&pv, pval.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    MLSQR_CUDA(cudaMemcpyAsync(&eps, vcycle_eps_dev(vc.get()), sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    MLSQR_CUDA(cudaStreamSynchronize(c->stream));
    hist.push_back(pv);
    mlsqr_outer_step& st = steps[k - 1];
    st.k = k;
    st.penalty_value = pv;
    st.inner_iterations = info.iterations;
    st.inner_stop = info.stop_reason;
    st.final_residual = info.iterations == 0 ? be[0] : trace[(size_t)info.iterations - 1].res_data;
    st.eps_used = eps;
    if (alphas) std::memcpy(alphas + (size_t)(k - 1) * ab, al.data(), sizeof(double) * (size_t)info.n_alphas);
    if (betas) std::memcpy(betas + (size_t)(k - 1) * bb, be.data(), sizeof(double) * (size_t)info.n_betas);
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
