// include/mlsqr_b200.hpp -- header-only C++ layer over the C-ABI (mlsqr_b200.h).
//
// 1. check(): maps status codes back to the reference's exception types
//    (errors.hpp:9-41) when the reference headers are visible, so
//    reference-style callers see the same contract (DimensionError,
//    BreakdownError(iteration), std::invalid_argument).
// 2. With MLSQR_B200_WITH_REFERENCE_API defined and the reference's include/
//    on the include path, the adapters
//        mlsqr_b200::GpuLinearOperator : mlsqr::LinearOperator   (linop.hpp:21-47)
//        mlsqr_b200::GpuSpdMap         : mlsqr::SpdMap           (spdsolve.hpp:15-22)
//    let the UNMODIFIED reference mlsqr() / lsqr() / solve_nonlinear-style
//    callers drive the B200 kernels ("parity mode": host spans, one H2D/D2H
//    per call), and gpu_mlsqr() runs the whole solve device-resident and
//    returns a reference mlsqr::SolveResult ("throughput mode").
#pragma once

#include <cstddef>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "mlsqr_b200.h"

#ifdef MLSQR_B200_WITH_REFERENCE_API
#include "mlsqr/errors.hpp"
#include "mlsqr/krylov.hpp"
#include "mlsqr/linop.hpp"
#include "mlsqr/spdsolve.hpp"
#endif

namespace mlsqr_b200 {

inline void check(int status, int breakdown_iteration = 0) {
  if (status == MLSQR_OK) return;
  const std::string msg = mlsqr_last_error();
#ifdef MLSQR_B200_WITH_REFERENCE_API
  if (status == MLSQR_EDIM) throw mlsqr::DimensionError(msg);
  if (status == MLSQR_EBREAKDOWN) throw mlsqr::BreakdownError(msg, breakdown_iteration);
  if (status == MLSQR_EFACTOR) {  // "... nonpositive pivot at row N" (spdsolve.cpp:66-70)
    const auto sp = msg.find_last_of(' ');
    throw mlsqr::FactorizationError(msg, sp == std::string::npos ? 0 : std::stoul(msg.substr(sp + 1)));
  }
#else
  (void)breakdown_iteration;
  if (status == MLSQR_EDIM) throw std::invalid_argument(msg);
  if (status == MLSQR_EBREAKDOWN) throw std::runtime_error(msg);
#endif
  if (status == MLSQR_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("mlsqr_b200 status " + std::to_string(status) + ": " + msg);
}

class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) { check(mlsqr_ctx_create(device, stream, &h_)); }
  ~Context() { mlsqr_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  mlsqr_ctx* get() const { return h_; }

 private:
  mlsqr_ctx* h_ = nullptr;
};

#ifdef MLSQR_B200_WITH_REFERENCE_API

// LinearOperator whose apply / apply_adjoint run on the B200 (host spans in/out).
class GpuLinearOperator final : public mlsqr::LinearOperator {
 public:
  static GpuLinearOperator blur(Context& c, int dims, std::size_t nx, std::size_t ny, std::size_t nz,
                                std::span<const double> taps) {
    mlsqr_op* op = nullptr;
    check(mlsqr_blur_create(c.get(), dims, nx, ny, nz, taps.data(), static_cast<int>(taps.size() / 2), &op));
    return GpuLinearOperator(op);
  }
  // SeparableGaussianBlur2D with its own per-axis factors kx_(nx), ky_(ny) (linop.cpp:142-149)
  static GpuLinearOperator blur2d_axes(Context& c, std::size_t nx, std::size_t ny, std::span<const double> taps_x,
                                       std::span<const double> taps_y) {
    mlsqr_op* op = nullptr;
    check(mlsqr_blur2d_create_axes(c.get(), nx, ny, taps_x.data(), static_cast<int>(taps_x.size() / 2),
                                   taps_y.data(), static_cast<int>(taps_y.size() / 2), &op));
    return GpuLinearOperator(op);
  }
  static GpuLinearOperator dense(Context& c, std::size_t rows, std::size_t cols,
                                 std::span<const double> row_major, std::size_t sol_row_len = 0) {
    mlsqr_op* op = nullptr;
    check(mlsqr_dense_create(c.get(), rows, cols, row_major.data(), MLSQR_HOST, sol_row_len, &op));
    return GpuLinearOperator(op);
  }
  GpuLinearOperator(GpuLinearOperator&& o) noexcept : LinearOperator(o.shape()), op_(o.op_) { o.op_ = nullptr; }
  ~GpuLinearOperator() override { mlsqr_op_destroy(op_); }
  mlsqr_op* handle() const { return op_; }

 private:
  explicit GpuLinearOperator(mlsqr_op* op) : LinearOperator(shape_of(op)), op_(op) {}
  static mlsqr::OperatorShape shape_of(mlsqr_op* op) {
    std::size_t r = 0, c = 0;
    check(mlsqr_op_shape(op, &r, &c));
    return {r, c};
  }
  void do_apply(std::span<const double> x, std::span<double> y) const override {
    check(mlsqr_op_apply(op_, x.data(), x.size(), y.data(), y.size(), MLSQR_HOST));
  }
  void do_apply_adjoint(std::span<const double> y, std::span<double> x) const override {
    check(mlsqr_op_apply_adjoint(op_, y.data(), y.size(), x.data(), x.size(), MLSQR_HOST));
  }
  mlsqr_op* op_;
};

// SpdMap realized by the B200 V-cycle (or identity).
class GpuSpdMap final : public mlsqr::SpdMap {
 public:
  static GpuSpdMap vcycle(Context& c, int dims, std::size_t nx, std::size_t ny, std::size_t nz, double h,
                          int levels, int nu_pre = 2, int nu_post = 2, double omega = 2.0 / 3.0,
                          int coarse_sweeps = 4) {
    mlsqr_pc* pc = nullptr;
    check(mlsqr_vcycle_create(c.get(), dims, nx, ny, nz, h, levels, nu_pre, nu_post, omega, coarse_sweeps, &pc));
    return GpuSpdMap(pc);
  }
  // SpdSolver::factorize of the M a V-cycle map holds (spdsolve.cpp:22-75), on the device;
  // throws mlsqr::FactorizationError(pivot_row) like the reference
  static GpuSpdMap cholesky(const GpuSpdMap& m) {
    mlsqr_pc* pc = nullptr;
    check(mlsqr_chol_map_create(m.handle(), &pc, nullptr));
    return GpuSpdMap(pc);
  }
  // SpdSolver::inner_cg (spdsolve.cpp:77-85): k_inner CG iterations on a snapshot of m's M
  static GpuSpdMap inner_cg(const GpuSpdMap& m, int k_inner) {
    mlsqr_pc* pc = nullptr;
    check(mlsqr_inner_cg_map_create(m.handle(), k_inner, &pc));
    return GpuSpdMap(pc);
  }
  // a host SpdMap plug-in (mlsqr_callback_map_create): fn(user, p, v) on host vectors of length n
  static GpuSpdMap callback(Context& c, std::size_t n, mlsqr_host_map_fn fn, void* user) {
    mlsqr_pc* pc = nullptr;
    check(mlsqr_callback_map_create(c.get(), n, fn, user, &pc));
    return GpuSpdMap(pc);
  }
  GpuSpdMap(GpuSpdMap&& o) noexcept : pc_(o.pc_) { o.pc_ = nullptr; }
  ~GpuSpdMap() override { mlsqr_pc_destroy(pc_); }
  using SpdMap::solve;
  std::size_t dimension() const override {
    std::size_t n = 0;
    check(mlsqr_pc_dimension(pc_, &n));
    return n;
  }
  void solve(std::span<const double> p, std::span<double> v) const override {
    if (p.size() != v.size()) throw mlsqr::DimensionError("solve dimension mismatch");
    check(mlsqr_pc_solve(pc_, p.data(), v.data(), p.size(), MLSQR_HOST));
  }
  // assemble_m + auto_shift at field f (diffusion.cpp:59-87); returns eps
  double update(std::span<const double> f, int pen_kind, double T, double eps = -1.0) {
    double used = 0.0;
    check(mlsqr_vcycle_update(pc_, f.data(), MLSQR_HOST, pen_kind, T, eps, &used));
    return used;
  }
  mlsqr_pc* handle() const { return pc_; }

 private:
  explicit GpuSpdMap(mlsqr_pc* pc) : pc_(pc) {}
  mlsqr_pc* pc_;
};

namespace detail {
inline mlsqr_stop to_c(const mlsqr::StoppingConfig& stop) {
  return {stop.atol, stop.btol, stop.conlim, stop.delta, stop.eta, stop.max_iters,
          stop.use_s1, stop.use_s2, stop.use_s3, stop.use_s4};
}
inline void fill_trace(mlsqr::SolveResult& r, const std::vector<mlsqr_iter_rec>& tr, const mlsqr_solve_info& info) {
  r.iterations = info.iterations;
  static const mlsqr::StopReason kReasons[] = {mlsqr::StopReason::s1, mlsqr::StopReason::s2,
                                               mlsqr::StopReason::s3, mlsqr::StopReason::s4,
                                               mlsqr::StopReason::max_iters, mlsqr::StopReason::breakdown};
  r.stop_reason = kReasons[info.stop_reason];
  for (int i = 0; i < info.iterations; ++i) {
    const auto& t = tr[static_cast<std::size_t>(i)];
    mlsqr::IterationRecord rec;
    rec.iteration = t.iteration;
    rec.res_damped = t.res_damped;
    rec.res_data = t.res_data;
    rec.res_data_exact = t.res_data_exact != 0;
    rec.s2_value = t.s2_value;
    rec.anorm_est = t.anorm_est;
    rec.cond_est = t.cond_est;
    rec.xnorm_est = t.xnorm_est;
    rec.alpha = t.alpha;
    rec.beta = t.beta;
    r.trace.iterations.push_back(rec);
  }
}
}  // namespace detail

// Device-resident mlsqr with the reference's signature semantics (krylov.hpp:94-95) and its
// SolveOptions (krylov.hpp:77-80): store_basis returns the right and left bases, record_snapshots
// the iterate after every iteration (SolveTrace::snapshots).
inline mlsqr::SolveResult gpu_mlsqr(const GpuLinearOperator& a, const GpuSpdMap& m,
                                    std::span<const double> g, double tau,
                                    const mlsqr::StoppingConfig& stop, const mlsqr::SolveOptions& opts = {}) {
  stop.validate();
  if (g.size() != a.n_rows()) throw mlsqr::DimensionError("right-hand side length mismatch");
  const mlsqr_stop s = detail::to_c(stop);
  mlsqr::SolveResult r;
  const std::size_t n = a.n_cols(), k = static_cast<std::size_t>(stop.max_iters);
  r.solution.assign(n, 0.0);
  std::vector<mlsqr_iter_rec> tr(k);
  std::vector<double> al(k + 1), be(k + 2), basis, left, snaps;
  mlsqr_solve_info info{};
  mlsqr_solve_opts o{};
  if (opts.store_basis) {
    basis.assign((k + 1) * n, 0.0);
    left.assign((k + 1) * a.n_rows(), 0.0);
    o.store_basis = 1;
    o.basis = basis.data();
    o.left_basis = left.data();
  }
  if (opts.record_snapshots) {
    snaps.assign(k * n, 0.0);
    o.record_snapshots = 1;
    o.snapshots = snaps.data();
  }
  // status first: the breakdown iteration is only valid once the solve has returned
  // (function arguments are evaluated in an unspecified order)
  const int status = mlsqr_solve_with(a.handle(), m.handle(), g.data(), tau, &s, &o, r.solution.data(), tr.data(),
                                      al.data(), be.data(), &info, MLSQR_HOST);
  check(status, info.breakdown_iteration);
  detail::fill_trace(r, tr, info);
  for (int j = 0; opts.record_snapshots && j < info.iterations; ++j)
    r.trace.snapshots.emplace_back(snaps.begin() + j * n, snaps.begin() + (j + 1) * n);
  r.bidiag.alphas.assign(al.begin(), al.begin() + info.n_alphas);
  r.bidiag.betas.assign(be.begin(), be.begin() + info.n_betas);
  for (int j = 0; opts.store_basis && j < info.n_alphas; ++j)
    r.bidiag.basis.emplace_back(basis.begin() + j * n, basis.begin() + (j + 1) * n);
  const std::size_t mr = a.n_rows();
  for (int j = 0; opts.store_basis && j < info.n_left_basis; ++j)
    r.bidiag.left_basis.emplace_back(left.begin() + j * mr, left.begin() + (j + 1) * mr);
  return r;
}

// cg_normal (krylov.hpp:116-122) on the device; M is the V-cycle map's level-0 operator
// (its update() state), m may be null when tau == 0.
inline mlsqr::SolveResult gpu_cg_normal(const GpuLinearOperator& a, const GpuSpdMap* m, double tau,
                                        std::span<const double> g, const mlsqr::StoppingConfig& stop) {
  stop.validate();
  if (g.size() != a.n_rows()) throw mlsqr::DimensionError("right-hand side length mismatch");
  const mlsqr_stop s = detail::to_c(stop);
  mlsqr::SolveResult r;
  r.solution.assign(a.n_cols(), 0.0);
  std::vector<mlsqr_iter_rec> tr(static_cast<std::size_t>(stop.max_iters));
  mlsqr_solve_info info{};
  const int status = mlsqr_cg_normal_solve(a.handle(), m ? m->handle() : nullptr, g.data(), tau, &s,
                                           r.solution.data(), tr.data(), &info, MLSQR_HOST);
  check(status, info.breakdown_iteration);
  detail::fill_trace(r, tr, info);
  return r;
}

// solve_projected (krylov.hpp:124-127) through the library (bit-identical to the reference)
inline std::vector<double> gpu_solve_projected(const mlsqr::BidiagEntries& bd, double beta1, double tau) {
  std::vector<double> y(bd.alphas.size());
  check(mlsqr_solve_projected(bd.alphas.data(), bd.alphas.size(), bd.betas.data(), bd.betas.size(), beta1, tau,
                              y.data()));
  return y;
}

#endif  // MLSQR_B200_WITH_REFERENCE_API

}  // namespace mlsqr_b200
