// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference core compiled from
// /root/reference/proj/src (see oracle/Makefile).  Output goes only to
// oracle/_ref/libmlsqr_ref.so.  Used to (1) generate the golden fixtures in
// tests/golden/ from the reference itself, (2) drive the reference's own
// mlsqr() with other operators / maps through C callbacks (the oracle's
// restated 3D blur and V-cycle for the CPU baseline, or the CUDA product's
// C-ABI operators in "parity mode"), and (3) time the reference on the GPU
// box's host for bench.py --impl reference.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <vector>

#include "mlsqr/diffusion.hpp"
#include "mlsqr/grid.hpp"
#include "mlsqr/kernels.hpp"
#include "mlsqr/krylov.hpp"
#include "mlsqr/linop.hpp"
#include "mlsqr/outer.hpp"
#include "mlsqr/penalty.hpp"
#include "mlsqr/problems.hpp"
#include "mlsqr/rng.hpp"
#include "mlsqr/sparse.hpp"
#include "mlsqr/spdsolve.hpp"

using namespace mlsqr;

extern "C" {

typedef int (*ref_vec_fn)(void* ctx, const double* in, double* out);

// operator descriptor
typedef struct {
  int kind;  // 0 identity(n=cols) 1 dense 2 conv1d 3 blur2d 4 callback
  size_t rows, cols;
  const double* a;        // dense row-major
  size_t nx, ny;          // conv1d: nx; blur2d: nx, ny
  double sigma;           // conv1d / blur2d sigma_f (domain units)
  ref_vec_fn apply, adjoint;
  void* ctx;
} ref_op_desc;

// preconditioner-map descriptor
typedef struct {
  int kind;  // 0 identity 1 cholesky(dense m) 2 cholesky(assembled M) 3 inner_cg(assembled M) 4 callback
  size_t n;
  const double* m;        // dense SPD (kind 1)
  int dims;
  size_t nx, ny;
  double h;
  const double* f;        // field M is assembled at (kind 2/3)
  int pen_kind;
  double T;
  double eps;             // < 0: auto shift
  int k_inner;
  ref_vec_fn solve;
  void* ctx;
} ref_map_desc;

typedef struct {
  double atol, btol, conlim, delta, eta;
  int max_iters;
  int use_s1, use_s2, use_s3, use_s4;
} ref_stop;

typedef struct {
  int iteration;
  int res_data_exact;
  double res_damped, res_data, s2_value, anorm_est, cond_est, xnorm_est, alpha, beta;
} ref_iter_rec;

typedef struct {
  int iterations;
  int stop_reason;
  int n_alphas, n_betas;
  int breakdown_iteration;
} ref_solve_info;

}  // extern "C"

namespace {

// timing hook for the CPU baseline: steady_clock stamp at the mark-th forward apply
// (the forward apply happens once per mlsqr iteration and never in its init,
// krylov.cpp:389), so [stamp, end) covers exactly the iterations after the mark.
thread_local long g_apply_calls = 0;
thread_local long g_apply_mark = -1;
thread_local std::chrono::steady_clock::time_point g_mark_time;

class CallbackOperator final : public LinearOperator {
 public:
  CallbackOperator(const ref_op_desc& d) : LinearOperator({d.rows, d.cols}), d_(d) {}

 private:
  void do_apply(std::span<const double> x, std::span<double> y) const override {
    if (++g_apply_calls == g_apply_mark) g_mark_time = std::chrono::steady_clock::now();
    if (d_.apply(d_.ctx, x.data(), y.data()) != 0) throw std::runtime_error("callback apply failed");
  }
  void do_apply_adjoint(std::span<const double> y, std::span<double> x) const override {
    if (d_.adjoint(d_.ctx, y.data(), x.data()) != 0)
      throw std::runtime_error("callback adjoint failed");
  }
  ref_op_desc d_;
};

class CallbackMap final : public SpdMap {
 public:
  CallbackMap(size_t n, ref_vec_fn fn, void* ctx) : n_(n), fn_(fn), ctx_(ctx) {}
  using SpdMap::solve;
  std::size_t dimension() const override { return n_; }
  void solve(std::span<const double> p, std::span<double> v) const override {
    if (fn_(ctx_, p.data(), v.data()) != 0) throw std::runtime_error("callback solve failed");
  }

 private:
  size_t n_;
  ref_vec_fn fn_;
  void* ctx_;
};

PenaltySpec make_spec(int kind, double T) {
  switch (kind) {
    case 0: return PenaltySpec::tikhonov();
    case 1: return PenaltySpec::tv_smoothed(T);
    case 2: return PenaltySpec::perona_malik_log(T);
    default: return PenaltySpec::perona_malik_exp(T);
  }
}

Grid make_grid(int dims, size_t nx, size_t ny, double h) {
  return dims == 1 ? Grid::line(nx, h) : Grid::plane(nx, ny, h);
}

std::unique_ptr<LinearOperator> make_op(const ref_op_desc* d) {
  switch (d->kind) {
    case 0: return std::make_unique<IdentityOperator>(d->cols);
    case 1:
      return std::make_unique<DenseOperator>(
          d->rows, d->cols, std::vector<double>(d->a, d->a + d->rows * d->cols));
    case 2: return std::make_unique<GaussianConvolution1D>(d->nx, d->sigma, 1.0);
    case 3: return std::make_unique<SeparableGaussianBlur2D>(d->nx, d->ny, d->sigma);
    default: return std::make_unique<CallbackOperator>(*d);
  }
}

struct MapHolder {
  std::unique_ptr<SpdMap> map;
  std::unique_ptr<SpdSolver> solver;
  const SpdMap& get() const { return solver ? *solver : *map; }
};

MapHolder make_map(const ref_map_desc* d) {
  MapHolder h;
  switch (d->kind) {
    case 0: h.map = std::make_unique<IdentityMap>(d->n); break;
    case 1: {
      const SparseSpd m = SparseSpd::from_dense(d->n, std::span<const double>(d->m, d->n * d->n));
      h.solver = std::make_unique<SpdSolver>(SpdSolver::factorize(m));
      break;
    }
    case 2:
    case 3: {
      const Grid grid = make_grid(d->dims, d->nx, d->ny, d->h);
      SparseSpd m = assemble_m(grid, std::span<const double>(d->f, grid.num_nodes()),
                               make_spec(d->pen_kind, d->T), 0.0);
      m = m.with_shift(d->eps >= 0.0 ? d->eps : auto_shift(m));
      if (d->kind == 2) {
        h.solver = std::make_unique<SpdSolver>(SpdSolver::factorize(m));
      } else {
        h.solver = std::make_unique<SpdSolver>(SpdSolver::inner_cg(m, d->k_inner));
      }
      break;
    }
    default: h.map = std::make_unique<CallbackMap>(d->n, d->solve, d->ctx); break;
  }
  return h;
}

StoppingConfig make_stop(const ref_stop* s) {
  StoppingConfig c;
  c.atol = s->atol;
  c.btol = s->btol;
  c.conlim = s->conlim;
  c.delta = s->delta;
  c.eta = s->eta;
  c.max_iters = s->max_iters;
  c.use_s1 = s->use_s1;
  c.use_s2 = s->use_s2;
  c.use_s3 = s->use_s3;
  c.use_s4 = s->use_s4;
  return c;
}

int reason_code(StopReason r) {
  switch (r) {
    case StopReason::s1: return 0;
    case StopReason::s2: return 1;
    case StopReason::s3: return 2;
    case StopReason::s4: return 3;
    case StopReason::max_iters: return 4;
    case StopReason::breakdown: return 5;
  }
  return -1;
}

void export_result(const SolveResult& r, size_t n, double* f, ref_iter_rec* trace,
                   double* alphas, double* betas, double* snapshots, ref_solve_info* info) {
  if (f) std::memcpy(f, r.solution.data(), sizeof(double) * n);
  if (trace) {
    for (size_t i = 0; i < r.trace.iterations.size(); ++i) {
      const auto& t = r.trace.iterations[i];
      trace[i] = {t.iteration, t.res_data_exact ? 1 : 0, t.res_damped, t.res_data, t.s2_value,
                  t.anorm_est, t.cond_est, t.xnorm_est, t.alpha, t.beta};
    }
  }
  if (alphas) std::memcpy(alphas, r.bidiag.alphas.data(), sizeof(double) * r.bidiag.alphas.size());
  if (betas) std::memcpy(betas, r.bidiag.betas.data(), sizeof(double) * r.bidiag.betas.size());
  if (snapshots) {
    for (size_t i = 0; i < r.trace.snapshots.size(); ++i)
      std::memcpy(snapshots + i * n, r.trace.snapshots[i].data(), sizeof(double) * n);
  }
  if (info) {
    info->iterations = r.iterations;
    info->stop_reason = reason_code(r.stop_reason);
    info->n_alphas = static_cast<int>(r.bidiag.alphas.size());
    info->n_betas = static_cast<int>(r.bidiag.betas.size());
  }
}

template <typename F>
int guarded(F&& fn, ref_solve_info* info = nullptr) {
  try {
    fn();
    return 0;
  } catch (const DimensionError&) {
    return 1;
  } catch (const BreakdownError& e) {
    if (info) info->breakdown_iteration = e.iteration();
    return 3;
  } catch (const FactorizationError&) {
    return 4;
  } catch (const std::invalid_argument&) {
    return 2;
  } catch (...) {
    return 5;
  }
}

}  // namespace

extern "C" {

const char* ref_kernel_backend() {
  static std::string name(kernels::backend_name());
  return name.c_str();
}

int ref_select_backend(int scalar) {
  return kernels::select(scalar ? kernels::Backend::scalar : kernels::Backend::avx2) ? 0 : 1;
}

int ref_taps(size_t n, double sigma, double* out, int* radius) {
  return guarded([&] {
    GaussianConvolution1D c(n, sigma, 1.0);
    *radius = static_cast<int>(c.radius());
    if (out) std::memcpy(out, c.taps().data(), sizeof(double) * c.taps().size());
  });
}

int ref_op_apply(const ref_op_desc* d, const double* x, double* y) {
  return guarded([&] {
    auto op = make_op(d);
    op->apply(std::span<const double>(x, op->n_cols()), std::span<double>(y, op->n_rows()));
  });
}

int ref_op_adjoint(const ref_op_desc* d, const double* y, double* x) {
  return guarded([&] {
    auto op = make_op(d);
    op->apply_adjoint(std::span<const double>(y, op->n_rows()), std::span<double>(x, op->n_cols()));
  });
}

double ref_diffusivity(int kind, double T, double t) { return diffusivity(make_spec(kind, T), t); }
double ref_r_value(int kind, double T, double t) { return r_value(make_spec(kind, T), t); }

int ref_assemble_m_dense(int dims, size_t nx, size_t ny, double h, const double* f, int kind,
                         double T, double eps, double* dense_out, double* eps_used) {
  return guarded([&] {
    const Grid grid = make_grid(dims, nx, ny, h);
    SparseSpd m = assemble_m(grid, std::span<const double>(f, grid.num_nodes()),
                             make_spec(kind, T), 0.0);
    const double e = eps >= 0.0 ? eps : auto_shift(m);
    m = m.with_shift(e);
    if (eps_used) *eps_used = e;
    if (dense_out) {
      const auto d = m.to_dense();
      std::memcpy(dense_out, d.data(), sizeof(double) * d.size());
    }
  });
}

// krylov_basis (krylov.cpp:700-754): md != null -> priorconditioned space; else with_m ->
// K^{A^T A + tau M} with M assembled at f (shift eps < 0: auto); else K^{A^T A}
int ref_krylov_basis(const ref_op_desc* od, const ref_map_desc* md, int with_m, int dims, size_t nx,
                     size_t ny, double h, const double* f, int kind, double T, double eps, double tau,
                     const double* g, int k, double* out, int* count, int* rank_exhausted) {
  return guarded([&] {
    auto a = make_op(od);
    KrylovBasis b;
    if (md) {
      MapHolder mh = make_map(md);
      b = krylov_basis(*a, &mh.get(), nullptr, tau, std::span<const double>(g, a->n_rows()), k);
    } else if (with_m) {
      const Grid grid = make_grid(dims, nx, ny, h);
      SparseSpd m = assemble_m(grid, std::span<const double>(f, grid.num_nodes()), make_spec(kind, T), 0.0);
      m = m.with_shift(eps >= 0.0 ? eps : auto_shift(m));
      b = krylov_basis(*a, nullptr, &m, tau, std::span<const double>(g, a->n_rows()), k);
    } else {
      b = krylov_basis(*a, nullptr, nullptr, tau, std::span<const double>(g, a->n_rows()), k);
    }
    *count = (int)b.vectors.size();
    *rank_exhausted = b.rank_exhausted ? 1 : 0;
    for (size_t j = 0; j < b.vectors.size(); ++j)
      std::copy(b.vectors[j].begin(), b.vectors[j].end(), out + j * a->n_cols());
  });
}

// one SpdMap::solve (spdsolve.hpp:15-22) of a freshly built map
int ref_map_solve(const ref_map_desc* md, const double* p, double* v) {
  return guarded([&] {
    MapHolder h = make_map(md);
    const SpdMap& m = h.get();
    m.solve(std::span<const double>(p, m.dimension()), std::span<double>(v, m.dimension()));
  });
}

int ref_m_multiply(int dims, size_t nx, size_t ny, double h, const double* f, int kind, double T,
                   double eps, const double* x, double* y) {
  return guarded([&] {
    const Grid grid = make_grid(dims, nx, ny, h);
    SparseSpd m = assemble_m(grid, std::span<const double>(f, grid.num_nodes()),
                             make_spec(kind, T), 0.0);
    m = m.with_shift(eps >= 0.0 ? eps : auto_shift(m));
    m.multiply(std::span<const double>(x, grid.num_nodes()), std::span<double>(y, grid.num_nodes()));
  });
}

double ref_penalty_functional(int dims, size_t nx, size_t ny, double h, const double* f,
                              int kind, double T) {
  const Grid grid = make_grid(dims, nx, ny, h);
  return penalty_functional(grid, std::span<const double>(f, grid.num_nodes()), make_spec(kind, T));
}

void ref_gauss_fill(uint64_t seed, size_t n, double stddev, double* out) {
  GaussianSampler s(seed);
  s.fill(std::span<double>(out, n), stddev);
}

// The reference's own solve_projected (krylov.cpp:631-678)
int ref_solve_projected(const double* alphas, size_t k, const double* betas, size_t nb, double beta1,
                        double tau, double* y) {
  return guarded([&] {
    BidiagEntries bd;
    bd.alphas.assign(alphas, alphas + k);
    bd.betas.assign(betas, betas + nb);
    const auto v = mlsqr::solve_projected(bd, beta1, tau);
    std::memcpy(y, v.data(), sizeof(double) * v.size());
  });
}

// The reference's own cg_normal (krylov.cpp:551-628): CG on (A^T A + tau M) f = A^T g, with M
// assembled at fM (diffusion.cpp:27-87) and shifted by eps (< 0: auto shift).
int ref_cg_normal(const ref_op_desc* od, int dims, size_t nx, size_t ny, double h, const double* fM,
                  int pen_kind, double T, double eps, double tau, const double* g, const ref_stop* stop,
                  double* f, ref_iter_rec* trace, ref_solve_info* info) {
  if (info) std::memset(info, 0, sizeof(*info));
  return guarded(
      [&] {
        auto op = make_op(od);
        const Grid grid = make_grid(dims, nx, ny, h);
        SparseSpd m = assemble_m(grid, std::span<const double>(fM, grid.num_nodes()),
                                 make_spec(pen_kind, T), 0.0);
        m = m.with_shift(eps >= 0.0 ? eps : auto_shift(m));
        const auto r = mlsqr::cg_normal(*op, m, tau, std::span<const double>(g, op->n_rows()), make_stop(stop));
        export_result(r, op->n_cols(), f, trace, nullptr, nullptr, nullptr, info);
      },
      info);
}

int ref_mlsqr(const ref_op_desc* od, const ref_map_desc* md, const double* g, double tau,
              const ref_stop* stop, int snapshots_on, double* f, ref_iter_rec* trace,
              double* alphas, double* betas, double* snapshots, ref_solve_info* info) {
  if (info) std::memset(info, 0, sizeof(*info));
  return guarded(
      [&] {
        auto op = make_op(od);
        MapHolder mh = make_map(md);
        SolveOptions opts;
        opts.record_snapshots = snapshots_on != 0;
        const auto r = mlsqr::mlsqr(*op, mh.get(), std::span<const double>(g, op->n_rows()),
                                    tau, make_stop(stop), opts);
        export_result(r, op->n_cols(), f, trace, alphas, betas, snapshots, info);
      },
      info);
}

// The reference's own mlsqr, timed: seconds spent in iterations warm+1 .. max_iters
// (init and the first `warm` iterations excluded).  Single thread, like the reference.
int ref_mlsqr_timed(const ref_op_desc* od, const ref_map_desc* md, const double* g, double tau,
                    const ref_stop* stop, int warm, double* f, double* seconds,
                    ref_solve_info* info) {
  if (info) std::memset(info, 0, sizeof(*info));
  return guarded(
      [&] {
        auto op = make_op(od);
        MapHolder mh = make_map(md);
        g_apply_calls = 0;
        g_apply_mark = warm + 1;
        const auto t0 = std::chrono::steady_clock::now();
        const auto r = mlsqr::mlsqr(*op, mh.get(), std::span<const double>(g, op->n_rows()), tau,
                                    make_stop(stop), SolveOptions{});
        const auto t1 = std::chrono::steady_clock::now();
        const auto start = g_apply_calls >= g_apply_mark ? g_mark_time : t0;
        *seconds = std::chrono::duration<double>(t1 - start).count();
        g_apply_mark = -1;
        export_result(r, op->n_cols(), f, nullptr, nullptr, nullptr, nullptr, info);
      },
      info);
}

int ref_lsqr(const ref_op_desc* od, const double* g, double tau, const ref_stop* stop,
             int snapshots_on, double* f, ref_iter_rec* trace, double* alphas, double* betas,
             double* snapshots, ref_solve_info* info) {
  if (info) std::memset(info, 0, sizeof(*info));
  return guarded(
      [&] {
        auto op = make_op(od);
        SolveOptions opts;
        opts.record_snapshots = snapshots_on != 0;
        const auto r = lsqr(*op, std::span<const double>(g, op->n_rows()), tau, make_stop(stop), opts);
        export_result(r, op->n_cols(), f, trace, alphas, betas, snapshots, info);
      },
      info);
}

typedef struct {
  double tau;
  int pen_kind;
  double T;
  ref_stop inner_stop;
  int inner_cap;
  double rel_decrease_threshold;
  int max_outer;
  int spd_mode;  // 0 cholesky 1 inner_cg
  int k_inner;
  double epsilon;  // < 0: auto
} ref_outer_cfg;

typedef struct {
  int k;
  int inner_iterations;
  int inner_stop;
  double penalty_value;
  double final_residual;
  double eps_used;
} ref_outer_step;

int ref_solve_nonlinear(const ref_op_desc* od, const double* g, int dims, size_t nx, size_t ny,
                        double h, const ref_outer_cfg* cfg, double* f_out,
                        ref_outer_step* steps, int* n_steps, int* stop_reason,
                        int* triggered_at, double* iterates) {
  return guarded([&] {
    auto op = make_op(od);
    const Grid grid = make_grid(dims, nx, ny, h);
    OuterConfig c;
    c.tau = cfg->tau;
    c.penalty = make_spec(cfg->pen_kind, cfg->T);
    c.inner_stop = make_stop(&cfg->inner_stop);
    c.inner_cap = cfg->inner_cap;
    c.rel_decrease_threshold = cfg->rel_decrease_threshold;
    c.max_outer = cfg->max_outer;
    c.spd_mode = cfg->spd_mode == 0 ? SpdSolverMode::direct_cholesky : SpdSolverMode::inner_cg;
    c.k_inner = cfg->k_inner;
    if (cfg->epsilon >= 0.0) c.epsilon = cfg->epsilon;
    c.keep_iterates = iterates != nullptr;
    const auto rep = solve_nonlinear(*op, std::span<const double>(g, op->n_rows()), grid, c);
    std::memcpy(f_out, rep.solution.data(), sizeof(double) * rep.solution.size());
    *n_steps = static_cast<int>(rep.steps.size());
    *stop_reason = rep.stop_reason == OuterStopReason::stagnation ? 0 : 1;
    *triggered_at = rep.triggered_at;
    for (size_t k = 0; k < rep.steps.size(); ++k) {
      const auto& s = rep.steps[k];
      steps[k] = {s.k, s.inner_iterations, reason_code(s.inner_stop), s.penalty_value,
                  s.final_residual, 0.0};
      if (iterates)
        std::memcpy(iterates + k * grid.num_nodes(), s.solution.data(),
                    sizeof(double) * grid.num_nodes());
    }
  });
}

}  // extern "C"
