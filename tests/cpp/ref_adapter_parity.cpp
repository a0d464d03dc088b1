// tests/cpp/ref_adapter_parity.cpp -- "parity mode" of the drop-in boundary.
//
// The UNMODIFIED reference mlsqr() (compiled from /root/reference/proj/src
// into oracle/_ref) drives the B200 blur through the C++ adapter
// mlsqr_b200::GpuLinearOperator (include/mlsqr_b200.hpp), with the
// reference's own envelope-Cholesky SpdSolver as M^{-1}.  With the
// reference's scalar BLAS-1 backend selected, the result must equal the
// all-CPU reference run bit for bit (the GPU blur sums each output in the
// reference's order).  Also checks the exception contract across the
// boundary and gpu_mlsqr() (throughput mode) against the reference loop.
//
// Built by `make -C oracle adapter` into oracle/_ref/ref_adapter_parity;
// run by tests/test_gpu_reference_adapter.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <vector>

#include "mlsqr/diffusion.hpp"
#include "mlsqr/kernels.hpp"
#include "mlsqr/krylov.hpp"
#include "mlsqr/linop.hpp"
#include "mlsqr/problems.hpp"
#include "mlsqr/spdsolve.hpp"
#include "mlsqr_b200.hpp"

using namespace mlsqr;

static int failures = 0;
#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++failures;                                                  \
    }                                                              \
  } while (0)

int main() {
  kernels::select(kernels::Backend::scalar);
  mlsqr_b200::Context ctx(0);

  // 2D deblur 48x48 with the reference operator's own taps (6 sigma radius)
  const std::size_t nx = 48;
  const double sigma = 0.04;
  const auto bundle = make_deblur2d(nx, nx, sigma, 0.01, Phantom2D::default_phantom(), 17);
  const auto& cpu_op = *bundle.op;
  GaussianConvolution1D k1(nx, sigma, 1.0);
  auto gpu_op = mlsqr_b200::GpuLinearOperator::blur(ctx, 2, nx, nx, 1, k1.taps());

  // operator parity
  const auto y_cpu = cpu_op.apply(bundle.f_true);
  const auto y_gpu = gpu_op.apply(bundle.f_true);
  EXPECT(y_cpu == y_gpu);

  // reference mlsqr with the reference's Cholesky M^-1 at the truth
  SparseSpd m = assemble_m(bundle.grid, bundle.f_true, PenaltySpec::tv_smoothed(0.05), 0.0);
  m = m.with_shift(1.0);
  const SpdSolver chol = SpdSolver::factorize(m);
  const auto stop = StoppingConfig::max_iterations(25);
  const auto r_cpu = mlsqr::mlsqr(cpu_op, chol, bundle.g, 1e-2, stop);
  const auto r_gpu = mlsqr::mlsqr(gpu_op, chol, bundle.g, 1e-2, stop);
  EXPECT(r_cpu.solution == r_gpu.solution);
  EXPECT(r_cpu.bidiag.alphas == r_gpu.bidiag.alphas);
  EXPECT(r_cpu.bidiag.betas == r_gpu.bidiag.betas);

  // exception contract across the C-ABI (linop.cpp:15-20 -> DimensionError)
  bool threw = false;
  try {
    std::vector<double> bad(nx * nx - 1), out(nx * nx);
    gpu_op.apply(bad, out);
  } catch (const DimensionError&) {
    threw = true;
  }
  EXPECT(threw);

  // throughput mode: device-resident mlsqr with the B200 V-cycle vs the reference loop
  // driving the same V-cycle through the SpdMap adapter (host round trips per call)
  auto vc = mlsqr_b200::GpuSpdMap::vcycle(ctx, 2, nx, nx, 1, 1.0 / nx, 3);
  vc.update(bundle.f_true, MLSQR_PEN_TV, 0.05);
  const auto r_dev = mlsqr_b200::gpu_mlsqr(gpu_op, vc, bundle.g, 1e-2, stop);
  const auto r_mix = mlsqr::mlsqr(gpu_op, vc, bundle.g, 1e-2, stop);
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < r_dev.solution.size(); ++i) {
    num += (r_dev.solution[i] - r_mix.solution[i]) * (r_dev.solution[i] - r_mix.solution[i]);
    den += r_mix.solution[i] * r_mix.solution[i];
  }
  const double relf = std::sqrt(num / den);
  double worst_a = 0.0;
  for (std::size_t i = 0; i < r_dev.bidiag.alphas.size(); ++i)
    worst_a = std::fmax(worst_a, std::fabs(r_dev.bidiag.alphas[i] - r_mix.bidiag.alphas[i]) / r_mix.bidiag.alphas[i]);
  std::printf("device-resident vs reference loop (V-cycle M^-1): rel f %.3e, max rel alpha %.3e\n", relf, worst_a);
  EXPECT(r_dev.iterations == r_mix.iterations);
  // canonical tree reductions vs the reference's sequential dots: rounding-level
  EXPECT(worst_a < 1e-9);
  EXPECT(relf < 1e-6);

  // multi-tau: the library's solve_projected equals the reference's bit for bit, and the
  // device basis re-expands to the device solve
  for (double tau : {0.0, 1e-3, 1e-2, 0.5}) {
    const auto y_ref = mlsqr::solve_projected(r_cpu.bidiag, r_cpu.bidiag.betas[0], tau);
    EXPECT(mlsqr_b200::gpu_solve_projected(r_cpu.bidiag, r_cpu.bidiag.betas[0], tau) == y_ref);
  }
  SolveOptions so;
  so.store_basis = true;
  const auto r_basis = mlsqr_b200::gpu_mlsqr(gpu_op, vc, bundle.g, 1e-2, stop, so);
  EXPECT(r_basis.solution == r_dev.solution);
  EXPECT(r_basis.bidiag.basis.size() == r_basis.bidiag.alphas.size());
  EXPECT(r_basis.bidiag.left_basis.size() == r_basis.bidiag.alphas.size() + 1);
  {
    const auto y = mlsqr_b200::gpu_solve_projected(r_basis.bidiag, r_basis.bidiag.betas[0], 1e-2);
    const auto f = mlsqr::reconstruct_from_basis(r_basis.bidiag, y);
    double n2 = 0.0, d2 = 0.0;
    for (std::size_t i = 0; i < f.size(); ++i) {
      n2 += (f[i] - r_basis.solution[i]) * (f[i] - r_basis.solution[i]);
      d2 += r_basis.solution[i] * r_basis.solution[i];
    }
    std::printf("stored-basis re-solve: rel %.3e\n", std::sqrt(n2 / d2));
    EXPECT(std::sqrt(n2 / d2) < 1e-8);
  }

  // cg_normal: device vs the reference's own cg_normal with the same M (assembled at the
  // truth with the V-cycle's shift); canonical vs sequential reductions -> rounding level
  {
    const double eps = vc.update(bundle.f_true, MLSQR_PEN_TV, 0.05);
    SparseSpd m2 = assemble_m(bundle.grid, bundle.f_true, PenaltySpec::tv_smoothed(0.05), 0.0).with_shift(eps);
    const auto st10 = StoppingConfig::max_iterations(10);
    const auto c_ref = mlsqr::cg_normal(cpu_op, m2, 1e-2, bundle.g, st10);
    const auto c_dev = mlsqr_b200::gpu_cg_normal(gpu_op, &vc, 1e-2, bundle.g, st10);
    double n2 = 0.0, d2 = 0.0;
    for (std::size_t i = 0; i < c_ref.solution.size(); ++i) {
      n2 += (c_dev.solution[i] - c_ref.solution[i]) * (c_dev.solution[i] - c_ref.solution[i]);
      d2 += c_ref.solution[i] * c_ref.solution[i];
    }
    std::printf("cg_normal device vs reference: rel f %.3e\n", std::sqrt(n2 / d2));
    EXPECT(c_dev.iterations == c_ref.iterations);
    EXPECT(std::sqrt(n2 / d2) < 1e-9);
  }

  // both seams on the B200 inside the UNMODIFIED reference loop: the GPU blur as A and the
  // GPU envelope Cholesky (SpdSolver::factorize on the device) as M^-1 -- bit for bit the all-CPU
  // reference (PM-log: no hypot in the diffusivity, so the device M is the reference's M exactly)
  {
    auto holder = mlsqr_b200::GpuSpdMap::vcycle(ctx, 2, nx, nx, 1, 1.0 / nx, 1);
    holder.update(bundle.f_true, MLSQR_PEN_PM_LOG, 0.05, 1.0);
    const auto gchol = mlsqr_b200::GpuSpdMap::cholesky(holder);
    const SparseSpd mp = assemble_m(bundle.grid, bundle.f_true, PenaltySpec::perona_malik_log(0.05), 0.0).with_shift(1.0);
    const SpdSolver cchol = SpdSolver::factorize(mp);
    const auto r_ref = mlsqr::mlsqr(cpu_op, cchol, bundle.g, 1e-2, stop);
    const auto r_both = mlsqr::mlsqr(gpu_op, gchol, bundle.g, 1e-2, stop);
    std::printf("reference mlsqr, GPU blur + GPU Cholesky vs all-CPU: %s\n",
                r_both.solution == r_ref.solution ? "bit-identical" : "DIFFERENT");
    EXPECT(r_both.solution == r_ref.solution);
    EXPECT(r_both.bidiag.alphas == r_ref.bidiag.alphas);
    // the inner-CG mode runs too (canonical dots inside the map: rounding-level agreement)
    const auto gcg = mlsqr_b200::GpuSpdMap::inner_cg(holder, 60);
    const auto r_cg = mlsqr::mlsqr(gpu_op, gcg, bundle.g, 1e-2, StoppingConfig::max_iterations(5));
    EXPECT(r_cg.iterations == 5);
    // SolveOptions::record_snapshots through the device loop
    SolveOptions rs;
    rs.record_snapshots = true;
    const auto r_snap = mlsqr_b200::gpu_mlsqr(gpu_op, vc, bundle.g, 1e-2, stop, rs);
    EXPECT(r_snap.trace.snapshots.size() == static_cast<std::size_t>(r_snap.iterations));
    EXPECT(!r_snap.trace.snapshots.empty() && r_snap.trace.snapshots.back() == r_snap.solution);
    // FactorizationError crosses the boundary as the reference's exception
    bool fthrew = false;
    auto bad = mlsqr_b200::GpuSpdMap::vcycle(ctx, 1, 8, 1, 1, 1.0 / 8, 1);
    try {
      std::vector<double> negc(8, -1.0);
      mlsqr_b200::check(mlsqr_vcycle_set_coefficients(bad.handle(), negc.data(), nullptr, nullptr, 0.0, MLSQR_HOST));
      const auto never = mlsqr_b200::GpuSpdMap::cholesky(bad);
    } catch (const FactorizationError& e) {
      fthrew = e.pivot_row() == 0;
    }
    EXPECT(fthrew);
  }

  // BreakdownError(iteration) with iteration > 0 crosses the boundary with the iteration the
  // reference reports (krylov.cpp:401-406): a map that is the identity for its first 6 calls and
  // -I afterwards, once as a reference SpdMap and once as a device-loop host plug-in
  {
    struct LateFlip final : SpdMap {
      std::size_t n;
      mutable int calls = 0;
      explicit LateFlip(std::size_t n_) : n(n_) {}
      std::size_t dimension() const override { return n; }
      using SpdMap::solve;
      void solve(std::span<const double> p, std::span<double> v) const override {
        const double s = calls++ < 6 ? 1.0 : -1.0;
        for (std::size_t i = 0; i < n; ++i) v[i] = s * p[i];
      }
    };
    LateFlip cpu_flip(nx * nx), dev_flip(nx * nx);
    auto fn = [](void* user, const double* p, double* v) -> int {
      auto* m = static_cast<LateFlip*>(user);
      m->solve(std::span<const double>(p, m->n), std::span<double>(v, m->n));
      return 0;
    };
    auto gflip = mlsqr_b200::GpuSpdMap::callback(ctx, nx * nx, fn, &dev_flip);
    int it_ref = -1, it_dev = -1;
    try {
      (void)mlsqr::mlsqr(cpu_op, cpu_flip, bundle.g, 1e-2, stop);
    } catch (const BreakdownError& e) {
      it_ref = e.iteration();
    }
    try {
      (void)mlsqr_b200::gpu_mlsqr(gpu_op, gflip, bundle.g, 1e-2, stop);
    } catch (const BreakdownError& e) {
      it_dev = e.iteration();
    }
    std::printf("late breakdown: reference iteration %d, device loop iteration %d\n", it_ref, it_dev);
    EXPECT(it_ref > 0);
    EXPECT(it_dev == it_ref);
  }

  // a non-square grid: the reference operator's two factors on the device, bit for bit
  {
    const SeparableGaussianBlur2D ref2(40, 24, 0.04);
    GaussianConvolution1D kx(40, 0.04, 1.0), ky(24, 0.04, 1.0);
    auto g2 = mlsqr_b200::GpuLinearOperator::blur2d_axes(ctx, 40, 24, kx.taps(), ky.taps());
    std::vector<double> xin(40 * 24);
    for (std::size_t i = 0; i < xin.size(); ++i) xin[i] = std::sin(0.37 * static_cast<double>(i));
    EXPECT(g2.apply(xin) == ref2.apply(xin));
  }

  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
