// projected.cu -- solve_projected (krylov.hpp:124-127, krylov.cpp:631-678): one
// bidiagonalization serves every tau.  Minimises |[B_k; sqrt(tau) I] y - beta1 e1| for the
// lower-bidiagonal B_k (alphas on the diagonal, betas[1..k] below it) by Householder QR of
// the (2k+1) x k stacked matrix, in the reference's operation order (column norms and
// projections accumulated top-down, reflector head chosen away from cancellation, columns
// below the 1e-14 relative rank tolerance skipped and their coefficients left at 0), so the
// result is bit-identical to the reference's.  Host arithmetic: k is the iteration count.
#include <cmath>
#include <vector>

#include "internal.cuh"

namespace mlsqr_b200 {

std::vector<double> solve_projected(const double* alphas, size_t k, const double* betas, size_t nb,
                                    double beta1, double tau) {
  require(k > 0, MLSQR_EINVAL, "empty bidiagonalization");
  require(nb >= k + 1, MLSQR_EINVAL, "bidiagonalization needs k+1 betas for k alphas");
  require(tau >= 0.0, MLSQR_EINVAL, "tau must be nonnegative");
  const size_t m = 2 * k + 1;
  // column-major stacked matrix: column j holds alpha_j at row j, beta_{j+1} at row j+1 and
  // sqrt(tau) at row k+1+j
  std::vector<double> col(k * m, 0.0);
  auto at = [&](size_t r, size_t c) -> double& { return col[c * m + r]; };
  const double st = std::sqrt(tau);
  for (size_t j = 0; j < k; ++j) {
    at(j, j) = alphas[j];
    at(j + 1, j) = betas[j + 1];
    at(k + 1 + j, j) = st;
  }
  std::vector<double> rhs(m, 0.0);
  rhs[0] = beta1;
  double big = 0.0;
  for (double v : col) big = std::fmax(big, std::fabs(v));
  const double tol = big * 1e-14;

  std::vector<double> h(m);
  for (size_t j = 0; j < k; ++j) {
    double nn = 0.0;
    for (size_t r = j; r < m; ++r) nn += at(r, j) * at(r, j);
    const double nrm = std::sqrt(nn);
    if (nrm <= tol) continue;
    const double head = at(j, j);
    const double v0 = head + (head >= 0.0 ? 1.0 : -1.0) * nrm;
    h[0] = v0;  // reflector (v0, column j below the diagonal)
    for (size_t r = j + 1; r < m; ++r) h[r - j] = at(r, j);
    const double hh = nn - head * head + v0 * v0;
    auto reflect = [&](auto&& elem) {
      double pr = 0.0;
      for (size_t r = j; r < m; ++r) pr += h[r - j] * elem(r);
      const double cf = 2.0 * pr / hh;
      for (size_t r = j; r < m; ++r) elem(r) -= cf * h[r - j];
    };
    for (size_t c = j; c < k; ++c) reflect([&](size_t r) -> double& { return at(r, c); });
    reflect([&](size_t r) -> double& { return rhs[r]; });
  }
  std::vector<double> y(k, 0.0);
  for (size_t j = k; j-- > 0;) {
    double s = rhs[j];
    for (size_t c = j + 1; c < k; ++c) s -= at(j, c) * y[c];
    const double d = at(j, j);
    y[j] = std::fabs(d) <= tol ? 0.0 : s / d;
  }
  return y;
}

// reconstruct_from_basis (krylov.cpp:680-689): f = sum_j y_j vtilde_j, accumulated in j order
// like the reference's axpy sequence
__global__ void reconstruct_kernel(const double* __restrict__ basis, size_t n, const double* __restrict__ y,
                                   size_t ny, double* __restrict__ f) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (size_t j = 0; j < ny; ++j) acc = acc + y[j] * basis[j * n + i];
    f[i] = acc;
  }
}

void reconstruct_from_basis(Ctx* c, const double* basis, size_t n, const double* y, size_t ny, double* f) {
  const unsigned g = (unsigned)((n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192);
  reconstruct_kernel<<<g, 256, 0, c->stream>>>(basis, n, y, ny, f);
  c->count();
  c->check_launch();
}

}  // namespace mlsqr_b200
