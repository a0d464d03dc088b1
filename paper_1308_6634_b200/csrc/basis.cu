// basis.cu -- krylov_basis (krylov.hpp:133-145, krylov.cpp:700-754): the first k orthonormalized
// basis vectors of one of the three Krylov spaces the reference's runner dumps as basis_###.csv
// (runner.cpp:245-275):
//   msolver == m == null : K^{A^T A}            seeded by A^T g
//   m != null            : K^{A^T A + tau M}    seeded by A^T g
//   msolver != null      : K^{M^-1 A^T A}       seeded by M^-1 A^T g
// Gram-Schmidt with one reorthogonalization pass, every dot a canonical segment tree, every
// update the reference's axpy / scal element formula.  Host-driven: one scalar read-back per
// vector for the rank test (analysis output, not the hot path).
#include "internal.cuh"
#include "vec.cuh"

namespace mlsqr_b200 {

namespace {

// y += a x with a = sign * *s (device scalar): axpy (kernels_scalar.cpp:13-15)
__global__ void kb_axpy_kernel(const double* __restrict__ s, double sign, const double* __restrict__ x,
                               double* __restrict__ y, size_t n) {
  const double a = sign < 0.0 ? -*s : *s;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}

// y += a x, host scalar
__global__ void kb_axpy_h_kernel(double a, const double* __restrict__ x, double* __restrict__ y, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}

// out = t * (1 / after): scal (kernels_scalar.cpp:21-23)
__global__ void kb_scal_kernel(double a, const double* __restrict__ t, double* __restrict__ out, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = t[i] * a;
}

}  // namespace

int krylov_basis(Op* op, Pc* msolver, VCycle* m, double tau, const double* g, int k, double* vecs,
                 int* rank_exhausted) {
  Ctx* c = op->ctx;
  require(!(msolver && m), MLSQR_EINVAL, "pass the preconditioner solver or the regularizer matrix, not both");
  require(k >= 1, MLSQR_EINVAL, "need at least one basis vector");
  require(!c->data_distributed(), MLSQR_EINVAL, "krylov_basis runs on a single-rank context");
  if (msolver) require(msolver->n == op->cols, MLSQR_EDIM, "preconditioner dimension does not match operator columns");
  const size_t n = op->cols;
  const RowShape S = op->sol_shape;
  const size_t J = S.segments();
  DevBuf<double> t(n), scratch(n), rows(op->rows), seg(J), scr(reduce_scratch_size(J) + J), sc(2);
  const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)c->sm_count * 8);
  auto dot_to = [&](const double* x, const double* y, double* out) {
    seg_dot(c, x, y, S, seg.p, nullptr);
    reduce_segments(c, seg.p, J, scr.p, out, nullptr);
  };
  auto nrm2 = [&](const double* x) {
    dot_to(x, x, sc.p);
    double v = 0.0;
    MLSQR_CUDA(cudaMemcpyAsync(&v, sc.p, sizeof v, cudaMemcpyDeviceToHost, c->stream));
    MLSQR_CUDA(cudaStreamSynchronize(c->stream));
    return std::sqrt(v);
  };
  auto precond = [&]() {  // t <- M^{-1} t (krylov.cpp:713-716, 734-737)
    if (!msolver) return;
    msolver->solve(t.p, scratch.p, nullptr, nullptr, S);
    MLSQR_CUDA(cudaMemcpyAsync(t.p, scratch.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  };

  *rank_exhausted = 0;
  op->adjoint(g, t.p, Epi{});
  precond();
  const double seed_norm = nrm2(t.p);
  if (seed_norm == 0.0) {
    *rank_exhausted = 1;
    return 0;
  }
  int count = 0;
  for (int j = 0; j < k; ++j) {
    if (j > 0) {
      const double* prev = vecs + (size_t)(count - 1) * n;
      op->apply(prev, rows.p, Epi{});
      op->adjoint(rows.p, t.p, Epi{});
      if (m && tau > 0.0) {
        vcycle_m_apply(m, prev, scratch.p);
        kb_axpy_h_kernel<<<blocks, 256, 0, c->stream>>>(tau, scratch.p, t.p, n);
        c->count();
      }
      precond();
    }
    const double before = nrm2(t.p);
    for (int pass = 0; pass < 2; ++pass) {  // Gram-Schmidt with reorthogonalization
      for (int q = 0; q < count; ++q) {
        const double* qv = vecs + (size_t)q * n;
        dot_to(qv, t.p, sc.p + 1);
        kb_axpy_kernel<<<blocks, 256, 0, c->stream>>>(sc.p + 1, -1.0, qv, t.p, n);
        c->count();
      }
    }
    const double after = nrm2(t.p);
    if (after <= 1e-12 * std::max(before, seed_norm)) {
      *rank_exhausted = 1;
      break;
    }
    kb_scal_kernel<<<blocks, 256, 0, c->stream>>>(1.0 / after, t.p, vecs + (size_t)count * n, n);
    c->count();
    ++count;
  }
  c->check_launch();
  MLSQR_CUDA(cudaStreamSynchronize(c->stream));
  return count;
}

}  // namespace mlsqr_b200
