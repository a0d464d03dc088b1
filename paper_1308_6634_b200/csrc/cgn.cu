// cgn.cu -- cg_normal (krylov.cpp:551-628): conjugate gradients on the normal equation
// (A^T A + tau M) f = A^T g, the reference's unpriorconditioned baseline, on the same
// operators (blur / dense) and the same matrix-free M (the V-cycle's level-0 edge operator,
// CSR row order of sparse.cpp:65-74) as the mlsqr path.
//
// Every inner product is the canonical segment tree (vec.cu), every vector update is the
// reference's axpy / xpby element formula, so the iterates, the trace and the stopping
// decisions equal the oracle's device-order cg_normal bit for bit.  The loop is host-driven:
// one 5-scalar read-back per iteration (the baseline is not the hot path).
#include "internal.cuh"
#include "vec.cuh"

namespace mlsqr_b200 {

namespace {

// q = q + tau * mx  (axpy, krylov.cpp:583); then <d, q> segment partials
__global__ void cgn_q_kernel(double* __restrict__ q, const double* __restrict__ mx, double tau,
                             const double* __restrict__ d, size_t len, size_t rows, size_t chunks,
                             double* __restrict__ seg) {
  for (size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += (size_t)gridDim.y * blockDim.y) {  // gridDim.y <= 65535
    const size_t xi = (size_t)blockIdx.x * 32 + threadIdx.x;
    double v = 0.0;
    if (xi < len) {
      const size_t i = row * len + xi;
      double qi = q[i];
      if (mx) {
        qi = qi + tau * mx[i];
        q[i] = qi;
      }
      v = d[i] * qi;
    }
    v = tree32(v);
    if (threadIdx.x == 0) seg[row * chunks + blockIdx.x] = v;
  }
}

// gamma = rho / curv (krylov.cpp:591), on the device so the update needs no host round trip
__global__ void cgn_gamma_kernel(const double* rho, const double* curv, double* gamma) {
  const double g = *rho / *curv;
  gamma[0] = g;
  gamma[1] = -g;
}

// x += gamma d; r += (-gamma) q (krylov.cpp:592-593); then <r, r> segment partials
__global__ void cgn_update_kernel(double* __restrict__ x, double* __restrict__ r,
                                  const double* __restrict__ d, const double* __restrict__ q,
                                  const double* __restrict__ gamma, size_t len, size_t rows,
                                  size_t chunks, double* __restrict__ seg) {
  for (size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += (size_t)gridDim.y * blockDim.y) {  // gridDim.y <= 65535
    const size_t xi = (size_t)blockIdx.x * 32 + threadIdx.x;
    double v = 0.0;
    if (xi < len) {
      const size_t i = row * len + xi;
      const double gm = gamma[0], ng = gamma[1];
      x[i] = x[i] + gm * d[i];
      const double ri = r[i] + ng * q[i];
      r[i] = ri;
      v = ri * ri;
    }
    v = tree32(v);
    if (threadIdx.x == 0) seg[row * chunks + blockIdx.x] = v;
  }
}

// d = r + beta d  (xpby, krylov.cpp:625)
__global__ void cgn_xpby_kernel(const double* __restrict__ r, double beta, double* __restrict__ d, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = r[i] + beta * d[i];
}

}  // namespace

void solve_cg_normal(Op* op, VCycle* m, const double* g, double tau, const mlsqr_stop& stop,
                     double* x, mlsqr_iter_rec* trace, mlsqr_solve_info* info, double* snap) {
  Ctx* c = op->ctx;
  validate_stop(stop);
  require(tau >= 0.0, MLSQR_EINVAL, "tau must be nonnegative");
  require(!c->data_distributed(), MLSQR_EINVAL, "cg_normal runs on a single-rank context");
  require(tau == 0.0 || m != nullptr, MLSQR_EINVAL, "cg_normal with tau > 0 needs the M of a V-cycle map");
  const size_t n = op->cols, rows = op->rows;
  const RowShape S = op->sol_shape, D = op->data_shape;
  DevBuf<double> r(n), d(n), q(n), mx(n), tmp(rows);
  const size_t JS = S.segments(), JD = D.segments(), J = JS > JD ? JS : JD;
  DevBuf<double> seg(J), scratch(reduce_scratch_size(J) + J);
  // device scalars: rho, curv, rho_next, res2, qf, xx, gamma, -gamma, -1
  DevBuf<double> sc(9);
  double* rho_d = sc.p;
  double* curv_d = sc.p + 1;
  double* rhon_d = sc.p + 2;
  double* res2_d = sc.p + 3;
  double* qf_d = sc.p + 4;
  double* xx_d = sc.p + 5;
  double* gam_d = sc.p + 6;
  double* m1_d = sc.p + 8;
  const double minus_one = -1.0;
  MLSQR_CUDA(cudaMemcpyAsync(m1_d, &minus_one, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  MLSQR_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c->stream));
  MLSQR_CUDA(cudaMemsetAsync(qf_d, 0, sizeof(double), c->stream));
  const dim3 blk(32, 8), grdS((unsigned)S.chunks(), row_grid(S.rows));
  auto reduce = [&](double* out, size_t nseg) { reduce_segments(c, seg.p, nseg, scratch.p, out, nullptr); };

  // b = A^T g; r = b; d = r (krylov.cpp:564-566)
  op->adjoint(g, r.p, Epi{});
  MLSQR_CUDA(cudaMemcpyAsync(d.p, r.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  seg_dot(c, r.p, r.p, S, seg.p, nullptr);
  reduce(rho_d, JS);
  double rho = 0.0;
  MLSQR_CUDA(cudaMemcpyAsync(&rho, rho_d, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  MLSQR_CUDA(cudaStreamSynchronize(c->stream));
  const double nres0 = std::sqrt(rho);
  mlsqr_solve_info inf{};
  inf.stop_reason = MLSQR_STOP_MAX_ITERS;
  if (nres0 == 0.0) {
    inf.stop_reason = MLSQR_STOP_BREAKDOWN;
    if (info) *info = inf;
    return;
  }
  const double nan = std::nan("");
  for (int iter = 1; iter <= stop.max_iters; ++iter) {
    // q = (A^T A + tau M) d, curvature d.q
    op->apply(d.p, tmp.p, Epi{});
    op->adjoint(tmp.p, q.p, Epi{});
    if (tau > 0.0) vcycle_m_apply(m, d.p, mx.p);
    cgn_q_kernel<<<grdS, blk, 0, c->stream>>>(q.p, tau > 0.0 ? mx.p : nullptr, tau, d.p, S.len, S.rows, S.chunks(),
                                              seg.p);
    reduce(curv_d, JS);
    cgn_gamma_kernel<<<1, 1, 0, c->stream>>>(rho_d, curv_d, gam_d);
    cgn_update_kernel<<<grdS, blk, 0, c->stream>>>(x, r.p, d.p, q.p, gam_d, S.len, S.rows, S.chunks(), seg.p);
    reduce(rhon_d, JS);
    // exact data residual |g - A x| (krylov.cpp:110-123): (A x - g)^2 partials
    Epi er;
    er.old = g;
    er.coef = m1_d;
    er.seg = seg.p;
    op->apply(x, tmp.p, er);
    reduce(res2_d, JD);
    if (tau > 0.0) {  // SparseSpd::quadratic_form = x . (M x) (sparse.cpp:82-93)
      vcycle_m_apply(m, x, mx.p);
      seg_dot(c, x, mx.p, S, seg.p, nullptr);
      reduce(qf_d, JS);
    }
    seg_dot(c, x, x, S, seg.p, nullptr);
    reduce(xx_d, JS);
    c->count(3);
    c->check_launch();
    double h[6];
    MLSQR_CUDA(cudaMemcpyAsync(h, curv_d, sizeof(double) * 5, cudaMemcpyDeviceToHost, c->stream));
    MLSQR_CUDA(cudaStreamSynchronize(c->stream));
    const double curv = h[0], rho_next = h[1], res2 = h[2], qf = h[3], xx = h[4];
    if (!(curv > 0.0))
      throw Error(MLSQR_EBREAKDOWN,
                  "nonpositive curvature at iteration " + std::to_string(iter) +
                      "; the normal-equation matrix is not positive definite",
                  iter);
    mlsqr_iter_rec row{};
    row.iteration = iter;
    row.res_data = std::sqrt(res2);
    row.res_data_exact = 1;
    row.res_damped = tau > 0.0 ? std::sqrt(row.res_data * row.res_data + tau * qf) : row.res_data;
    row.s2_value = std::sqrt(rho_next) / nres0;
    row.anorm_est = nan;
    row.cond_est = nan;
    row.xnorm_est = std::sqrt(xx);
    if (trace) trace[iter - 1] = row;
    if (snap)  // SolveOptions::record_snapshots (krylov.cpp:608)
      MLSQR_CUDA(cudaMemcpyAsync(snap + (size_t)(iter - 1) * n, x, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                 c->stream));
    inf.iterations = iter;
    if (stop.use_s4 && row.res_data <= stop.eta * stop.delta) {
      inf.stop_reason = MLSQR_STOP_S4;
      break;
    }
    if (stop.use_s2 && row.s2_value <= stop.atol) {
      inf.stop_reason = MLSQR_STOP_S2;
      break;
    }
    if (rho_next == 0.0) {
      inf.stop_reason = MLSQR_STOP_BREAKDOWN;
      break;
    }
    if (iter >= stop.max_iters) break;
    cgn_xpby_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(r.p, rho_next / rho, d.p, n);
    c->count();
    MLSQR_CUDA(cudaMemcpyAsync(rho_d, rhon_d, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    rho = rho_next;
  }
  if (info) *info = inf;
}

}  // namespace mlsqr_b200
