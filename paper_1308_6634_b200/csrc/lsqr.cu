// lsqr.cu -- the device-resident priorconditioned LSQR loop (mlsqr,
// krylov.cpp:335-440) and its M = I reduction (lsqr, krylov.cpp:256-333).
//
// Every scalar of the reference loop lives in device memory (DevState); the
// LsqrRecurrence (krylov.cpp:24-108), finish_iteration (krylov.cpp:131-180)
// and evaluate_stopping (krylov.cpp:240-254) run in one device thread after
// each canonical reduction, so an iteration never waits on the host and the
// whole iteration is one replayable CUDA graph.  Vectors are stored
// UNSCALED (u_s, p_s, v_s) with their 1/beta, 1/alpha factors kept on the
// device; every consumer multiplies on load, which reproduces the
// reference's scal() results bit-for-bit while saving a full pass each.
//
// Per iteration (gates skip work once stopped / on clean breakdown):
//   K_A   u_s <- A(v_s*sv) - alpha (u_s*su)     + |u|^2 segments   (krylov.cpp:389-391)
//   F_b   beta = sqrt(.), su = 1/beta
//   K_B   p_s <- A^T(u_s*su) - beta (p_s*sv)    + |p|^2 segments   (krylov.cpp:395-398)
//   F_p   p != 0 ?
//   MG    v_s <- M^{-1} p_s                     + v.p segments     (krylov.cpp:399-400)
//   F_a   alpha' = sqrt(v.p), LsqrRecurrence::advance               (krylov.cpp:401-415)
//   K_U   f += phi/rho w; w <- v - theta/rho w; q <- p - theta/rho q + w.q segments
//   [K_R  |g - A f| when S4 needs the exact residual (krylov.cpp:142-144)]
//   F_i   trace row + stopping                                        (krylov.cpp:131-180)
#include <cstdlib>

#include "internal.cuh"
#include "vec.cuh"

namespace mlsqr_b200 {

struct DevState {
  // LSQR scalars
  double alpha, beta, sv, su, neg_alpha, neg_beta, sc, neg_dc, wnorm2, alpha_next;
  double minus_one;
  // reduction outputs
  double red_u, red_p, red_vp, red_wq, red_res;
  // LsqrRecurrence (krylov.cpp:101-117)
  double tau, damp, alpha_cur, phibar, rhobar, bnorm, rnorm, arnorm, anorm2, ddnorm, res2, cs2,
      sn2, z, xxnorm, xnorm;
  // flags: 0 active, 1 beta > 0, 2 p != 0 (run M^-1), 3 no breakdown (update w, q)
  int flags[4];
  int iter, iterations, stop_reason, error, error_iter, n_alphas, n_betas, breakdown;
  int n_left;  // left basis vectors stored (store_basis)
};

// vector with a zero guard zone on both sides (operator ghost planes when z-sharded)
struct GVec {
  DevBuf<double> raw;
  double* p = nullptr;
  void alloc(size_t n, size_t g, cudaStream_t s) {
    raw.alloc(n + 2 * g);
    if (g) MLSQR_CUDA(cudaMemsetAsync(raw.p, 0, sizeof(double) * raw.n, s));
    p = raw.p + g;
  }
};

struct Workspace {
  Ctx* ctx;
  size_t rows, cols, guard;
  RowShape data, sol;
  int max_iters;
  GVec u, p, v;  // blur inputs (u for A^T, v -- or p in lsqr mode -- for A)
  DevBuf<double> w, q, tmp_rows;
  DevBuf<double> seg_u, seg_p, seg_vp, seg_wq, seg_res, scratch, gathered;
  DevBuf<DevState> st;
  DevBuf<mlsqr_iter_rec> trace;
  DevBuf<double> alphas, betas;
  DevBuf<double> g;  // device copy of host data
  DevBuf<double> f;
  // the instantiated iteration graph of the last solve on this workspace: the next solve captures
  // its iteration again and UPDATES this executable (new pointers and scalars, same topology)
  // instead of instantiating a new one
  cudaGraphExec_t ge = nullptr;
  ~Workspace() {
    if (ge) cudaGraphExecDestroy(ge);
  }
};

Workspace* workspace_new(Ctx* c, size_t rows, size_t cols, RowShape data, RowShape sol,
                         int max_iters, size_t guard) {
  auto* w = new Workspace();
  w->ctx = c;
  w->rows = rows;
  w->cols = cols;
  w->guard = guard;
  w->data = data;
  w->sol = sol;
  w->max_iters = max_iters;
  w->u.alloc(rows, guard, c->stream);
  w->p.alloc(cols, guard, c->stream);
  w->v.alloc(cols, guard, c->stream);
  w->w.alloc(cols);
  w->q.alloc(cols);
  w->seg_u.alloc(data.segments());
  w->seg_res.alloc(data.segments());
  w->seg_p.alloc(sol.segments());
  w->seg_vp.alloc(sol.segments());
  w->seg_wq.alloc(sol.segments());
  const size_t J = data.segments() > sol.segments() ? data.segments() : sol.segments();
  const size_t G = dist_gather_size(c, J);
  w->scratch.alloc(reduce_scratch_size(G > J ? G : J) + J);
  w->gathered.alloc(G > 0 ? G : 1);
  w->st.alloc(1);
  w->trace.alloc((size_t)max_iters);
  w->alphas.alloc((size_t)max_iters + 1);
  w->betas.alloc((size_t)max_iters + 2);
  return w;
}

void workspace_free(Workspace* w) { delete w; }

// ---------------------------------------------------------------------------
// device scalar logic
// ---------------------------------------------------------------------------
__device__ __forceinline__ void rec_init(DevState& s, double alpha1, double beta1, double tau) {
  s.tau = tau;
  s.damp = sqrt(tau);
  s.alpha_cur = alpha1;
  s.phibar = beta1;
  s.rhobar = alpha1;
  s.bnorm = beta1;
  s.rnorm = beta1;
  s.arnorm = 0.0;
  s.anorm2 = 0.0;
  s.ddnorm = 0.0;
  s.res2 = 0.0;
  s.cs2 = -1.0;
  s.sn2 = 0.0;
  s.z = 0.0;
  s.xxnorm = 0.0;
  s.xnorm = 0.0;
}

// LsqrRecurrence::advance (krylov.cpp:40-81), same operation order; hypot -> dhypot
__device__ __forceinline__ void rec_advance(DevState& r, double beta_next, double alpha_next,
                                            double wnorm2, double* sol_coeff, double* dir_coeff) {
  r.anorm2 = r.anorm2 + (r.alpha_cur * r.alpha_cur + beta_next * beta_next + r.tau);
  double rhobar1 = r.rhobar, psi = 0.0;
  if (r.damp > 0.0) {
    rhobar1 = dhypot(r.rhobar, r.damp);
    const double cs1 = r.rhobar / rhobar1;
    psi = (r.damp / rhobar1) * r.phibar;
    r.phibar = cs1 * r.phibar;
  }
  const double rho = dhypot(rhobar1, beta_next);
  const double cs = rhobar1 / rho;
  const double sn = beta_next / rho;
  const double theta = sn * alpha_next;
  r.rhobar = -cs * alpha_next;
  const double phi = cs * r.phibar;
  r.phibar = sn * r.phibar;
  r.ddnorm = r.ddnorm + wnorm2 / (rho * rho);
  const double delta = r.sn2 * rho;
  const double gambar = -r.cs2 * rho;
  const double rhs = phi - delta * r.z;
  const double zbar = rhs / gambar;
  r.xnorm = sqrt(r.xxnorm + zbar * zbar);
  const double gamma = dhypot(gambar, theta);
  r.cs2 = gambar / gamma;
  r.sn2 = theta / gamma;
  r.z = rhs / gamma;
  r.xxnorm = r.xxnorm + r.z * r.z;
  r.res2 = r.res2 + psi * psi;
  r.rnorm = sqrt(r.phibar * r.phibar + r.res2);
  r.arnorm = alpha_next * fabs(sn * phi);
  r.alpha_cur = alpha_next;
  *sol_coeff = phi / rho;
  *dir_coeff = theta / rho;
}

__global__ void init_state_kernel(DevState* s, double tau) {
  DevState z = {};
  z.tau = tau;
  z.minus_one = -1.0;
  z.flags[0] = 1;
  z.stop_reason = MLSQR_STOP_MAX_ITERS;
  *s = z;
}

// FI1: beta1 = |g|
__global__ void fin_beta1_kernel(DevState* s, double* betas) {
  s->beta = sqrt(s->red_u);
  betas[0] = s->beta;
  s->n_betas = 1;
  if (s->beta == 0.0) {
    s->stop_reason = MLSQR_STOP_BREAKDOWN;
    s->flags[0] = 0;
    return;
  }
  s->su = 1.0 / s->beta;
}

// FI2: |A^T u| == 0 -> clean breakdown before the first iteration
__global__ void fin_p0_kernel(DevState* s) {
  if (!s->flags[0]) return;
  if (sqrt(s->red_p) == 0.0) {
    s->stop_reason = MLSQR_STOP_BREAKDOWN;
    s->flags[0] = 0;
  }
}

// FI3: alpha1 = sqrt(v.p) > 0 else BreakdownError(0)
__global__ void fin_alpha1_kernel(DevState* s, double* alphas) {
  if (!s->flags[0]) return;
  const double s0 = s->red_vp;
  if (!(s0 > 0.0)) {
    s->error = 1;
    s->error_iter = 0;
    s->flags[0] = 0;
    return;
  }
  const double alpha1 = sqrt(s0);
  s->sv = 1.0 / alpha1;
  alphas[0] = alpha1;
  s->n_alphas = 1;
  rec_init(*s, alpha1, s->beta, s->tau);
  s->alpha = alpha1;
  s->neg_alpha = -alpha1;
  s->iter = 1;
}

__global__ void fin_wq0_kernel(DevState* s) {
  if (!s->flags[0]) return;
  s->wnorm2 = s->red_wq;
}

// F_b (krylov.cpp:391-395)
__device__ __forceinline__ void fin_beta_dev(DevState* s) {
  if (!s->flags[0]) return;
  const double beta = sqrt(s->red_u);
  s->beta = beta;
  s->flags[1] = beta > 0.0 ? 1 : 0;
  s->flags[2] = 0;
  if (beta > 0.0) {
    s->su = 1.0 / beta;
    s->neg_beta = -beta;
  }
}

// F_p (krylov.cpp:398)
__device__ __forceinline__ void fin_p_dev(DevState* s) {
  if (!s->flags[0] || !s->flags[1]) return;
  s->flags[2] = sqrt(s->red_p) > 0.0 ? 1 : 0;
}

// SolveOptions::store_basis (krylov.cpp:375-377, 421-423): row n_alphas-1 of the basis is the
// scaled vtilde (v * (1/alpha), the reference's scal), written when this step produced an alpha
__global__ void basis_kernel(const DevState* __restrict__ s, const double* __restrict__ v,
                             double* __restrict__ basis, size_t n, int in_loop) {
  if (!s->flags[0] || (in_loop && !s->flags[3])) return;
  double* row = basis + (size_t)(s->n_alphas - 1) * n;
  const double sv = s->sv;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    row[i] = v[i] * sv;
}

// left basis (krylov.cpp:375-377, 421-425): u_1 once alpha_1 exists, then u_{i+1} whenever
// beta_{i+1} > 0 -- the scaled u (u * (1/beta), the reference's scal)
__global__ void left_basis_kernel(DevState* __restrict__ s, const double* __restrict__ u,
                                  double* __restrict__ basis, size_t m, int in_loop) {
  if (!s->flags[0] || (in_loop && !s->flags[1])) return;
  const int row = in_loop ? s->n_left : 0;
  double* out = basis + (size_t)row * m;
  const double su = s->su;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x)
    out[i] = u[i] * su;
}
// SolveOptions::record_snapshots (krylov.cpp:159-161): f after this iteration's update, row
// iter-1, for every iteration that records a trace row (active at its start)
__global__ void snapshot_kernel(const DevState* __restrict__ s, const double* __restrict__ f,
                                double* __restrict__ snaps, size_t n) {
  if (!s->flags[0]) return;
  double* row = snaps + (size_t)(s->iter - 1) * n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    row[i] = f[i];
}
__global__ void left_count_kernel(DevState* s, int in_loop) {
  if (!s->flags[0] || (in_loop && !s->flags[1])) return;
  s->n_left = in_loop ? s->n_left + 1 : 1;
}

// F_a (krylov.cpp:399-431)
__device__ __forceinline__ void fin_alpha_dev(DevState* s, double* alphas, double* betas) {
  if (!s->flags[0]) return;
  double alpha_next = 0.0;
  int breakdown = 1;
  if (s->flags[2]) {
    const double sv = s->red_vp;
    if (!(sv > 0.0)) {
      s->error = 1;
      s->error_iter = s->iter;
      s->flags[0] = s->flags[1] = s->flags[2] = s->flags[3] = 0;
      return;
    }
    alpha_next = sqrt(sv);
    s->sv = 1.0 / alpha_next;
    breakdown = 0;
  }
  double sc, dc;
  rec_advance(*s, s->beta, alpha_next, s->wnorm2, &sc, &dc);
  s->sc = sc;
  s->neg_dc = -dc;
  s->breakdown = breakdown;
  s->flags[3] = breakdown ? 0 : 1;
  if (!breakdown) alphas[s->n_alphas++] = alpha_next;
  betas[s->n_betas++] = s->beta;
  s->alpha_next = alpha_next;
  s->alpha = alpha_next;
  s->neg_alpha = -alpha_next;
}

// F_i: finish_iteration (krylov.cpp:131-180) + evaluate_stopping (krylov.cpp:240-254)
__device__ __forceinline__ void fin_iter_dev(DevState* s, mlsqr_iter_rec* trace, mlsqr_stop stop) {
  if (!s->flags[0]) return;
  if (s->flags[3]) s->wnorm2 = s->red_wq;
  const int iter = s->iter;
  mlsqr_iter_rec row;
  row.iteration = iter;
  row.res_damped = s->rnorm;
  if (s->tau == 0.0) {
    row.res_data = s->rnorm;
    row.res_data_exact = 1;
  } else if (stop.use_s4) {
    row.res_data = sqrt(s->red_res);
    row.res_data_exact = 1;
  } else {
    const double est = s->rnorm * s->rnorm - s->tau * s->xnorm * s->xnorm;
    row.res_data = sqrt(est > 0.0 ? est : 0.0);
    row.res_data_exact = 0;
  }
  const double anorm = sqrt(s->anorm2);
  const double acond = anorm * sqrt(s->ddnorm);
  const double den = anorm * s->rnorm;
  row.s2_value = den > 0.0 ? s->arnorm / den : 0.0;
  row.anorm_est = anorm;
  row.cond_est = acond;
  row.xnorm_est = s->xnorm;
  row.alpha = s->alpha_next;
  row.beta = s->beta;
  trace[iter - 1] = row;
  s->iterations = iter;
  int fired = -1;
  if (stop.use_s4 && row.res_data <= stop.eta * stop.delta) fired = MLSQR_STOP_S4;
  else if (stop.use_s1 && s->rnorm <= stop.btol * s->bnorm + stop.atol * anorm * s->xnorm) fired = MLSQR_STOP_S1;
  else if (stop.use_s2 && (s->arnorm <= stop.atol * den || den == 0.0)) fired = MLSQR_STOP_S2;
  else if (stop.use_s3 && stop.conlim > 0.0 && acond >= stop.conlim) fired = MLSQR_STOP_S3;
  else if (iter >= stop.max_iters) fired = MLSQR_STOP_MAX_ITERS;
  if (fired < 0 && s->breakdown) fired = MLSQR_STOP_BREAKDOWN;
  if (fired >= 0) {
    s->stop_reason = fired;
    s->flags[0] = s->flags[1] = s->flags[2] = s->flags[3] = 0;
  }
  s->iter = iter + 1;
}

// K_U (krylov.cpp:416-419): f += sc w; [w <- v*sv - dc w; q <- p*sv - dc q; w.q partials]
__global__ void __launch_bounds__(256) update_kernel(const DevState* __restrict__ s,
                                                     double* __restrict__ f,
                                                     double* __restrict__ w,
                                                     double* __restrict__ q,
                                                     const double* __restrict__ v,
                                                     const double* __restrict__ p, size_t len,
                                                     size_t rows, double* __restrict__ seg) {
  if (!s->flags[0]) return;
  // rows in a block-stride loop (the scalars and the column index are loaded / formed once)
  const size_t xi = (size_t)blockIdx.x * 32 + threadIdx.x;
  const bool upd = s->flags[3] != 0;
  const double sc = s->sc, sv = s->sv, ndc = s->neg_dc;
  const size_t chunks = (len + 31) / 32, rstep = (size_t)gridDim.y * blockDim.y;
#pragma unroll 4
  for (size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += rstep) {
    double prod = 0.0;
    if (xi < len) {
      const size_t i = row * len + xi;
      const double wi = w[i];
      f[i] = f[i] + sc * wi;
      if (upd) {
        const double wn = v[i] * sv + ndc * wi;
        const double qn = p[i] * sv + ndc * q[i];
        w[i] = wn;
        q[i] = qn;
        prod = wn * qn;
      }
    }
    if (upd) {
      const double t = tree32(prod);
      if (threadIdx.x == 0) seg[row * chunks + blockIdx.x] = t;
    }
  }
}

// init: w = v*sv, q = p*sv, f = 0, w.q partials
__global__ void init_wq_kernel(const DevState* __restrict__ s, double* __restrict__ f,
                               double* __restrict__ w, double* __restrict__ q,
                               const double* __restrict__ v, const double* __restrict__ p,
                               size_t len, size_t rows, double* __restrict__ seg) {
  if (!s->flags[0]) return;
  for (size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += (size_t)gridDim.y * blockDim.y) {
    const size_t xi = (size_t)blockIdx.x * 32 + threadIdx.x;
    double prod = 0.0;
    if (xi < len) {
      const size_t i = row * len + xi;
      const double sv = s->sv;
      const double wn = v[i] * sv, qn = p[i] * sv;
      w[i] = wn;
      q[i] = qn;
      f[i] = 0.0;
      prod = wn * qn;
    }
    const double t = tree32(prod);
    if (threadIdx.x == 0) seg[row * ((len + 31) / 32) + blockIdx.x] = t;
  }
}

__global__ void zero_kernel(double* __restrict__ f, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = 0.0;
}

void validate_stop(const mlsqr_stop& s) {  // StoppingConfig::validate (krylov.cpp:219-226)
  require(s.max_iters >= 1, MLSQR_EINVAL, "max_iters must be at least 1");
  require(!s.use_s4 || s.eta > 1.0, MLSQR_EINVAL, "discrepancy stopping needs a safety factor eta > 1");
  require(!s.use_s4 || s.delta >= 0.0, MLSQR_EINVAL, "noise level delta must be >= 0");
  require(s.atol >= 0.0 && s.btol >= 0.0, MLSQR_EINVAL, "tolerances must be >= 0");
}


// the same scalar steps as epilogues of the final reduction pass (vec.cuh reduce_final_fin)
struct FinBeta {
  DevState* s;
  __device__ void operator()() const { fin_beta_dev(s); }
};
struct FinP {
  DevState* s;
  __device__ void operator()() const { fin_p_dev(s); }
};
struct FinAlpha {
  DevState* s;
  double *alphas, *betas;
  __device__ void operator()() const { fin_alpha_dev(s, alphas, betas); }
};
struct FinIter {
  DevState* s;
  mlsqr_iter_rec* trace;
  mlsqr_stop stop;
  __device__ void operator()() const { fin_iter_dev(s, trace, stop); }
};

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
namespace {

struct Runner {
  Op* op;
  Pc* pc;  // nullptr: plain lsqr (v aliases p)
  Workspace* ws;
  double tau;
  mlsqr_stop stop;
  DevState* st;
  Ctx* c;
  double* basis = nullptr;  // [(max_iters + 1) x cols] when the basis is stored
  double* lbasis = nullptr; // [(max_iters + 1) x rows] left basis
  double* snaps = nullptr;  // [max_iters x cols] f snapshots (record_snapshots)
  void store_snapshot() {
    if (!snaps) return;
    const size_t n = op->cols;
    const unsigned g = (unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    snapshot_kernel<<<g, 256, 0, c->stream>>>(st, ws->f.p, snaps, n);
    c->count();
  }
  void store_left(int in_loop) {
    if (!lbasis) return;
    const size_t m = op->rows;
    const unsigned g = (unsigned)((m + 255) / 256 < 4096 ? (m + 255) / 256 : 4096);
    left_basis_kernel<<<g, 256, 0, c->stream>>>(st, ws->u.p, lbasis, m, in_loop);
    left_count_kernel<<<1, 1, 0, c->stream>>>(st, in_loop);
    c->count(2);
  }

  const int* flag(int k) const { return &st->flags[k]; }
  void store_basis(int in_loop) {
    if (!basis) return;
    const size_t n = op->cols;
    const unsigned g = (unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    basis_kernel<<<g, 256, 0, c->stream>>>(st, vbuf(), basis, n, in_loop);
    c->count();
  }
  const int* gate_active() const { return flag(0); }

  // data-space vectors are distributed under z slabs and row shards; solution-space ones
  // only under z slabs (row shards replicate the solution space)
  void reduce(double* seg, size_t nseg, double* out, const int* gate, bool data) {
    reduce_segments_dist(c, seg, nseg, ws->scratch.p, ws->gathered.p, out, gate,
                         data ? c->data_distributed() : c->sharded());
  }

  // reduce, then the scalar step F in the same final one-warp pass; z slabs / row shards first
  // allgather the block-aligned tree partials (every rank finishes the canonical tree identically)
  template <class F>
  void reduce_fin(double* seg, size_t nseg, double* out, const int* gate, bool data, F fin) {
    const bool dist = (data ? c->data_distributed() : c->sharded()) && c->data_distributed();
    if (!dist) {
      reduce_segments_fin(c, seg, nseg, ws->scratch.p, out, gate, fin);
      return;
    }
    size_t J = 0;
    const double* g = dist_gather_partials(c, seg, nseg, ws->scratch.p, ws->gathered.p, gate, &J);
    reduce_segments_fin(c, g, J, ws->scratch.p, out, gate, fin);
  }

  double* vbuf() const { return pc ? ws->v.p : ws->p.p; }

  // z slabs, mlsqr mode: K_A's input vtilde is final after the V-cycle, so its R ghost planes
  // travel on the side stream while fin_alpha, K_U and the w.q reduction run on the main
  // stream (SURVEY §8e overlap); joined before the iteration ends (graph-capture safe).
  bool vghost_async() const { return pc && c->sharded() && op->halo_planes_needed() > 0; }
  void fork_vghost() {
    if (!vghost_async()) return;
    cudaStream_t s = c->side_stream();
    MLSQR_CUDA(cudaEventRecord(c->ev_fork, c->stream));
    MLSQR_CUDA(cudaStreamWaitEvent(s, c->ev_fork, 0));
    const size_t plane = op->plane_size();
    halo_planes(c, ws->v.p, plane, (long)(op->cols / plane), op->halo_planes_needed(), s);
    MLSQR_CUDA(cudaEventRecord(c->ev_join, s));
  }
  void join_vghost() {
    if (vghost_async()) MLSQR_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  }

  // M^{-1} p and the <v, p> partials; in the loop the reduction's final pass also runs F_a
  void precond(const int* gate, bool fin_alpha = false) {
    if (pc) {
      pc->in_guarded = ws->guard > 0;
      pc->solve(ws->p.p, ws->v.p, ws->seg_vp.p, gate, ws->sol);
      pc->in_guarded = false;
    } else {
      seg_dot(c, ws->p.p, ws->p.p, ws->sol, ws->seg_vp.p, gate);
    }
    if (!fin_alpha) {
      reduce(ws->seg_vp.p, ws->sol.segments(), &st->red_vp, gate, false);
      return;
    }
    reduce_fin(ws->seg_vp.p, ws->sol.segments(), &st->red_vp, gate, false, FinAlpha{st, ws->alphas.p, ws->betas.p});
  }

  void init(const double* g) {
    // f = 0 before anything can stop the solve (SolveResult::solution.assign(n, 0.0))
    MLSQR_CUDA(cudaMemsetAsync(ws->f.p, 0, sizeof(double) * ws->cols, c->stream));
    init_state_kernel<<<1, 1, 0, c->stream>>>(st, tau);
    // u_s = g, |g|^2
    Epi e;
    e.seg = ws->seg_u.p;
    axpby_epi(c, g, ws->u.p, ws->data, e);
    reduce(ws->seg_u.p, ws->data.segments(), &st->red_u, nullptr, true);
    fin_beta1_kernel<<<1, 1, 0, c->stream>>>(st, ws->betas.p);
    // p_s = A^T (u_s * su), |p|^2
    Epi eb;
    eb.sx = &st->su;
    eb.seg = ws->seg_p.p;
    eb.gate = gate_active();
    eb.in_guarded = true;
    op->adjoint(ws->u.p, ws->p.p, eb);
    reduce(ws->seg_p.p, ws->sol.segments(), &st->red_p, gate_active(), false);
    fin_p0_kernel<<<1, 1, 0, c->stream>>>(st);
    precond(gate_active());
    fork_vghost();
    fin_alpha1_kernel<<<1, 1, 0, c->stream>>>(st, ws->alphas.p);
    store_basis(0);
    store_left(0);
    dim3 blk(32, 8), grd((unsigned)ws->sol.chunks(), row_grid(ws->sol.rows));
    init_wq_kernel<<<grd, blk, 0, c->stream>>>(st, ws->f.p, ws->w.p, ws->q.p, vbuf(), ws->p.p,
                                               ws->sol.len, ws->sol.rows, ws->seg_wq.p);
    reduce(ws->seg_wq.p, ws->sol.segments(), &st->red_wq, gate_active(), false);
    fin_wq0_kernel<<<1, 1, 0, c->stream>>>(st);
    join_vghost();
    c->count(6);
    c->check_launch();
  }

  void iteration(const double* g) {
    TimedRegion it(c, MLSQR_TCLASS_ITER);
    // K_A: u_s <- A(v_s*sv) + (-alpha)(u_s*su)
    Epi ea;
    ea.sx = &st->sv;
    ea.old = ws->u.p;
    ea.so = &st->su;
    ea.coef = &st->neg_alpha;
    ea.seg = ws->seg_u.p;
    ea.gate = gate_active();
    ea.in_guarded = true;
    ea.ghosts_ready = vghost_async();
    op->apply(vbuf(), ws->u.p, ea);
    reduce_fin(ws->seg_u.p, ws->data.segments(), &st->red_u, gate_active(), true, FinBeta{st});
    store_left(1);
    // K_B: p_s <- A^T(u_s*su) + (-beta)(p_s*sv)
    Epi eb;
    eb.sx = &st->su;
    eb.old = ws->p.p;
    eb.so = &st->sv;
    eb.coef = &st->neg_beta;
    eb.seg = ws->seg_p.p;
    eb.gate = flag(1);
    eb.in_guarded = true;
    op->adjoint(ws->u.p, ws->p.p, eb);
    reduce_fin(ws->seg_p.p, ws->sol.segments(), &st->red_p, flag(1), false, FinP{st});
    // M^{-1}
    precond(flag(2), true);  // + F_a
    fork_vghost();
    store_basis(1);
    // K_U
    {
      TimedRegion tr(c, MLSQR_TCLASS_UPDATE);
      dim3 blk(32, 8), grd((unsigned)ws->sol.chunks(), row_grid(ws->sol.rows));
      // four rows per thread (the row loop keeps every warp one row segment)
      const dim3 grd4(grd.x, (unsigned)((ws->sol.rows + 31) / 32));
      update_kernel<<<grd4, blk, 0, c->stream>>>(st, ws->f.p, ws->w.p, ws->q.p, vbuf(), ws->p.p,
                                                 ws->sol.len, ws->sol.rows, ws->seg_wq.p);
    }
    store_snapshot();  // f is final after K_U; F_i (which advances iter / flags) runs last
    if (tau != 0.0 && stop.use_s4) {
      reduce(ws->seg_wq.p, ws->sol.segments(), &st->red_wq, flag(3), false);
      // exact data residual |g - A f| (krylov.cpp:142-144): (A f - g)^2 partials
      Epi er;
      er.old = g;
      er.coef = &st->minus_one;
      er.seg = ws->seg_res.p;
      er.gate = gate_active();
      op->apply(ws->f.p, ws->tmp_rows.p, er);
      reduce_fin(ws->seg_res.p, ws->data.segments(), &st->red_res, gate_active(), true,
                 FinIter{st, ws->trace.p, stop});
    } else {
      reduce_fin(ws->seg_wq.p, ws->sol.segments(), &st->red_wq, flag(3), false, FinIter{st, ws->trace.p, stop});
    }
    join_vghost();
    c->count(1);  // update_kernel
    c->check_launch();
  }
};

}  // namespace

int solve_mlsqr(Op* op, Pc* pc, const double* g_dev, double tau, const mlsqr_stop& stop,
                double* f_dev, mlsqr_iter_rec* trace, double* alphas, double* betas,
                mlsqr_solve_info* info, Workspace* ws_in, bool use_graph, double* basis_dev,
                double* left_dev, double* snap_dev) {
  Ctx* c = op->ctx;
  validate_stop(stop);
  require(tau >= 0.0, MLSQR_EINVAL, "tau must be nonnegative");
  if (pc) require(pc->n == op->cols, MLSQR_EDIM, "preconditioner dimension does not match operator columns");
  if (pc && pc->row_len())
    require(pc->row_len() == op->sol_shape.len, MLSQR_EDIM,
            "operator solution-space rows (sol_row_len) must match the V-cycle grid x extent");
  Workspace* ws = ws_in;
  auto fits = [&](Workspace* w) {
    return w && w->rows == op->rows && w->cols == op->cols && w->max_iters >= stop.max_iters &&
           w->data.len == op->data_shape.len && w->sol.len == op->sol_shape.len &&
           w->guard >= op_guard(op);
  };
  if (!fits(ws)) {
    // reuse the context's cached workspace (no cudaMalloc per solve)
    ws = static_cast<Workspace*>(c->ws_cache);
    if (!fits(ws)) {
      if (ws) workspace_free(ws);
      c->ws_cache = nullptr;
      ws = workspace_new(c, op->rows, op->cols, op->data_shape, op->sol_shape, stop.max_iters, op_guard(op));
      c->ws_cache = ws;
      c->ws_free = [](void* p) { workspace_free(static_cast<Workspace*>(p)); };
    }
  }
  if (tau != 0.0 && stop.use_s4) ws->tmp_rows.ensure(op->rows);
  // f lives in the caller's buffer
  struct FGuard {
    Workspace* ws;
    double* saved;
    size_t n;
    ~FGuard() { ws->f.p = saved; ws->f.n = n; }
  } fg{ws, ws->f.p, ws->f.n};
  ws->f.p = f_dev;
  ws->f.n = op->cols;

  Runner r{op, pc, ws, tau, stop, ws->st.p, c, basis_dev, left_dev, snap_dev};
  const bool host_cb = pc && pc->host_callback();
  // MLSQR_NO_GRAPH=1 replays the same launches eagerly (bisects a capture failure on a new path)
  static const bool no_graph = [] {
    const char* e = getenv("MLSQR_NO_GRAPH");
    return e && e[0] && e[0] != '0';
  }();
  const bool graph = use_graph && !no_graph && !host_cb && !c->timing && (!c->comm || c->comm->capturable());
  r.init(g_dev);
  if (graph) {
    cudaGraph_t gr = nullptr;
    cudaGraphExec_t ge = nullptr;
    MLSQR_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const uint64_t before = c->launches;
    // iterations per graph replay: the graph holds `per` gated iterations (fewer replay gaps; the
    // largest of 5, 4, 2 that divides max_iters; MLSQR_GRAPH_ITERS overrides)
    static const int per_env = [] {
      const char* e = getenv("MLSQR_GRAPH_ITERS");
      return e ? atoi(e) : 0;
    }();
    int per = 1;
    for (int k : {5, 4, 2})
      if (per == 1 && stop.max_iters % k == 0) per = k;
    if (per_env >= 1) per = stop.max_iters % per_env == 0 ? per_env : 1;
    try {
      for (int k = 0; k < per; ++k) r.iteration(g_dev);
    } catch (...) {
      cudaStreamEndCapture(c->stream, &gr);
      if (gr) cudaGraphDestroy(gr);
      throw;
    }
    MLSQR_CUDA(cudaStreamEndCapture(c->stream, &gr));
    if (ws->ge) {
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(ws->ge, gr, &info) == cudaSuccess) {
        ge = ws->ge;
      } else {  // another topology (a different operator / map on this workspace): instantiate anew
        (void)cudaGetLastError();
        cudaGraphExecDestroy(ws->ge);
        ws->ge = nullptr;
      }
    }
    if (!ge) {
      MLSQR_CUDA(cudaGraphInstantiate(&ge, gr, 0));
      ws->ge = ge;
    }
    // every replay launches the captured kernels (gated ones exit at once)
    c->launches += (c->launches - before) * (uint64_t)(stop.max_iters / per - 1);
    for (int i = 0; i < stop.max_iters / per; ++i) MLSQR_CUDA(cudaGraphLaunch(ge, c->stream));
    MLSQR_CUDA(cudaStreamSynchronize(c->stream));
    cudaGraphDestroy(gr);
  } else {
    for (int i = 0; i < stop.max_iters; ++i) {
      if (host_cb) {
        // a host plug-in map must see every iteration's state: stop enqueueing once done
        int active = 0;
        MLSQR_CUDA(cudaMemcpyAsync(&active, &ws->st.p->flags[0], sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        MLSQR_CUDA(cudaStreamSynchronize(c->stream));
        if (!active) break;
      }
      r.iteration(g_dev);
    }
  }
  DevState hs;
  MLSQR_CUDA(cudaMemcpyAsync(&hs, ws->st.p, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  MLSQR_CUDA(cudaStreamSynchronize(c->stream));
  TimedRegion::collect(c);
  const int na = hs.n_alphas > hs.iterations ? hs.iterations : hs.n_alphas;  // trim_bidiag
  if (trace && hs.iterations > 0)
    MLSQR_CUDA(cudaMemcpy(trace, ws->trace.p, sizeof(mlsqr_iter_rec) * hs.iterations, cudaMemcpyDeviceToHost));
  if (alphas && hs.n_alphas > 0)
    MLSQR_CUDA(cudaMemcpy(alphas, ws->alphas.p, sizeof(double) * hs.n_alphas, cudaMemcpyDeviceToHost));
  if (betas && hs.n_betas > 0)
    MLSQR_CUDA(cudaMemcpy(betas, ws->betas.p, sizeof(double) * hs.n_betas, cudaMemcpyDeviceToHost));
  if (info) {
    info->iterations = hs.iterations;
    info->stop_reason = hs.stop_reason;
    info->n_alphas = hs.error ? hs.n_alphas : na;
    info->n_betas = hs.n_betas;
    info->breakdown_iteration = hs.error_iter;
    info->n_left_basis = left_dev ? hs.n_left : 0;
  }
  if (hs.error) {
    throw Error(MLSQR_EBREAKDOWN,
                "nonpositive M-weighted square norm at " +
                    (hs.error_iter == 0 ? std::string("initialization")
                                        : "iteration " + std::to_string(hs.error_iter)) +
                    "; the preconditioner map is not symmetric positive definite",
                hs.error_iter);
  }
  return MLSQR_OK;
}

}  // namespace mlsqr_b200
