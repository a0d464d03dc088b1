// spdmaps.cu -- the reference's two SpdSolver modes (spdsolve.hpp:42-70, spdsolve.cpp:22-137)
// as device SpdMaps over the edge-based M (+ shift) held by a V-cycle map's level 0:
//
//  - EnvelopeCholMap: SpdSolver::factorize (spdsolve.cpp:22-75) + solve_cholesky (:101-117).
//    Envelope (skyline) storage in natural order, row i spanning [first_col(i), i].  The
//    factorization and both substitutions run in the reference's exact operation order: every
//    dot product is the scalar backend's sequential `acc += x*y` from 0, subtracted once
//    (`sum -= dot(...)`, spdsolve.cpp:62), every axpy is `y += a*x` (kernels_scalar.cpp:13-15).
//    So the factor and each solve are bit-identical to the reference's scalar backend.  The
//    recurrences are sequential by construction; this map is the direct solver of the
//    reference's small configs (deconv1d 512, deblur2d 64^2), not the hot path -- the V-cycle is.
//  - InnerCgMap: SpdSolver::inner_cg / solve_cg (spdsolve.cpp:77-85, 119-137): exactly k_inner
//    CG iterations from v = 0 with the early exits on rho == 0 or curvature == 0, on a snapshot
//    of M.  Dots are canonical segment trees, updates the reference's axpy / xpby
//    element formulas; fully device-resident (device scalars + a device "active" flag), so an
//    mlsqr loop using it is still captured as one CUDA graph.
#include "internal.cuh"
#include "vec.cuh"

namespace mlsqr_b200 {

// level-0 view of a V-cycle map (vcycle.cu)
void vcycle_level0(VCycle* v, int* dims, int* nx, int* ny, int* nz, double* h, const double** cx,
                   const double** cy, const double** cz, const double** eps);

namespace {

struct Grid3 {
  int nx, ny, nz;  // inactive axes have extent 1
  __host__ __device__ size_t n() const { return (size_t)nx * ny * nz; }
};

// smallest column of row i of the assembled M (sparse.cpp row order): z-, y-, x- neighbour
__host__ __device__ inline size_t first_col(const Grid3& g, size_t i) {
  const size_t nxy = (size_t)g.nx * g.ny;
  const size_t z = i / nxy, y = (i / g.nx) % g.ny, x = i % g.nx;
  if (z > 0) return i - nxy;
  if (y > 0) return i - g.nx;
  if (x > 0) return i - 1;
  return i;
}

// diagonal of M in the reference's edge enumeration order (x edges, then y, then z; the same
// order as vcycle.cu diag_at), then the shift (SparseSpd::with_shift, sparse.cpp:125-134)
__device__ inline double m_diag(const Grid3& g, const double* cx, const double* cy, const double* cz,
                                size_t i) {
  const size_t nxy = (size_t)g.nx * g.ny;
  const size_t z = i / nxy, y = (i / g.nx) % g.ny, x = i % g.nx;
  double d = 0.0;
  if (x > 0) d = d + cx[i - 1];
  if (x + 1 < (size_t)g.nx) d = d + cx[i];
  if (cy) {
    if (y > 0) d = d + cy[i - g.nx];
    if (y + 1 < (size_t)g.ny) d = d + cy[i];
  }
  if (cz) {
    if (z > 0) d = d + cz[i - nxy];
    if (z + 1 < (size_t)g.nz) d = d + cz[i];
  }
  return d;
}

// envelope element (i, j), j in [i - b, i]: env[i * (b + 1) + b + (j - i)]
struct Env {
  double* e;
  size_t b;
  __device__ double& at(size_t i, size_t j) const { return e[i * (b + 1) + b + j - i]; }
};

// lower triangle of M + eps I into the envelope (spdsolve.cpp:40-48)
__global__ void env_fill_kernel(Env E, Grid3 g, const double* __restrict__ cx,
                                const double* __restrict__ cy, const double* __restrict__ cz,
                                const double* __restrict__ eps) {
  const size_t n = g.n(), nxy = (size_t)g.nx * g.ny;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    for (size_t k = 0; k <= E.b; ++k) E.e[i * (E.b + 1) + k] = 0.0;
    const size_t z = i / nxy, y = (i / g.nx) % g.ny, x = i % g.nx;
    if (cz && z > 0) E.at(i, i - nxy) = -cz[i - nxy];
    if (cy && y > 0) E.at(i, i - g.nx) = -cy[i - g.nx];
    if (x > 0) E.at(i, i - 1) = -cx[i - 1];
    E.at(i, i) = m_diag(g, cx, cy, cz, i) + *eps;
  }
}

// in-place skyline Cholesky M = L L^T (spdsolve.cpp:51-73), one thread, reference order
__global__ void env_factor_kernel(Env E, Grid3 g, long long* bad_row) {
  const size_t n = g.n();
  for (size_t i = 0; i < n; ++i) {
    const size_t fi = first_col(g, i);
    for (size_t j = fi; j <= i; ++j) {
      const size_t fj = first_col(g, j);
      const size_t lo = fi > fj ? fi : fj;
      double sum = E.at(i, j);
      if (j > lo) {
        double acc = 0.0;  // kernels_scalar.cpp:7-11
        for (size_t k = lo; k < j; ++k) acc += E.at(i, k) * E.at(j, k);
        sum -= acc;
      }
      if (j < i) {
        E.at(i, j) = sum / E.at(j, j);
      } else {
        if (!(sum > 0.0)) {
          *bad_row = (long long)i;
          return;
        }
        E.at(i, i) = sqrt(sum);
      }
    }
  }
}

// solve_cholesky (spdsolve.cpp:101-117): L z = p by rows, then L^T v = z column-oriented
__global__ void env_solve_kernel(Env E, Grid3 g, const double* __restrict__ p, double* __restrict__ v,
                                 const int* gate) {
  if (gate && *gate == 0) return;
  const size_t n = g.n();
  for (size_t i = 0; i < n; ++i) {
    const size_t fi = first_col(g, i);
    double sum = p[i];
    if (i > fi) {
      double acc = 0.0;
      for (size_t k = fi; k < i; ++k) acc += E.at(i, k) * v[k];
      sum -= acc;
    }
    v[i] = sum / E.at(i, i);
  }
  for (size_t ii = n; ii-- > 0;) {
    const size_t fi = first_col(g, ii);
    const double vi = v[ii] / E.at(ii, ii);
    v[ii] = vi;
    const double a = -vi;
    for (size_t k = fi; k < ii; ++k) v[k] += a * E.at(ii, k);  // kernels_scalar.cpp:13-15
  }
}

class EnvelopeCholMap final : public Pc {
 public:
  EnvelopeCholMap(VCycle* src, long long* pivot_row) {
    int dims = 0, nx = 0, ny = 0, nz = 0;
    double h = 0.0;
    const double *cx, *cy, *cz, *eps;
    vcycle_level0(src, &dims, &nx, &ny, &nz, &h, &cx, &cy, &cz, &eps);
    ctx = vcycle_as_pc(src)->ctx;
    require(!ctx->data_distributed(), MLSQR_EINVAL, "the envelope Cholesky map runs on a single-rank context");
    g_ = Grid3{nx, ny, nz};
    n = g_.n();
    E_.b = dims >= 3 ? (size_t)nx * ny : dims >= 2 ? (size_t)nx : 1;
    const double bytes = (double)n * (double)(E_.b + 1) * 8.0;
    require(bytes <= 8e9, MLSQR_EINVAL,
            "envelope Cholesky of this grid needs " + std::to_string(bytes / 1e9) +
                " GB; use the V-cycle map for large grids");
    // the recurrences are sequential (the reference's order): ~n b^2 / 2 dependent steps on one thread
    const double steps = (double)n * (double)E_.b * (double)E_.b / 2.0;
    require(steps <= 2e9, MLSQR_EINVAL,
            "envelope Cholesky of this grid is ~" + std::to_string(steps / 1e9) +
                " G sequential steps on one device thread; use the inner-CG or V-cycle map");
    env_.alloc(n * (E_.b + 1));
    E_.e = env_.p;
    DevBuf<long long> bad(1);
    const long long minus1 = -1;
    MLSQR_CUDA(cudaMemcpyAsync(bad.p, &minus1, sizeof minus1, cudaMemcpyHostToDevice, ctx->stream));
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)ctx->sm_count * 8);
    env_fill_kernel<<<blocks, 256, 0, ctx->stream>>>(E_, g_, cx, cy, cz, eps);
    env_factor_kernel<<<1, 1, 0, ctx->stream>>>(E_, g_, bad.p);
    ctx->count(2);
    ctx->check_launch();
    long long row = -1;
    MLSQR_CUDA(cudaMemcpyAsync(&row, bad.p, sizeof row, cudaMemcpyDeviceToHost, ctx->stream));
    MLSQR_CUDA(cudaStreamSynchronize(ctx->stream));
    if (pivot_row) *pivot_row = row;
    if (row >= 0)  // FactorizationError (spdsolve.cpp:66-70)
      throw Error(MLSQR_EFACTOR,
                  "matrix is not positive definite: nonpositive pivot at row " + std::to_string(row),
                  (int)row);
  }
  size_t row_len() const override { return (size_t)g_.nx; }
  void solve(const double* p, double* v, double* seg, const int* gate, RowShape shape) override {
    env_solve_kernel<<<1, 1, 0, ctx->stream>>>(E_, g_, p, v, gate);
    ctx->count();
    ctx->check_launch();
    if (seg) seg_dot(ctx, v, p, shape, seg, gate);
  }

 private:
  Grid3 g_{};
  Env E_{};
  DevBuf<double> env_;
};

// ---------------------------------------------------------------------------
// inner CG (spdsolve.cpp:119-137)
// ---------------------------------------------------------------------------
struct CgScalars {  // device block
  double rho, curv, rho_next, gamma, ngamma, beta;
  int run, active;
};

// v = 0, r = p, d = p (spdsolve.cpp:122-124); partials of r.r; run/active <- gate
__global__ void cg_init_kernel(const double* __restrict__ p, double* __restrict__ v, double* __restrict__ r,
                               double* __restrict__ d, size_t len, size_t rows, size_t chunks,
                               double* __restrict__ seg, const int* gate, CgScalars* s) {
  const int on = gate ? *gate : 1;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0) {
    s->run = on;
    s->active = on;
  }
  if (!on) return;
  const size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y;
  if (row >= rows) return;
  const size_t xi = (size_t)blockIdx.x * 32 + threadIdx.x;
  double t = 0.0;
  if (xi < len) {
    const size_t i = row * len + xi;
    const double pi = p[i];
    v[i] = 0.0;
    r[i] = pi;
    d[i] = pi;
    t = pi * pi;
  }
  t = tree32(t);
  if (threadIdx.x == 0) seg[row * chunks + blockIdx.x] = t;
}

// `if (rho == 0.0) break;` (spdsolve.cpp:127)
__global__ void cg_check_rho_kernel(CgScalars* s) {
  if (s->active && s->rho == 0.0) s->active = 0;
}

// `if (curv == 0.0) break; gamma = rho / curv` (spdsolve.cpp:129-131)
__global__ void cg_gamma_kernel(CgScalars* s) {
  if (!s->active) return;
  if (s->curv == 0.0) {
    s->active = 0;
    return;
  }
  const double g = s->rho / s->curv;
  s->gamma = g;
  s->ngamma = -g;
}

// <d, q> partials
__global__ void cg_dq_kernel(const double* __restrict__ d, const double* __restrict__ q, size_t len,
                             size_t rows, size_t chunks, double* __restrict__ seg, const CgScalars* s) {
  if (!s->active) return;
  const size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y;
  if (row >= rows) return;
  const size_t xi = (size_t)blockIdx.x * 32 + threadIdx.x;
  double t = 0.0;
  if (xi < len) {
    const size_t i = row * len + xi;
    t = d[i] * q[i];
  }
  t = tree32(t);
  if (threadIdx.x == 0) seg[row * chunks + blockIdx.x] = t;
}

// v += gamma d; r += (-gamma) q (spdsolve.cpp:132-133); partials of r.r
__global__ void cg_update_kernel(double* __restrict__ v, double* __restrict__ r, const double* __restrict__ d,
                                 const double* __restrict__ q, size_t len, size_t rows, size_t chunks,
                                 double* __restrict__ seg, const CgScalars* s) {
  if (!s->active) return;
  const size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y;
  if (row >= rows) return;
  const size_t xi = (size_t)blockIdx.x * 32 + threadIdx.x;
  double t = 0.0;
  if (xi < len) {
    const size_t i = row * len + xi;
    v[i] += s->gamma * d[i];
    const double ri = r[i] + s->ngamma * q[i];
    r[i] = ri;
    t = ri * ri;
  }
  t = tree32(t);
  if (threadIdx.x == 0) seg[row * chunks + blockIdx.x] = t;
}

// d = r + (rho_next / rho) d; rho = rho_next (spdsolve.cpp:134-136)
__global__ void cg_beta_kernel(CgScalars* s) {
  if (!s->active) return;
  s->beta = s->rho_next / s->rho;
}
__global__ void cg_xpby_kernel(const double* __restrict__ r, double* __restrict__ d, size_t n, CgScalars* s) {
  if (!s->active) return;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = r[i] + s->beta * d[i];
}
__global__ void cg_roll_kernel(CgScalars* s) {
  if (s->active) s->rho = s->rho_next;
}

// out = v when the caller's gate was open; partials of out . p
__global__ void cg_out_kernel(const double* __restrict__ v, const double* __restrict__ p, double* __restrict__ out,
                              size_t len, size_t rows, size_t chunks, double* __restrict__ seg,
                              const CgScalars* s) {
  if (!s->run) return;
  const size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y;
  if (row >= rows) return;
  const size_t xi = (size_t)blockIdx.x * 32 + threadIdx.x;
  double t = 0.0;
  if (xi < len) {
    const size_t i = row * len + xi;
    const double vi = v[i];
    out[i] = vi;
    t = vi * p[i];
  }
  if (seg) {
    t = tree32(t);
    if (threadIdx.x == 0) seg[row * chunks + blockIdx.x] = t;
  }
}

class InnerCgMap final : public Pc {
 public:
  InnerCgMap(VCycle* src, int k) : k_(k) {
    require(k >= 1, MLSQR_EINVAL, "inner CG needs k_inner >= 1");
    int dims = 0, nx = 0, ny = 0, nz = 0;
    double h = 0.0;
    const double *cx, *cy, *cz, *eps;
    vcycle_level0(src, &dims, &nx, &ny, &nz, &h, &cx, &cy, &cz, &eps);
    ctx = vcycle_as_pc(src)->ctx;
    require(!ctx->data_distributed(), MLSQR_EINVAL, "the inner-CG map runs on a single-rank context");
    n = (size_t)nx * ny * nz;
    S_ = RowShape{(size_t)nx, n / (size_t)nx};
    // snapshot of M (the reference moves the matrix into the solver, spdsolve.cpp:77-85)
    m_ = make_vcycle(ctx, dims, (size_t)nx, (size_t)ny, (size_t)nz, h, 1, 1, 1, 1.0, 1);
    double e = 0.0;
    MLSQR_CUDA(cudaMemcpyAsync(&e, eps, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
    MLSQR_CUDA(cudaStreamSynchronize(ctx->stream));
    vcycle_set_coefficients(m_, cx, cy, cz, e);
    v_.alloc(n);
    r_.alloc(n);
    d_.alloc(n);
    q_.alloc(n);
    seg_.alloc(S_.segments());
    scr_.alloc(reduce_scratch_size(S_.segments()) + S_.segments());
    sc_.alloc(1);
    MLSQR_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  ~InnerCgMap() override { delete vcycle_as_pc(m_); }
  size_t row_len() const override { return S_.len; }
  void solve(const double* p, double* out, double* seg, const int* gate, RowShape shape) override {
    CgScalars* s = sc_.p;
    const int* act = &s->active;
    const dim3 blk(32, 8), grd((unsigned)S_.chunks(), (unsigned)((S_.rows + 7) / 8));
    const size_t J = S_.segments();
    cg_init_kernel<<<grd, blk, 0, ctx->stream>>>(p, v_.p, r_.p, d_.p, S_.len, S_.rows, S_.chunks(), seg_.p, gate, s);
    ctx->count();
    reduce_segments(ctx, seg_.p, J, scr_.p, &s->rho, act);
    for (int it = 0; it < k_; ++it) {
      cg_check_rho_kernel<<<1, 1, 0, ctx->stream>>>(s);
      vcycle_m_apply(m_, d_.p, q_.p);  // SparseSpd::multiply (sparse.cpp:65-74) + shift
      cg_dq_kernel<<<grd, blk, 0, ctx->stream>>>(d_.p, q_.p, S_.len, S_.rows, S_.chunks(), seg_.p, s);
      reduce_segments(ctx, seg_.p, J, scr_.p, &s->curv, act);
      cg_gamma_kernel<<<1, 1, 0, ctx->stream>>>(s);
      cg_update_kernel<<<grd, blk, 0, ctx->stream>>>(v_.p, r_.p, d_.p, q_.p, S_.len, S_.rows, S_.chunks(), seg_.p, s);
      reduce_segments(ctx, seg_.p, J, scr_.p, &s->rho_next, act);
      cg_beta_kernel<<<1, 1, 0, ctx->stream>>>(s);
      cg_xpby_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(r_.p, d_.p, n, s);
      cg_roll_kernel<<<1, 1, 0, ctx->stream>>>(s);
      ctx->count(7);
    }
    // the caller's partials follow its own row shape (the operator's solution space)
    const bool same = shape.len == S_.len;
    cg_out_kernel<<<grd, blk, 0, ctx->stream>>>(v_.p, p, out, S_.len, S_.rows, S_.chunks(),
                                                 same ? seg : nullptr, s);
    ctx->count();
    ctx->check_launch();
    if (seg && !same) seg_dot(ctx, out, p, shape, seg, gate);
  }

 private:
  int k_;
  RowShape S_{};
  VCycle* m_ = nullptr;
  DevBuf<double> v_, r_, d_, q_, seg_, scr_;
  DevBuf<CgScalars> sc_;
};

}  // namespace

Pc* make_chol_map(VCycle* src, long long* pivot_row) { return new EnvelopeCholMap(src, pivot_row); }
Pc* make_inner_cg_map(VCycle* src, int k_inner) { return new InnerCgMap(src, k_inner); }

}  // namespace mlsqr_b200
