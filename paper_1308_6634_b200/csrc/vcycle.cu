// vcycle.cu -- the priorconditioner M^{-1} as a multigrid V-cycle on the
// edge-based diffusion operator M = L_D^T L_D + eps I, plus the per-outer-step
// diffusivity update (SURVEY.md §2.1 K_D, K_H, K_S, K_R, K_P, K_alpha).
//
//  - K_D  edge_coeffs_kernel: c_e = c(|d_e|) w_e / h^2 per axis
//         (assemble_m / for_each_edge, diffusion.cpp:27-79; penalty.cpp:60-84)
//  - max diagonal -> eps = 1e-8 max diag (auto_shift, diffusion.cpp:81)
//  - K_H  coarsen_kernel: Galerkin edge sums under 2^d aggregation
//  - K_S  sweep_kernel: omega-Jacobi on the 5/7-point stencil, row sums in
//         the CSR ascending-column order of sparse.cpp:65-74; the first sweep
//         from zero, the prolongation and the final <v, p> partials are fused
//  - K_R  restrict_kernel: r = b - M x summed over the 2^d children
//  - R(f) penalty_kernel: diffusion.cpp:89-101 in canonical order
// Storage: per level the d edge-coefficient arrays (cx, cy, cz), zero where
// an edge is missing; no CSR is ever built (sparse.cpp's std::map assembly
// is replaced by one pass over the field).
#include <cudaTypedefs.h>

#include <mutex>

#include "internal.cuh"
#include "vec.cuh"

namespace mlsqr_b200 {

struct Lvl {  // POD view of one level for kernels
  int nx, ny, nz;
  const double* cx;
  const double* cy;  // nullptr below 2D
  const double* cz;  // nullptr below 3D
  const double* eps; // device scalar
};

__device__ __forceinline__ double diag_at(const Lvl& L, int x, int y, int z, size_t i) {
  const size_t nxy = (size_t)L.nx * L.ny;
  double d = 0.0;
  if (x > 0) d = d + L.cx[i - 1];
  if (x + 1 < L.nx) d = d + L.cx[i];
  if (L.cy) {
    if (y > 0) d = d + L.cy[i - L.nx];
    if (y + 1 < L.ny) d = d + L.cy[i];
  }
  if (L.cz) {
    if (z > 0) d = d + L.cz[i - nxy];
    if (z + 1 < L.nz) d = d + L.cz[i];
  }
  return d;
}

// value of the (possibly prolongated) iterate at fine index j
template <bool PROLONG>
__device__ __forceinline__ double xval(const double* __restrict__ x, const double* __restrict__ xc,
                                       const Lvl& L, int cnx, int cny, int xx, int yy, int zz,
                                       size_t j) {
  double v = x[j];
  if (PROLONG) {
    const int Z = L.cz ? zz / 2 : 0, Y = L.cy ? yy / 2 : 0;
    v = v + xc[((size_t)Z * cny + Y) * cnx + xx / 2];
  }
  return v;
}

// (M x)_i in ascending column order: z-, y-, x-, diag, x+, y+, z+
template <bool PROLONG>
__device__ __forceinline__ double m_row(const Lvl& L, const double* __restrict__ x,
                                        const double* __restrict__ xc, int cnx, int cny, int xx,
                                        int yy, int zz, size_t i, double diag) {
  const size_t nxy = (size_t)L.nx * L.ny;
  double acc = 0.0;
  if (L.cz && zz > 0) acc = acc + -L.cz[i - nxy] * xval<PROLONG>(x, xc, L, cnx, cny, xx, yy, zz - 1, i - nxy);
  if (L.cy && yy > 0) acc = acc + -L.cy[i - L.nx] * xval<PROLONG>(x, xc, L, cnx, cny, xx, yy - 1, zz, i - L.nx);
  if (xx > 0) acc = acc + -L.cx[i - 1] * xval<PROLONG>(x, xc, L, cnx, cny, xx - 1, yy, zz, i - 1);
  acc = acc + diag * xval<PROLONG>(x, xc, L, cnx, cny, xx, yy, zz, i);
  if (xx + 1 < L.nx) acc = acc + -L.cx[i] * xval<PROLONG>(x, xc, L, cnx, cny, xx + 1, yy, zz, i + 1);
  if (L.cy && yy + 1 < L.ny) acc = acc + -L.cy[i] * xval<PROLONG>(x, xc, L, cnx, cny, xx, yy + 1, zz, i + L.nx);
  if (L.cz && zz + 1 < L.nz) acc = acc + -L.cz[i] * xval<PROLONG>(x, xc, L, cnx, cny, xx, yy, zz + 1, i + nxy);
  return acc;
}

enum SweepMode { kFirst = 0, kNormal = 1, kProlong = 2 };

// one omega-Jacobi sweep: out = x + (omega * (b - M x)) / D   (x = 0 for kFirst,
// x = x + P xc for kProlong); seg (optional) <- partials of out * b  (stencil_zm.cuh)
#include "stencil_zm.cuh"
#include "tma.cuh"
#include "sweep_fn.cuh"
#include "stencil_ym.cuh"

// y = (M + eps I) x   (tests; penalty_gradient, diffusion.cpp:103-106)
__global__ void m_apply_kernel(Lvl L, const double* __restrict__ x, double* __restrict__ y) {
  const int rows = L.ny * L.nz;
  const int xx = blockIdx.x * 32 + threadIdx.x;
  if (xx >= L.nx) return;
  for (int row = blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += gridDim.y * blockDim.y) {  // gridDim.y <= 65535
    const int yy = row % L.ny, zz = row / L.ny;
    const size_t i = (size_t)row * L.nx + xx;
    const double d = diag_at(L, xx, yy, zz, i) + *L.eps;
    y[i] = m_row<false>(L, x, nullptr, 0, 0, xx, yy, zz, i, d);
  }
}

// Galerkin coarse edges (oracle coarsen()): sum of the fine edges crossing each coarse face
__global__ void coarsen_kernel(Lvl F, int cnx, int cny, int cnz, int czoff, int cnzg,
                               double* __restrict__ ccx, double* __restrict__ ccy,
                               double* __restrict__ ccz) {
  const int crows = cny * cnz;
  const int X = blockIdx.x * 32 + threadIdx.x;
  if (X >= cnx) return;
  for (int row = blockIdx.y * blockDim.y + threadIdx.y; row < crows; row += gridDim.y * blockDim.y) {  // gridDim.y <= 65535
    const int Y = row % cny, Z = row / cny;
    const size_t fnx = F.nx, fnxy = (size_t)F.nx * F.ny;
    const int zc = F.cz ? 2 : 1, yc = F.cy ? 2 : 1;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (int dz = 0; dz < zc; ++dz)
      for (int dy = 0; dy < yc; ++dy)
        if (X + 1 < cnx) sx = sx + F.cx[(size_t)(zc * Z + dz) * fnxy + (size_t)(yc * Y + dy) * fnx + 2 * X + 1];
    if (F.cy)
      for (int dz = 0; dz < zc; ++dz)
        for (int dx = 0; dx < 2; ++dx)
          if (Y + 1 < cny) sy = sy + F.cy[(size_t)(zc * Z + dz) * fnxy + (size_t)(2 * Y + 1) * fnx + 2 * X + dx];
    if (F.cz)
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx)
          if (Z + czoff + 1 < cnzg) sz = sz + F.cz[(size_t)(2 * Z + 1) * fnxy + (size_t)(2 * Y + dy) * fnx + 2 * X + dx];
    const size_t I = (size_t)row * cnx + X;
    ccx[I] = sx;
    if (ccy) ccy[I] = sy;
    if (ccz) ccz[I] = sz;
  }
}

// K_D: edge coefficients from a field, plus the max unshifted diagonal (atomic max on
// the bit pattern of non-negative doubles: order-independent, deterministic)
__global__ void edge_coeffs_kernel(const double* __restrict__ f, int nx, int ny, int nz, int dims,
                                   int kind, double T, double h, double scale, int zoff, int nzg,
                                   double* __restrict__ cx, double* __restrict__ cy,
                                   double* __restrict__ cz) {
  const int rows = ny * nz;
  const int xx = blockIdx.x * 32 + threadIdx.x;
  if (xx >= nx) return;
  for (int row = blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += gridDim.y * blockDim.y) {  // gridDim.y <= 65535
    const int yy = row % ny, zz = row / ny;
    const size_t i = (size_t)row * nx + xx, nxy = (size_t)nx * ny;
    const double fi = f[i];
    cx[i] = xx + 1 < nx ? diffusivity(kind, T, fabs((f[i + 1] - fi) / h)) * scale : 0.0;
    if (dims >= 2) cy[i] = yy + 1 < ny ? diffusivity(kind, T, fabs((f[i + nx] - fi) / h)) * scale : 0.0;
    // global top plane has no +z edge; a slab's top plane reads f from the ghost plane above
    if (dims >= 3) cz[i] = zz + zoff + 1 < nzg ? diffusivity(kind, T, fabs((f[i + nxy] - fi) / h)) * scale : 0.0;
  }
}

__global__ void max_diag_kernel(Lvl L, unsigned long long* __restrict__ out) {
  __shared__ double wmax[8];
  const int rows = L.ny * L.nz;
  const int xx = blockIdx.x * 32 + threadIdx.x;
  double d = 0.0;
  // grid-stride over rows; the max is exact in any order
  for (int row = blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += gridDim.y * blockDim.y)
    if (xx < L.nx) d = fmax(d, diag_at(L, xx, row % L.ny, row / L.ny, (size_t)row * L.nx + xx));
  for (int off = 16; off >= 1; off >>= 1) d = fmax(d, __shfl_down_sync(kFull, d, off));
  if (threadIdx.x == 0) wmax[threadIdx.y] = d;
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    for (int w = 1; w < (int)blockDim.y; ++w) d = fmax(d, wmax[w]);
    if (d > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(d));  // one atomic per block
  }
}

// eps_0 = given (>= 0) or 1e-8 * max diag; eps_l = eps_{l-1} * 2^d (exact)
__global__ void set_eps_kernel(const unsigned long long* __restrict__ maxd, double eps_cfg,
                               double mult, int levels, double* __restrict__ eps) {
  double e = eps_cfg >= 0.0 ? eps_cfg : 1e-8 * __longlong_as_double((long long)*maxd);
  for (int l = 0; l < levels; ++l) {
    eps[l] = e;
    e = e * mult;
  }
}

// the eps chain of an agglomerated coarse hierarchy continues the fine one's: eps_l = e * 2^(d l)
__global__ void set_eps_from_kernel(const double* __restrict__ e0, double mult, int levels, double* __restrict__ eps) {
  double e = *e0;
  for (int l = 0; l < levels; ++l) {
    eps[l] = e;
    e = e * mult;
  }
}

// R(f): per-node sum of its x/y/z edge terms, canonical segment partials
__global__ void penalty_kernel(const double* __restrict__ f, int nx, int ny, int nz, int dims,
                               int kind, double T, double h, double w, int zoff, int nzg,
                               double* __restrict__ seg) {
  const int rows = ny * nz;
  for (int row = blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += gridDim.y * blockDim.y) {  // gridDim.y <= 65535
    const int xx = blockIdx.x * 32 + threadIdx.x;
    double v = 0.0;
    if (xx < nx) {
      const int yy = row % ny, zz = row / ny;
      const size_t i = (size_t)row * nx + xx, nxy = (size_t)nx * ny;
      const double fi = f[i];
      if (xx + 1 < nx) v = v + w * r_value(kind, T, fabs((f[i + 1] - fi) / h));
      if (dims >= 2 && yy + 1 < ny) v = v + w * r_value(kind, T, fabs((f[i + nx] - fi) / h));
      if (dims >= 3 && zz + zoff + 1 < nzg) v = v + w * r_value(kind, T, fabs((f[i + nxy] - fi) / h));
    }
    const double s = tree32(v);
    if (threadIdx.x == 0) seg[(size_t)row * ((nx + 31) / 32) + blockIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static inline dim3 row_grid(int nx, int rows) {
  return dim3((unsigned)((nx + 31) / 32), row_grid((size_t)rows));
}

class VCycle final : public Pc {
 public:
  // device array with a zero guard zone of g elements on both sides (branch-free stencils)
  struct GBuf {
    DevBuf<double> raw;
    double* p = nullptr;
    void alloc(size_t n, size_t g, cudaStream_t s) {
      raw.alloc(n + 2 * g);
      MLSQR_CUDA(cudaMemsetAsync(raw.p, 0, sizeof(double) * (n + 2 * g), s));
      p = raw.p + g;
    }
  };
  struct Level {
    int nx, ny, nz;
    size_t n;
    GBuf cx, cy, cz, xa, xb, b;
  };

  VCycle(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, double h, int levels, int nu_pre,
         int nu_post, double omega, int kc)
      : dims_(dims), h_(h), nu_pre_(nu_pre), nu_post_(nu_post), kc_(kc), omega_(omega) {
    ctx = c;
    require(dims >= 1 && dims <= 3, MLSQR_EINVAL, "grid must be 1D, 2D or 3D");
    const size_t ey = dims >= 2 ? ny : 1, ez = dims >= 3 ? nz : 1;
    require(nx >= 2 && (dims < 2 || ey >= 2) && (dims < 3 || ez >= 2), MLSQR_EDIM,
            "grid extents must be at least 2");
    require(h > 0.0, MLSQR_EINVAL, "grid spacing must be positive");
    require(levels >= 1 && levels <= 16 && nu_pre >= 1 && kc >= 1, MLSQR_EINVAL,
            "V-cycle needs levels >= 1, nu_pre >= 1, coarse sweeps >= 1");
    // the SpdMap contract (spdsolve.hpp:11-14): M^-1 must be a fixed SYMMETRIC positive definite
    // map, which a V-cycle with omega-Jacobi smoothing is only when the post-smoother mirrors the
    // pre-smoother; an asymmetric cycle would silently break the bidiagonalization
    require(nu_post == nu_pre, MLSQR_EINVAL,
            "V-cycle SpdMap needs nu_post == nu_pre (a symmetric map, spdsolve.hpp:11-14)");
    const size_t f = (size_t)1 << (levels - 1);
    require(nx % f == 0 && nx / f >= 2 && (dims < 2 || (ey % f == 0 && ey / f >= 2)) &&
                (dims < 3 || (ez % f == 0 && ez / f >= 2)),
            MLSQR_EINVAL, "every active grid extent must halve evenly down to the coarsest level");
    n = nx * ey * ez;
    lv_.resize((size_t)levels);
    for (int l = 0; l < levels; ++l) {
      Level& L = lv_[(size_t)l];
      L.nx = (int)(nx >> l);
      L.ny = (int)(dims >= 2 ? ey >> l : 1);
      L.nz = (int)(dims >= 3 ? ez >> l : 1);
      L.n = (size_t)L.nx * L.ny * L.nz;
      // guard: one plane + 64 (x[i +- nxy], and the prefetch of plane z+2 = nz)
      const size_t g = (size_t)L.nx * L.ny + 64;
      // coefficients: two guard planes -- the fused first sweeps on a slab form D on ghost plane -1
      // (cz one plane further down, cy one row up: cy[i - nx] of row 0)
      const size_t gc = g + (size_t)L.nx * L.ny;
      L.cx.alloc(L.n, gc, c->stream);
      if (dims >= 2) L.cy.alloc(L.n, gc, c->stream);
      if (dims >= 3) L.cz.alloc(L.n, gc, c->stream);
      L.xa.alloc(L.n, g, c->stream);
      L.xb.alloc(L.n, g, c->stream);
      if (l > 0) L.b.alloc(L.n, g, c->stream);  // guarded: ghost planes of the restricted rhs
    }
    if (c->sharded()) {
      // z slabs: every level's local planes must stay even-aligned with the global grid
      require(dims == 3, MLSQR_EINVAL, "z-slab decomposition needs a 3D grid");
      require(c->zoff % (long)f == 0 && c->nzg % (long)f == 0 && c->zoff + (long)ez <= c->nzg,
              MLSQR_EINVAL, "slab offsets and the global z extent must be multiples of 2^(levels-1)");
      fg_.alloc(n, (size_t)nx * ey + 64, c->stream);
    }
    eps_.alloc((size_t)levels);
    maxd_.alloc(1);
    if (const char* e = getenv("MLSQR_FN_SWEEPS")) fn_enabled_ = e[0] != '0';
    MLSQR_CUDA(cudaMemsetAsync(eps_.p, 0, sizeof(double) * levels, c->stream));
    if (c->sharded()) setup_agglomeration(nu_pre, nu_post, omega, kc);
  }

  ~VCycle() override {
    delete coarse_;
    delete cctx_;
  }

  // Coarse-level agglomeration: from the first level whose slab holds at most
  // kAggPlanes planes, every rank runs the rest of the V-cycle redundantly on the whole coarse
  // grid (an unsharded hierarchy on a private unsharded context) instead of exchanging ghost
  // planes on every coarse sweep: one allgather of the restricted rhs per V-cycle replaces ~4
  // latency-bound exchanges per coarse level.  Per element the arithmetic is the slab path's, so
  // results stay bit-identical.  MLSQR_AGG_PLANES overrides the threshold (0 disables).
  void setup_agglomeration(int nu_pre, int nu_post, double omega, int kc) {
    int planes = kAggPlanes;
    if (const char* e = getenv("MLSQR_AGG_PLANES")) planes = atoi(e);
    const int P = ctx->comm->size;
    for (int l = 1; l < (int)lv_.size() && planes > 0; ++l) {
      const Level& L = lv_[(size_t)l];
      if (L.nz > planes) continue;
      if ((long)L.nz * P != nzg_l(l)) return;  // unequal slabs: stay sharded
      la_ = l;
      break;
    }
    if (la_ <= 0) return;
    cctx_ = new Ctx();
    cctx_->device = ctx->device;
    cctx_->stream = ctx->stream;
    cctx_->sm_count = ctx->sm_count;
    cctx_->l2_bytes = ctx->l2_bytes;
    const Level& A = lv_[(size_t)la_];
    coarse_ = new VCycle(cctx_, dims_, (size_t)A.nx, (size_t)A.ny, (size_t)nzg_l(la_), h_ * (double)(1 << la_),
                         (int)lv_.size() - la_, nu_pre, nu_post, omega, kc);
    coarse_->fn_enabled_ = fn_enabled_;
    cb_.alloc(coarse_->n);
  }

  Lvl view(int l) const {
    const Level& L = lv_[(size_t)l];
    return Lvl{L.nx, L.ny, L.nz, L.cx.p, dims_ >= 2 ? L.cy.p : nullptr,
               dims_ >= 3 ? L.cz.p : nullptr, eps_.p + l};
  }

  double mult() const {
    double m = 2.0;
    if (dims_ >= 2) m *= 2.0;
    if (dims_ >= 3) m *= 2.0;
    return m;
  }

  // build coarse levels from level 0 (device-resident); eps_cfg < 0 -> auto shift
  // global z offset / extent of level l (slab decomposition; identity when unsharded)
  int zoff_l(int l) const { return ctx->sharded() ? (int)(ctx->zoff >> l) : 0; }
  int nzg_l(int l) const { return ctx->sharded() ? (int)(ctx->nzg >> l) : lv_[(size_t)l].nz; }

  void build(double eps_cfg) {
    Level& L0 = lv_[0];
    MLSQR_CUDA(cudaMemsetAsync(maxd_.p, 0, sizeof(unsigned long long), ctx->stream));
    {
      dim3 grd = row_grid(L0.nx, L0.ny * L0.nz);
      const unsigned cap = (unsigned)(ctx->sm_count * 16 / (grd.x ? grd.x : 1) + 1);
      if (grd.y > cap) grd.y = cap;
      max_diag_kernel<<<grd, dim3(32, 8), 0, ctx->stream>>>(view(0), maxd_.p);
    }
    ctx->count();
    if (ctx->sharded()) {
      TimedRegion tc(ctx, MLSQR_TCLASS_COLL);
      ctx->comm->allreduce_max_u64(maxd_.p, ctx->stream);  // order-free max
    }
    set_eps_kernel<<<1, 1, 0, ctx->stream>>>(maxd_.p, eps_cfg, mult(), (int)lv_.size(), eps_.p);
    ctx->count();
    coarsen_all();
    if (coarse_) {
      // the whole level-la_ operator on every rank: gather the slabs' coefficients (slabs are
      // contiguous z ranges in rank order), continue the eps chain, coarsen from there
      const Level& A = lv_[(size_t)la_];
      VCycle::Level& C0 = coarse_->lv_[0];
      ctx->comm->allgather(A.cx.p, A.n, C0.cx.p, ctx->stream);
      ctx->comm->allgather(A.cy.p, A.n, C0.cy.p, ctx->stream);
      ctx->comm->allgather(A.cz.p, A.n, C0.cz.p, ctx->stream);
      set_eps_from_kernel<<<1, 1, 0, ctx->stream>>>(eps_.p + la_, mult(), (int)coarse_->lv_.size(), coarse_->eps_.p);
      ctx->count();
      coarse_->coarsen_all();
      ctx->count((int)cctx_->launches);
      cctx_->launches = 0;
    }
    ctx->check_launch();
  }

  void coarsen_all() {
    for (size_t l = 1; l < lv_.size(); ++l) {
      Level& C = lv_[l];
      coarsen_kernel<<<row_grid(C.nx, C.ny * C.nz), dim3(32, 8), 0, ctx->stream>>>(
          view((int)l - 1), C.nx, C.ny, C.nz, zoff_l((int)l), nzg_l((int)l), C.cx.p,
          dims_ >= 2 ? C.cy.p : nullptr, dims_ >= 3 ? C.cz.p : nullptr);
      ctx->count();
    }
    // the sweeps read cz[z-1] of the plane below a slab; the fused first sweeps also form D on
    // the ghost planes -1 and nz (cx, cy there, cz two planes below): fill those ghosts on every level
    if (ctx->sharded() && dims_ >= 3)
      for (size_t l = 0; l < lv_.size(); ++l) {
        const Level& L = lv_[l];
        const size_t pl = (size_t)L.nx * L.ny;
        halo_planes(ctx, L.cz.p, pl, L.nz, L.nz >= 2 ? 2 : 1);
        if (L.nz >= 2) {
          halo_planes(ctx, L.cx.p, pl, L.nz, 1);
          halo_planes(ctx, L.cy.p, pl, L.nz, 1);
        }
      }
    ctx->check_launch();
  }

  void set_coefficients(const double* cx, const double* cy, const double* cz, double eps) {
    Level& L0 = lv_[0];
    MLSQR_CUDA(cudaMemcpyAsync(L0.cx.p, cx, sizeof(double) * L0.n, cudaMemcpyDeviceToDevice, ctx->stream));
    if (dims_ >= 2) MLSQR_CUDA(cudaMemcpyAsync(L0.cy.p, cy, sizeof(double) * L0.n, cudaMemcpyDeviceToDevice, ctx->stream));
    if (dims_ >= 3) MLSQR_CUDA(cudaMemcpyAsync(L0.cz.p, cz, sizeof(double) * L0.n, cudaMemcpyDeviceToDevice, ctx->stream));
    zero_boundary_edges_kernel<<<row_grid(L0.nx, L0.ny * L0.nz), dim3(32, 8), 0, ctx->stream>>>(
        view(0), zoff_l(0), nzg_l(0), L0.cx.p, dims_ >= 2 ? L0.cy.p : nullptr, dims_ >= 3 ? L0.cz.p : nullptr);
    ctx->count();
    build(eps);
  }

  // K_D from a field f (device, unguarded): the slab's top plane needs f one plane above
  void edge_coeffs(const double* f, int kind, double T) {
    Level& L0 = lv_[0];
    const double h = h_;
    double w = h;
    if (dims_ >= 2) w = h * h;
    if (dims_ >= 3) w = h * h * h;
    const double scale = w / (h * h);
    const double* src = f;
    if (ctx->sharded()) {
      MLSQR_CUDA(cudaMemcpyAsync(fg_.p, f, sizeof(double) * L0.n, cudaMemcpyDeviceToDevice, ctx->stream));
      halo_planes(ctx, fg_.p, (size_t)L0.nx * L0.ny, L0.nz, 1);
      src = fg_.p;
    }
    edge_coeffs_kernel<<<row_grid(L0.nx, L0.ny * L0.nz), dim3(32, 8), 0, ctx->stream>>>(
        src, L0.nx, L0.ny, L0.nz, dims_, kind, T, h, scale, zoff_l(0), nzg_l(0), L0.cx.p, L0.cy.p, L0.cz.p);
    ctx->count();
  }

  double update(const double* f, int kind, double T, double eps_cfg) {
    edge_coeffs(f, kind, T);
    build(eps_cfg);
    double e = 0.0;
    MLSQR_CUDA(cudaMemcpyAsync(&e, eps_.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    MLSQR_CUDA(cudaStreamSynchronize(ctx->stream));
    return e;
  }

  // device-resident variant used by the outer loop (no host sync); eps stays on device
  void update_async(const double* f, int kind, double T, double eps_cfg) {
    edge_coeffs(f, kind, T);
    build(eps_cfg);
  }
  const double* eps_dev() const { return eps_.p; }
  void level0(int* dims, int* nx, int* ny, int* nz, double* h, const double** cx, const double** cy,
              const double** cz, const double** eps) const {
    const Level& L = lv_[0];
    *dims = dims_;
    *nx = L.nx;
    *ny = L.ny;
    *nz = L.nz;
    *h = h_;
    *cx = L.cx.p;
    *cy = dims_ >= 2 ? L.cy.p : nullptr;
    *cz = dims_ >= 3 ? L.cz.p : nullptr;
    *eps = eps_.p;
  }

  void m_apply(const double* x, double* y) {
    const Level& L0 = lv_[0];
    m_apply_kernel<<<row_grid(L0.nx, L0.ny * L0.nz), dim3(32, 8), 0, ctx->stream>>>(view(0), x, y);
    ctx->count();
    ctx->check_launch();
  }

  size_t row_len() const override { return (size_t)lv_[0].nx; }

  void solve(const double* p, double* v, double* seg, const int* gate, RowShape) override {
    TimedRegion tr(ctx, MLSQR_TCLASS_MG);
    level(0, p, v, seg, gate);
    ctx->check_launch();
  }

 private:
  // 32-bit element indices when the level, its guard planes and the kernels' look-ahead fit
  static bool fits_i32(const Level& L) { return ((long)L.nz + 4) * L.nx * L.ny + 1024 < 2147483647L; }

  template <int MODE>
  void sweep(int l, const double* x, const double* xc, const double* b, double* out, double* seg,
             const int* gate) {
    const Level& L = lv_[(size_t)l];
    int cnx = 0, cny = 0;
    if (l + 1 < (int)lv_.size()) {
      cnx = lv_[(size_t)l + 1].nx;
      cny = lv_[(size_t)l + 1].ny;
    }
    TimedRegion tr(ctx, l == 0 ? MLSQR_TCLASS_SMOOTH : -1);
    TimedRegion tk(ctx, l != 0 ? -1 : MODE == kProlong ? MLSQR_TCLASS_SWEEP_PROLONG
                                     : MODE == kNormal ? MLSQR_TCLASS_SWEEP_LAST : MLSQR_TCLASS_SWEEP_FN);
    const int zc = zm_chunk(L.nx, L.ny, L.nz, ctx->sm_count);
    dim3 grd((unsigned)((L.nx + 31) / 32), (unsigned)((L.ny + 7) / 8), (unsigned)((L.nz + zc - 1) / zc));
    if (dims_ == 3 && fits_i32(L))
      sweep_zm_kernel<3, MODE, int><<<grd, dim3(32, 8), 0, ctx->stream>>>(view(l), x, xc, cnx, cny, b, out, omega_, seg, gate, zc);
    else if (dims_ == 3)
      sweep_zm_kernel<3, MODE><<<grd, dim3(32, 8), 0, ctx->stream>>>(view(l), x, xc, cnx, cny, b, out, omega_, seg, gate, zc);
    else if (dims_ == 2 && ym_ && (long)((L.nx + 31) / 32) * ((L.ny + 7) / 8) > 4L * ctx->sm_count) {
      const int yc = ym_chunk(L.nx, L.ny, ctx->sm_count, 4);
      sweep_ym_kernel<MODE><<<dim3((unsigned)((L.nx + 31) / 32), (unsigned)((L.ny + 8 * yc - 1) / (8 * yc))), dim3(32, 8), 0,
                              ctx->stream>>>(view(l), x, xc, cnx, cny, b, out, omega_, seg, gate, yc);
    } else if (dims_ == 2)
      sweep_zm_kernel<2, MODE><<<grd, dim3(32, 8), 0, ctx->stream>>>(view(l), x, xc, cnx, cny, b, out, omega_, seg, gate, zc);
    else
      sweep_zm_kernel<1, MODE><<<grd, dim3(32, 8), 0, ctx->stream>>>(view(l), x, xc, cnx, cny, b, out, omega_, seg, gate, zc);
    ctx->count();
  }

  void restrict_to(int l, const double* x, const double* b, const int* gate) {
    const Level& L = lv_[(size_t)l];
    Level& C = lv_[(size_t)l + 1];
    TimedRegion tk(ctx, l == 0 ? MLSQR_TCLASS_RESTRICT : -1);
    const int zc = zm_chunk(L.nx, L.ny, L.nz, ctx->sm_count);
    dim3 grd((unsigned)((L.nx + 31) / 32), (unsigned)((L.ny + 7) / 8), (unsigned)((L.nz + zc - 1) / zc));
    if (dims_ == 3 && fits_i32(L))
      restrict_zm_kernel<3, int><<<grd, dim3(32, 8), 0, ctx->stream>>>(view(l), x, b, C.nx, C.ny, C.b.p, gate, zc);
    else if (dims_ == 3)
      restrict_zm_kernel<3><<<grd, dim3(32, 8), 0, ctx->stream>>>(view(l), x, b, C.nx, C.ny, C.b.p, gate, zc);
    else if (dims_ == 2 && ym_ && (long)((L.nx + 31) / 32) * ((L.ny + 7) / 8) > 4L * ctx->sm_count) {
      const int yc = ym_chunk(L.nx, L.ny, ctx->sm_count, 4);
      restrict_ym_kernel<<<dim3((unsigned)((L.nx + 31) / 32), (unsigned)((L.ny + 8 * yc - 1) / (8 * yc))), dim3(32, 8), 0,
                           ctx->stream>>>(view(l), x, b, C.nx, C.b.p, gate, yc);
    } else if (dims_ == 2)
      restrict_zm_kernel<2><<<grd, dim3(32, 8), 0, ctx->stream>>>(view(l), x, b, C.nx, C.ny, C.b.p, gate, zc);
    else
      restrict_zm_kernel<1><<<grd, dim3(32, 8), 0, ctx->stream>>>(view(l), x, b, C.nx, C.ny, C.b.p, gate, zc);
    ctx->count();
  }

  // returns the device pointer holding this level's result (== out when out != nullptr)
  const double* level(int l, const double* b, double* out, double* seg, const int* gate) {
    Level& L = lv_[(size_t)l];
    const bool coarsest = l + 1 == (int)lv_.size();
    const int pre = coarsest ? kc_ : nu_pre_;
    double* bufs[2] = {L.xa.p, L.xb.p};
    int nb = 0;
    // pre-smoothing (or the whole coarse solve) from zero
    const double* cur = nullptr;
    for (int s = 0; s < pre; ++s) {
      const bool fpair = fn_ok(l) && s == 0 && pre >= 2;  // sweeps 1 + 2 in one kernel, x1 on chip
      const bool last_here = coarsest && s + (fpair ? 2 : 1) == pre;
      double* dst = (last_here && out) ? out : bufs[nb];
      double* sg = (last_here && out) ? seg : nullptr;
      if (fpair) {
        if (ctx->sharded()) hx(l, b);  // x1 on the ghost planes needs b there
        sweep_fn(l, b, dst, sg, gate);
        ++s;
      } else if (s == 0) {
        sweep<kFirst>(l, nullptr, nullptr, b, dst, sg, gate);
      } else {
        hx(l, cur);
        sweep<kNormal>(l, cur, nullptr, b, dst, sg, gate);
      }
      cur = dst;
      if (dst == bufs[nb]) nb ^= 1;
    }
    if (coarsest) return cur;
    Level& C = lv_[(size_t)l + 1];
    hx(l, cur);
    restrict_to(l, cur, b, gate);
    const bool agg = coarse_ && l + 1 == la_;
    const double* xc = agg ? coarse_solve(C.b.p, gate) : level(l + 1, C.b.p, nullptr, nullptr, gate);
    for (int s = 0; s < nu_post_; ++s) {
      const bool last = s + 1 == nu_post_;
      double* dst = (last && out) ? out : bufs[nb];
      double* sg = (last && out) ? seg : nullptr;
      if (s == 0) {
        hx(l, cur);
        if (!agg) hx(l + 1, xc);  // an agglomerated correction is whole: its neighbour planes are real
        sweep<kProlong>(l, cur, xc, b, dst, sg, gate);
      } else {
        hx(l, cur);
        sweep<kNormal>(l, cur, nullptr, b, dst, sg, gate);
      }
      cur = dst;
      if (dst == bufs[nb]) nb ^= 1;
    }
    return cur;
  }

  // first + second pre-sweep in one kernel (3D): x1 halos are computed, not exchanged.  On a z
  // slab the kernel also computes x1 on the two ghost planes, from ghost planes of b (level 0:
  // only when the caller's p is guarded) and of the coefficients
  bool fn_ok(int l) const {
    if (!fn_enabled_ || dims_ < 2) return false;
    // small 3D levels: the fused pair marches each block's planes through one serial TMA / x1 ring
    // (~9 us from 64^3 down to 8^3) where two z-march launches take ~3 us each
    if (dims_ == 3 && (long)lv_[(size_t)l].n < fn_min_) return false;
    if (!ctx->sharded()) return true;
    return lv_[(size_t)l].nz >= 2 && (l > 0 || in_guarded);
  }

  void sweep_fn(int l, const double* b, double* out, double* seg, const int* gate) {
    const Level& L = lv_[(size_t)l];
    TimedRegion tr(ctx, l == 0 ? MLSQR_TCLASS_SMOOTH : -1);
    TimedRegion tk(ctx, l == 0 ? MLSQR_TCLASS_SWEEP_FN : -1);
    if (dims_ == 2) {
      // 32-row tiles where 8-row tiles would take more than a wave (MLSQR_YM=0: 8-row tiles)
      if (ym_ && (long)((L.nx + 31) / 32) * ((L.ny + 7) / 8) > 8L * ctx->sm_count)
        sweep_fn2d_kernel<32><<<dim3((unsigned)((L.nx + 31) / 32), (unsigned)((L.ny + 31) / 32)), dim3(32, 8), 0,
                                 ctx->stream>>>(view(l), b, out, omega_, seg, gate);
      else
        sweep_fn2d_kernel<8><<<row_grid(L.nx, L.ny), dim3(32, 8), 0, ctx->stream>>>(view(l), b, out, omega_, seg, gate);
      ctx->count();
      return;
    }
    const int zc = fn_chunk(L.nx, L.ny, L.nz, ctx->sm_count);
    dim3 grd((unsigned)((L.nx + fn::TX - 1) / fn::TX), (unsigned)((L.ny + fn::TY - 1) / fn::TY),
             (unsigned)((L.nz + zc - 1) / zc));
    if (fn_tma_ && sweep_fn_tma(l, b, out, seg, gate, zc, grd)) return;
    sweep_fn_kernel<<<grd, dim3(32, fn::WARPS), 0, ctx->stream>>>(view(l), b, out, omega_, seg, gate, zc, zoff_l(l),
                                                                   nzg_l(l));
    ctx->count();
  }

  // the TMA-fed kernel; false (nothing launched) when a stream cannot be tensor-mapped
  bool sweep_fn_tma(int l, const double* b, double* out, double* seg, const int* gate, int zc, dim3 grd) {
    const Level& L = lv_[(size_t)l];
    static std::once_flag attr;
    std::call_once(attr, [] {
      MLSQR_CUDA(cudaFuncSetAttribute(sweep_fn_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)fnt::SMEM));
    });
    // slabs read the ghost planes (b: one per side; the coefficients: two below for cz, mapped on both sides)
    const int gb = ctx->sharded() ? 1 : 0, gcz = ctx->sharded() ? 2 : 0;
    const size_t nxy = (size_t)L.nx * L.ny;
    CUtensorMap mb{}, mx{}, my{}, mz{};
    const int nz = L.nz;
    if (!tensor_map3d(&mb, b - gb * nxy, L.nx, L.ny, nz + 2 * gb, fnt::BX, fnt::BY) ||
        !tensor_map3d(&mx, L.cx.p - gcz * nxy, L.nx, L.ny, nz + 2 * gcz, fnt::BX, fnt::BY) ||
        !tensor_map3d(&my, L.cy.p - gcz * nxy, L.nx, L.ny, nz + 2 * gcz, fnt::BX, fnt::BY) ||
        !tensor_map3d(&mz, L.cz.p - gcz * nxy, L.nx, L.ny, nz + 2 * gcz, fnt::BX, fnt::BY))
      return false;
    sweep_fn_tma_kernel<<<grd, dim3(32, fn::WARPS), fnt::SMEM, ctx->stream>>>(
        view(l), out, omega_, seg, gate, zc, zoff_l(l), nzg_l(l), gb, gcz, mb, mx, my, mz);
    ctx->count();
    return true;
  }

 public:
  bool fn_enabled_ = true;
  const bool fn_tma_ = !(getenv("MLSQR_FN_TMA") && getenv("MLSQR_FN_TMA")[0] == '0');
  // 2D sweeps / restriction marching rows (stencil_ym.cuh); MLSQR_YM=0: one point per thread
  const bool ym_ = !(getenv("MLSQR_YM") && getenv("MLSQR_YM")[0] == '0');
  // the smallest 3D level (points) that runs the fused first sweeps (MLSQR_FN_MIN)
  const long fn_min_ = getenv("MLSQR_FN_MIN") ? atol(getenv("MLSQR_FN_MIN")) : 262144;

 private:

  int dims_;
  double h_;
  int nu_pre_, nu_post_, kc_;
  double omega_;
  std::vector<Level> lv_;
  DevBuf<double> eps_;
  DevBuf<unsigned long long> maxd_;
  GBuf fg_;  // guarded copy of the field for K_D (z-sharded)
  // coarse-level agglomeration (z-sharded): levels >= la_ run whole on every rank
  static constexpr int kAggPlanes = 8;
  int la_ = 0;
  VCycle* coarse_ = nullptr;
  Ctx* cctx_ = nullptr;
  DevBuf<double> cb_;

  // the agglomerated coarse levels: gather this level's rhs slabs, run the rest of the V-cycle
  // on the whole coarse grid, return this rank's slab of the (guarded, whole) coarse correction
  const double* coarse_solve(const double* b_local, const int* gate) {
    const Level& A = lv_[(size_t)la_];
    {
      TimedRegion tc(ctx, MLSQR_TCLASS_COLL);
      ctx->comm->allgather(b_local, A.n, cb_.p, ctx->stream);
    }
    const double* xfull = coarse_->level(0, cb_.p, nullptr, nullptr, gate);
    ctx->count((int)cctx_->launches);  // the coarse kernels are this library's launches too
    cctx_->launches = 0;
    return xfull + (size_t)zoff_l(la_) * A.nx * A.ny;
  }

  // fill the one-plane ghosts of a level-l iterate (z-sharded)
  void hx(int l, const double* v) {
    if (!ctx->sharded()) return;
    const Level& L = lv_[(size_t)l];
    halo_planes(ctx, const_cast<double*>(v), (size_t)L.nx * L.ny, L.nz, 1);
  }
};

VCycle* make_vcycle(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, double h, int levels,
                    int nu_pre, int nu_post, double omega, int coarse_sweeps) {
  return new VCycle(c, dims, nx, ny, nz, h, levels, nu_pre, nu_post, omega, coarse_sweeps);
}
void vcycle_set_coefficients(VCycle* v, const double* cx, const double* cy, const double* cz,
                             double eps) {
  v->set_coefficients(cx, cy, cz, eps);
}
double vcycle_update(VCycle* v, const double* f, int kind, double T, double eps) {
  return v->update(f, kind, T, eps);
}
void vcycle_update_async(VCycle* v, const double* f, int kind, double T, double eps) {
  v->update_async(f, kind, T, eps);
}
const double* vcycle_eps_dev(VCycle* v) { return v->eps_dev(); }
void vcycle_level0(VCycle* v, int* dims, int* nx, int* ny, int* nz, double* h, const double** cx,
                   const double** cy, const double** cz, const double** eps) {
  v->level0(dims, nx, ny, nz, h, cx, cy, cz, eps);
}
Pc* vcycle_as_pc(VCycle* v) { return v; }
void vcycle_m_apply(VCycle* v, const double* x, double* y) { v->m_apply(x, y); }

// ---------------------------------------------------------------------------
class IdentityMap final : public Pc {
 public:
  IdentityMap(Ctx* c, size_t nn) {
    ctx = c;
    n = nn;
  }
  void solve(const double* p, double* v, double* seg, const int* gate, RowShape shape) override {
    Epi e;
    e.gate = gate;
    axpby_epi(ctx, p, v, shape, e);
    if (seg) seg_dot(ctx, v, p, shape, seg, gate);
  }
};
Pc* make_identity_map(Ctx* c, size_t n) { return new IdentityMap(c, n); }

// R(f) on the device, canonical order; returns to the host (synchronizes)
// R(f) on the device in canonical order.  z-sharded: f is copied into the guarded
// buffer fguard (n + 2 planes) so the slab's top plane sees f one plane above, and the
// segment partials are reduced across ranks.
void penalty_functional_async(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, double h,
                              const double* f, int kind, double T, double* seg, double* scratch,
                              double* gathered, double* fguard, double* out) {
  const size_t ey = dims >= 2 ? ny : 1, ez = dims >= 3 ? nz : 1;
  RowShape s{nx, ey * ez};
  double w = h;
  if (dims >= 2) w = h * h;
  if (dims >= 3) w = h * h * h;
  const double* src = f;
  if (c->sharded()) {
    require(fguard != nullptr, MLSQR_EINVAL, "sharded R(f) needs a guarded buffer");
    MLSQR_CUDA(cudaMemcpyAsync(fguard, f, sizeof(double) * s.n(), cudaMemcpyDeviceToDevice, c->stream));
    halo_planes(c, fguard, nx * ey, (long)ez, 1);
    src = fguard;
  }
  const int zoff = c->sharded() ? (int)c->zoff : 0, nzg = c->sharded() ? (int)c->nzg : (int)ez;
  penalty_kernel<<<row_grid((int)nx, (int)(ey * ez)), dim3(32, 8), 0, c->stream>>>(
      src, (int)nx, (int)ey, (int)ez, dims, kind, T, h, w, zoff, nzg, seg);
  c->count();
  reduce_segments_dist(c, seg, s.segments(), scratch, gathered, out, nullptr);
}

double penalty_functional_dev(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, double h,
                              const double* f, int kind, double T) {
  const size_t ey = dims >= 2 ? ny : 1, ez = dims >= 3 ? nz : 1;
  RowShape s{nx, ey * ez};
  const size_t J = s.segments();
  const size_t G = dist_gather_size(c, J);
  DevBuf<double> seg(J), scratch(reduce_scratch_size(G > J ? G : J) + J), gathered(G > 0 ? G : 1), out(1);
  DevBuf<double> fg;
  double* fguard = nullptr;
  if (c->sharded()) {
    fg.alloc(s.n() + 2 * nx * ey);
    MLSQR_CUDA(cudaMemsetAsync(fg.p, 0, sizeof(double) * fg.n, c->stream));
    fguard = fg.p + nx * ey;
  }
  penalty_functional_async(c, dims, nx, ny, nz, h, f, kind, T, seg.p, scratch.p, gathered.p, fguard, out.p);
  double r = 0.0;
  MLSQR_CUDA(cudaMemcpyAsync(&r, out.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  MLSQR_CUDA(cudaStreamSynchronize(c->stream));
  return r;
}

}  // namespace mlsqr_b200
