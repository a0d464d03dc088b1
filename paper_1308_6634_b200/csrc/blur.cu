// blur.cu -- K_A / K_B: separable Gaussian blur A (= A^T) with the LSQR
// xpby + norm epilogue fused in (SURVEY.md §2.1 K_A, K_B).
//
// Replaces GaussianConvolution1D::convolve (linop.cpp:115-121) and
// SeparableGaussianBlur2D::blur (linop.cpp:151-162; z pass added for 3D).
// Per output the sum runs over the tap window in ascending source index,
// exactly like the reference's dot over [lo, hi] (zero extension: terms
// outside the domain contribute +0 and cannot change the sum), passes in
// the order x -> y -> z with rounded intermediates.  1D/2D use the
// reference's separate mul + add (bit-identical to its scalar backend);
// 3D (no reference implementation) uses fma chains -- the canonical
// DEVICE order the oracle restates with C fma().
//
// 3D main kernel: blur3d_pipe (blur3d_pipe.cuh) -- TMA plane ring, one barrier per
// plane, z accumulators, persistent round-robin (z chunk, column tile) items; the
// xpby epilogue with the old vector and the canonical |out|^2 segment partials are
// fused.  HBM traffic: read x once, read old once, write out once.
#include <cudaTypedefs.h>

#include <mutex>

#include "internal.cuh"
#include "vec.cuh"

namespace mlsqr_b200 {

constexpr int kMaxRadius = 36;   // taps passed by value (tile / fused kernels)
constexpr int kMaxWide = 512;    // 1D / 2D pass kernels with taps in device memory

struct Taps {
  double t[2 * kMaxRadius + 1];
  int R;
};

template <bool FMA>
__device__ __forceinline__ double mac(double t, double v, double acc) {
  if (FMA) return fma(t, v, acc);
  return acc + t * v;
}

// ---------------------------------------------------------------------------
// 2D tile kernel: x then y pass through shared memory (2D operator; also the
// xy stage of the generic 3D path).
// ---------------------------------------------------------------------------
template <int TY, bool FMA>
__global__ void __launch_bounds__(256) blur2d_tile_kernel(const double* __restrict__ in,
                                                          double* __restrict__ out, int nx,
                                                          int ny, int nz, Taps taps,
                                                          EpiArgs e) {
  if (e.gate && *e.gate == 0) return;
  extern __shared__ double sm[];
  const int R = taps.R;
  const int W = 32 + 2 * R, H = TY + 2 * R;
  double* tin = sm;
  double* tx = sm + (size_t)H * W;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * TY, z = blockIdx.z;
  const size_t plane = (size_t)z * nx * ny;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const double sx = e.sx ? *e.sx : 1.0;
  for (int k = tid; k < H * W; k += 256) {
    const int ly = k / W, lx = k - ly * W;
    const int gx = x0 + lx - R, gy = y0 + ly - R;
    double v = 0.0;
    if (gx >= 0 && gx < nx && gy >= 0 && gy < ny) {
      v = in[plane + (size_t)gy * nx + gx];
      if (e.sx) v = v * sx;
    }
    tin[k] = v;
  }
  __syncthreads();
  for (int ly = threadIdx.y; ly < H; ly += 8) {
    double acc = 0.0;
    const double* row = tin + (size_t)ly * W + threadIdx.x;
    for (int k = 0; k <= 2 * R; ++k) acc = mac<FMA>(taps.t[k], row[k], acc);
    tx[ly * 32 + threadIdx.x] = acc;
  }
  __syncthreads();
  for (int ty = threadIdx.y; ty < TY; ty += 8) {
    const int gy = y0 + ty, gx = x0 + threadIdx.x;
    double acc = 0.0;
    for (int k = 0; k <= 2 * R; ++k) acc = mac<FMA>(taps.t[k], tx[(ty + k) * 32 + threadIdx.x], acc);
    double v = 0.0;
    if (gx < nx && gy < ny) {
      const size_t i = plane + (size_t)gy * nx + gx;
      v = epilogue(acc, e, i);
      out[i] = v;
    }
    if (e.seg && gy < ny) {
      const double s = tree32(v * v);
      const size_t chunks = (size_t)(nx + 31) / 32;
      if (threadIdx.x == 0) e.seg[((size_t)z * ny + gy) * chunks + blockIdx.x] = s;
    }
  }
}

// 2D blur for the radii of the taps-by-value path (R <= 12), same order as blur2d_tile_kernel
// (reference scalar SeparableGaussianBlur2D, linop.cpp:151-162: rows then columns, acc + t * v):
// compile-time R; the x pass makes two outputs per thread from LDS.128 pairs and the y pass four
// rows per thread, both STREAMING their input window (each loaded value goes straight into every
// accumulator it feeds, so each accumulator still sums its taps in ascending order) instead of
// holding it in registers: 32 registers, 8 resident blocks per SM, so C2's 1024 tiles run as one
// wave; the |out|^2 row-segment partials are a register butterfly (tree32's pairs).
template <int R>
__global__ void __launch_bounds__(256, 8) blur2d_reg_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                            int nx, int ny, int nz, Taps taps, EpiArgs e) {
  if (e.gate && *e.gate == 0) return;
  constexpr int TH = 32, NTH = 256;
  constexpr int W = 32 + 2 * R, H = TH + 2 * R, P = (W + 1) & ~1, NT = 2 * R + 1;
  __shared__ __align__(16) double tin[H * P];  // input tile; the x results overwrite columns 0..31
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * TH, z = blockIdx.z;
  const size_t plane = (size_t)z * nx * ny;
  const int tid = threadIdx.y * 32 + threadIdx.x, lane = threadIdx.x, w = threadIdx.y;
  const double sx = e.sx ? *e.sx : 1.0;
  for (int k = tid; k < H * W; k += NTH) {
    const int ly = k / W, lx = k - ly * W;
    const int gx = x0 + lx - R, gy = y0 + ly - R;
    double v = 0.0;
    if (gx >= 0 && gx < nx && gy >= 0 && gy < ny) {
      v = in[plane + (size_t)gy * nx + gx];
      if (e.sx) v = v * sx;
    }
    tin[ly * P + lx] = v;
  }
  __syncthreads();
  // x pass: row r, outputs 2g (taps on window positions 0..2R) and 2g + 1 (positions 1..2R+1),
  // written in place over the row's first 32 columns once every thread of the round (whole rows)
  // has read its window
  for (int base = 0; base < H * 16; base += NTH) {
    const int t = base + tid;
    const bool act = t < H * 16;
    const int r = t >> 4, g = t & 15;
    double a0 = 0.0, a1 = 0.0;
    if (act) {
      const double2* row = reinterpret_cast<const double2*>(tin + r * P + 2 * g);
#pragma unroll
      for (int j = 0; j < R + 1; ++j) {
        const double2 q = row[j];
        a0 = a0 + taps.t[2 * j] * q.x;
        if (j > 0) a1 = a1 + taps.t[2 * j - 1] * q.x;
        if (j < R) a0 = a0 + taps.t[2 * j + 1] * q.y;
        a1 = a1 + taps.t[2 * j] * q.y;
      }
    }
    __syncthreads();
    if (act) *reinterpret_cast<double2*>(tin + r * P + 2 * g) = make_double2(a0, a1);
  }
  __syncthreads();
  // y pass: column `lane`, output rows 4w .. 4w + 3 from x-result rows 4w .. 4w + 3 + 2R
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < 4 + 2 * R; ++j) {
    const double c = tin[(4 * w + j) * P + lane];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (j - i >= 0 && j - i < NT) acc[i] = acc[i] + taps.t[j - i] * c;
  }
  const int gx = x0 + lane;
  double v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gy = y0 + 4 * w + i;
    v[i] = 0.0;
    if (gx < nx && gy < ny) {
      const size_t idx = plane + (size_t)gy * nx + gx;
      v[i] = epilogue(acc[i], e, idx);
      out[idx] = v[i];
    }
  }
  if (e.seg) {
    // tree32 of each row's 32 squares as a butterfly (rows 0/2 on lanes < 16, 1/3 on lanes >= 16)
    const bool h16 = lane & 16, h8 = lane & 8;
    double q[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = v[i] * v[i];
    const double a = (h16 ? q[1] : q[0]) + __shfl_xor_sync(0xffffffffu, h16 ? q[0] : q[1], 16);
    const double b = (h16 ? q[3] : q[2]) + __shfl_xor_sync(0xffffffffu, h16 ? q[2] : q[3], 16);
    double s = (h8 ? b : a) + __shfl_xor_sync(0xffffffffu, h8 ? a : b, 8);
    s = s + __shfl_xor_sync(0xffffffffu, s, 4);
    s = s + __shfl_xor_sync(0xffffffffu, s, 2);
    s = s + __shfl_xor_sync(0xffffffffu, s, 1);
    const int gy = y0 + 4 * w + ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1);
    if ((lane & 7) == 0 && gy < ny) e.seg[((size_t)z * ny + gy) * ((nx + 31) / 32) + blockIdx.x] = s;
  }
}

static bool launch_blur2d_reg(Ctx* c, const double* in, double* out, int nx, int ny, int nz, const Taps& t,
                              const EpiArgs& a) {
  const dim3 blk(32, 8), grd((unsigned)((nx + 31) / 32), (unsigned)((ny + 31) / 32), (unsigned)nz);
  switch (t.R) {
#define MLSQR_B2R(RR) \
  case RR: blur2d_reg_kernel<RR><<<grd, blk, 0, c->stream>>>(in, out, nx, ny, nz, t, a); break;
    MLSQR_B2R(1) MLSQR_B2R(2) MLSQR_B2R(3) MLSQR_B2R(4) MLSQR_B2R(5) MLSQR_B2R(6)
    MLSQR_B2R(7) MLSQR_B2R(8) MLSQR_B2R(9) MLSQR_B2R(10) MLSQR_B2R(11) MLSQR_B2R(12)
#undef MLSQR_B2R
    default: return false;
  }
  c->count();
  return true;
}

// ---------------------------------------------------------------------------
// generic single-axis pass (1D operator; z pass of the generic 3D path)
// ---------------------------------------------------------------------------
// taps by value (kernel parameter, radius <= kMaxRadius) or from device memory (wide kernels:
// the reference's 6 sigma radius on fine 1D/2D grids, e.g. deconv1d n = 512, sigma 0.03 -> R = 93)
struct WideTaps {
  const double* t;
  int R;
};

template <int AXIS, bool FMA, class TT = Taps>
__global__ void blur_pass_kernel(const double* __restrict__ in, double* __restrict__ out,
                                 size_t nx, size_t ny, size_t nz, TT taps, EpiArgs e,
                                 bool first, bool last) {
  if (e.gate && *e.gate == 0) return;
  const size_t rows = ny * nz;
  for (size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += (size_t)gridDim.y * blockDim.y) {  // gridDim.y <= 65535
    const size_t x = (size_t)blockIdx.x * 32 + threadIdx.x;
    const int R = taps.R;
    double v = 0.0;
    if (x < nx) {
      const size_t y = row % ny, z = row / ny;
      long c, N;
      size_t stride, base;
      if (AXIS == 0) {
        c = (long)x; N = (long)nx; stride = 1; base = row * nx;
      } else if (AXIS == 1) {
        c = (long)y; N = (long)ny; stride = nx; base = z * nx * ny + x;
      } else {
        c = (long)z; N = (long)nz; stride = nx * ny; base = y * nx + x;
      }
      const double sx = (first && e.sx) ? *e.sx : 1.0;
      double acc = 0.0;
      for (int k = 0; k <= 2 * R; ++k) {
        const long j = c + k - R;
        if (j < 0 || j >= N) continue;
        double a = in[base + (size_t)j * stride];
        if (first && e.sx) a = a * sx;
        acc = mac<FMA>(taps.t[k], a, acc);
      }
      const size_t i = row * nx + x;
      v = last ? epilogue(acc, e, i) : acc;
      out[i] = v;
    }
    if (last && e.seg) {
      const double s = tree32(v * v);
      if (threadIdx.x == 0) e.seg[row * ((nx + 31) / 32) + blockIdx.x] = s;
    }
  }
}

#include "tma.cuh"
#include "blur3d_pipe.cuh"
#include "blur3d_mma.cuh"

// x / y passes on the FP64 tensor cores (blur3d_mma.cuh) for the BASELINE radii; bit-identical
// to blur3d_pipe.  MLSQR_BLUR_MMA=0 selects the all-DFMA kernel (A/B measurements).
static bool blur_mma_enabled() {
  static const bool on = [] {
    const char* e = getenv("MLSQR_BLUR_MMA");
    return !(e && e[0] == '0');
  }();
  return on;
}
// radius dispatch for the fused kernel (BASELINE taps: 9 (R=4) and 13 (R=6))
static bool fused3d(Ctx* c, int R, const double* in, double* out, int nx, int ny, int nz, const Taps& t,
                    const EpiArgs& a) {
  switch (R) {
    case 1: launch_b3<1>(c, in, out, nx, ny, nz, t, a); return true;
    case 2: launch_b3<2>(c, in, out, nx, ny, nz, t, a); return true;
    case 3: launch_b3<3>(c, in, out, nx, ny, nz, t, a); return true;
    case 4:
      if (!(blur_mma_enabled() && launch_b3m<4>(c, in, out, nx, ny, nz, t, a))) launch_b3<4>(c, in, out, nx, ny, nz, t, a);
      return true;
    case 5: launch_b3<5>(c, in, out, nx, ny, nz, t, a); return true;
    case 6:
      if (!(blur_mma_enabled() && launch_b3m<6>(c, in, out, nx, ny, nz, t, a))) launch_b3<6>(c, in, out, nx, ny, nz, t, a);
      return true;
    case 8: launch_b3<8>(c, in, out, nx, ny, nz, t, a); return true;
    case 12: launch_b3<12>(c, in, out, nx, ny, nz, t, a); return true;
    default: return false;
  }
}

static bool symmetric(const double* t, int R) {
  for (int k = 0; k < R; ++k)
    if (!(t[k] == t[2 * R - k])) return false;
  return true;
}

class BlurOp final : public Op {
 public:
  BlurOp(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, const double* taps, int radius)
      : dims_(dims), nx_(nx), ny_(dims >= 2 ? ny : 1), nz_(dims >= 3 ? nz : 1) {
    ctx = c;
    require(radius >= 0 && radius <= (dims <= 2 ? kMaxWide : kMaxRadius), MLSQR_EINVAL,
            "blur radius must lie in [0, " + std::to_string(dims <= 2 ? kMaxWide : kMaxRadius) + "]");
    require(nx_ >= 1 && ny_ >= 1 && nz_ >= 1, MLSQR_EDIM, "blur grid must be non-empty");
    // adjoint() runs the forward pass (A = A^T, linop.cpp:168-170), which holds only for
    // symmetric taps: anything else would silently break the bidiagonalization
    require(symmetric(taps, radius), MLSQR_EINVAL, "blur taps must be symmetric (t[k] == t[2R-k]): A^T = A");
    if (radius > kMaxRadius) {
      // wide 1D/2D taps live in device memory; 2D runs as x pass + y pass
      wide_ = true;
      dtx_.alloc((size_t)(2 * radius + 1));
      MLSQR_CUDA(cudaMemcpyAsync(dtx_.p, taps, sizeof(double) * (2 * radius + 1), cudaMemcpyHostToDevice, ctx->stream));
      dty_ = dtx_.p;
      ry_ = radius;
      if (dims_ == 2) {
        axes_ = true;
        tmp_.alloc(nx_ * ny_);
      }
      radius = 0;  // the by-value copy is unused
    }
    for (int k = 0; k < 2 * radius + 1; ++k) taps_.t[k] = taps[k];
    taps_.R = wide_ ? (int)(dtx_.n / 2) : radius;
    rows = cols = nx_ * ny_ * nz_;
    data_shape = sol_shape = RowShape{nx_, ny_ * nz_};
    if (dims_ >= 2 && !wide_) {
      smem_ = sizeof(double) * ((size_t)(kTY + 2 * radius) * (32 + 2 * radius) + (size_t)(kTY + 2 * radius) * 32);
      if (smem_ > 48 * 1024) {
        MLSQR_CUDA(cudaFuncSetAttribute(blur2d_tile_kernel<kTY, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_));
        MLSQR_CUDA(cudaFuncSetAttribute(blur2d_tile_kernel<kTY, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_));
      }
    }
    // warm the fused 3D kernel's attribute outside any graph capture
    if (dims_ == 3) {
      bool sym = true;  // the fused kernel reads t[min(k, 2R-k)]
      for (int k = 0; k <= radius; ++k) sym = sym && taps_.t[k] == taps_.t[2 * radius - k];
      fused_ = sym && (radius == 1 || radius == 2 || radius == 3 || radius == 4 || radius == 5 ||
                       radius == 6 || radius == 8 || radius == 12);
      if (!fused_) tmp_.alloc(rows);
      else {
        EpiArgs none{};
        none.gate = nullptr;
        // zero-size probe launch is not allowed; set the attribute via a 1-plane dry run on a tiny grid
        DevBuf<double> probe(1);
        int zero = 0;
        DevBuf<int> g0(1);
        MLSQR_CUDA(cudaMemcpyAsync(g0.p, &zero, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
        none.gate = g0.p;  // gated off: the kernel returns at once
        fused3d(ctx, radius, probe.p, probe.p, 1, 1, 1, taps_, none);
        MLSQR_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->check_launch();
      }
    }
    if (ctx->sharded()) {
      // z-slab of a global grid: the fused 3D kernel reads R ghost planes per side
      require(dims_ == 3 && fused_, MLSQR_EINVAL,
              "z-sharded blur needs a 3D grid and a symmetric radius in {1..6, 8, 12}");
      require(nz_ >= (size_t)radius, MLSQR_EDIM, "z slab thinner than the blur radius");
      const size_t g = (size_t)radius * nx_ * ny_;
      gin_.alloc(rows + 2 * g);
      MLSQR_CUDA(cudaMemsetAsync(gin_.p, 0, sizeof(double) * gin_.n, ctx->stream));
    }
  }

  // SeparableGaussianBlur2D with per-axis factors (linop.cpp:142-149: kx_(nx), ky_(ny) -- a
  // non-square grid has different spacings, hence different taps and radii per axis)
  void set_y_taps(const double* ty, int ry) {
    require(dims_ == 2 && !ctx->sharded(), MLSQR_EINVAL, "per-axis taps are for the 2D operator");
    require(ry >= 0 && ry <= kMaxWide, MLSQR_EINVAL, "blur radius must lie in [0, " + std::to_string(kMaxWide) + "]");
    require(symmetric(ty, ry), MLSQR_EINVAL, "blur taps must be symmetric (t[k] == t[2R-k]): A^T = A");
    if (!wide_) {  // move the x taps to device memory too: both passes read WideTaps
      dtx_.alloc((size_t)(2 * taps_.R + 1));
      MLSQR_CUDA(cudaMemcpyAsync(dtx_.p, taps_.t, sizeof(double) * dtx_.n, cudaMemcpyHostToDevice, ctx->stream));
      wide_ = true;
    }
    dtyo_.alloc((size_t)(2 * ry + 1));
    MLSQR_CUDA(cudaMemcpyAsync(dtyo_.p, ty, sizeof(double) * dtyo_.n, cudaMemcpyHostToDevice, ctx->stream));
    dty_ = dtyo_.p;
    ry_ = ry;
    axes_ = true;
    tmp_.alloc(rows);
  }
  void apply(const double* x, double* y, const Epi& e) override { run(x, y, e); }
  void adjoint(const double* y, double* x, const Epi& e) override { run(y, x, e); }  // A = A^T
  int halo_planes_needed() const override { return ctx->sharded() && dims_ == 3 ? taps_.R : 0; }
  size_t plane_size() const override { return nx_ * ny_; }

 private:
  // z slabs, guarded input whose ghost planes are not filled yet (K_B's u, produced by K_A right
  // before): the R ghost planes per side travel on the side stream while the slab interior
  // (outputs R .. nz-R-1, which read no ghost plane) is blurred; then the two boundary bands.
  // Per output the arithmetic is unchanged, so the split is bit-identical to one launch.
  bool run_split(double* in, double* out, const Epi& e) {
    const int R = taps_.R;
    if (!(fused_ && dims_ == 3 && e.in_guarded && (R == 4 || R == 6) && blur_mma_enabled() &&
          nz_ > (size_t)(4 * R)))
      return false;
    const int nx = (int)nx_, ny = (int)ny_, nz = (int)nz_;
    const EpiArgs a = to_args(e);
    auto band = [&](int zb, int ze) {
      return R == 4 ? launch_b3m_range<4>(ctx, in, out, nx, ny, nz, zb, ze, taps_, a)
                    : launch_b3m_range<6>(ctx, in, out, nx, ny, nz, zb, ze, taps_, a);
    };
    cudaStream_t s = ctx->side_stream();
    MLSQR_CUDA(cudaEventRecord(ctx->ev_fork2, ctx->stream));
    MLSQR_CUDA(cudaStreamWaitEvent(s, ctx->ev_fork2, 0));
    halo_planes(ctx, in, nx_ * ny_, (long)nz_, R, s);
    MLSQR_CUDA(cudaEventRecord(ctx->ev_join2, s));
    const bool ok = band(R, nz - R);  // the TMA map covers the guarded slab: fails for all bands or none
    MLSQR_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_join2, 0));
    if (!ok) return false;
    band(0, R);
    band(nz - R, nz);
    ctx->check_launch();
    return true;
  }

  void run(const double* in, double* out, const Epi& e) {
    TimedRegion tr(ctx, MLSQR_TCLASS_BLUR);
    if (ctx->sharded() && !(e.in_guarded && e.ghosts_ready) && !split_off_ &&
        run_split(const_cast<double*>(in), out, e))
      return;
    if (ctx->sharded() && !(e.in_guarded && e.ghosts_ready)) {
      // fill the ghost planes: in place for guarded solver vectors, else via a staging copy
      const size_t plane = nx_ * ny_, g = (size_t)taps_.R * plane;
      double* src = const_cast<double*>(in);
      if (!e.in_guarded) {
        MLSQR_CUDA(cudaMemcpyAsync(gin_.p + g, in, sizeof(double) * rows, cudaMemcpyDeviceToDevice, ctx->stream));
        src = gin_.p + g;
      }
      halo_planes(ctx, src, plane, (long)nz_, taps_.R);
      in = src;
    }
    EpiArgs a = to_args(e);
    const size_t rows_ = ny_ * nz_;
    dim3 blk(32, 8);
    dim3 grd((unsigned)((nx_ + 31) / 32), row_grid(rows_));
    const WideTaps wx{dtx_.p, (int)(dtx_.n / 2)}, wy{dty_, ry_};
    if (dims_ == 1 && wide_) {
      blur_pass_kernel<0, false, WideTaps><<<grd, blk, 0, ctx->stream>>>(in, out, nx_, ny_, nz_, wx, a, true, true);
      ctx->count();
    } else if (dims_ == 1) {
      blur_pass_kernel<0, false><<<grd, blk, 0, ctx->stream>>>(in, out, nx_, ny_, nz_, taps_, a, true, true);
      ctx->count();
    } else if (dims_ == 3 && fused_) {
      fused3d(ctx, taps_.R, in, out, (int)nx_, (int)ny_, (int)nz_, taps_, a);
    } else {
      dim3 g2((unsigned)((nx_ + 31) / 32), (unsigned)((ny_ + kTY - 1) / kTY), (unsigned)nz_);
      if (dims_ == 2 && axes_) {
        // rows first (x, contiguous), then columns (linop.cpp:151-162), separate mul + add
        EpiArgs first = a;
        first.old = nullptr;
        first.seg = nullptr;
        blur_pass_kernel<0, false, WideTaps><<<grd, blk, 0, ctx->stream>>>(in, tmp_.p, nx_, ny_, nz_, wx, first, true,
                                                                          false);
        EpiArgs last = a;
        last.sx = nullptr;
        blur_pass_kernel<1, false, WideTaps><<<grd, blk, 0, ctx->stream>>>(tmp_.p, out, nx_, ny_, nz_, wy, last, false,
                                                                          true);
        ctx->count(2);
      } else if (dims_ == 2) {
        if (nz_ > 65535 || !launch_blur2d_reg(ctx, in, out, (int)nx_, (int)ny_, (int)nz_, taps_, a)) {
          blur2d_tile_kernel<kTY, false><<<g2, blk, smem_, ctx->stream>>>(in, out, (int)nx_, (int)ny_, (int)nz_, taps_, a);
          ctx->count();
        }
      } else {
        EpiArgs first = a;
        first.old = nullptr;
        first.seg = nullptr;
        blur2d_tile_kernel<kTY, true><<<g2, blk, smem_, ctx->stream>>>(in, tmp_.p, (int)nx_, (int)ny_, (int)nz_, taps_, first);
        EpiArgs last = a;
        last.sx = nullptr;
        blur_pass_kernel<2, true><<<grd, blk, 0, ctx->stream>>>(tmp_.p, out, nx_, ny_, nz_, taps_, last, false, true);
        ctx->count(2);
      }
    }
    ctx->check_launch();
  }

  static constexpr int kTY = 32;
  const bool split_off_ = getenv("MLSQR_BLUR_SPLIT") && getenv("MLSQR_BLUR_SPLIT")[0] == '0';
  DevBuf<double> gin_;  // guarded staging input (z-sharded, unguarded callers)
  int dims_;
  size_t nx_, ny_, nz_;
  size_t smem_ = 0;
  bool fused_ = false;
  Taps taps_{};
  bool axes_ = false;       // 2D as x pass + y pass with per-axis (device) taps
  bool wide_ = false;       // taps in device memory (radius > kMaxRadius or per-axis)
  DevBuf<double> dtx_, dtyo_;
  const double* dty_ = nullptr;
  int ry_ = 0;
  DevBuf<double> tmp_;
};

Op* make_blur(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, const double* taps, int radius) {
  require(dims >= 1 && dims <= 3, MLSQR_EINVAL, "blur dims must be 1, 2 or 3");
  return new BlurOp(c, dims, nx, ny, nz, taps, radius);
}

Op* make_blur2d_axes(Ctx* c, size_t nx, size_t ny, const double* tx, int rx, const double* ty, int ry) {
  BlurOp* b = new BlurOp(c, 2, nx, ny, 1, tx, rx);
  try {
    b->set_y_taps(ty, ry);
  } catch (...) {
    delete b;
    throw;
  }
  return b;
}

}  // namespace mlsqr_b200
