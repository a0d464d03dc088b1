// blur.cu -- K_A / K_B: separable Gaussian blur A (= A^T) with the LSQR
// xpby + norm epilogue fused in (SURVEY.md §2.1 K_A, K_B).
//
// Replaces GaussianConvolution1D::convolve (linop.cpp:115-121) and
// SeparableGaussianBlur2D::blur (linop.cpp:151-162; z pass added for 3D).
// Per output the sum runs over the tap window in ascending source index,
// exactly like the reference's dot over [lo, hi] (zero extension: terms
// outside the domain contribute +0 and cannot change the sum), passes in
// the order x -> y -> z with rounded intermediates.
#include "internal.cuh"
#include "vec.cuh"

namespace mlsqr_b200 {

constexpr int kMaxRadius = 36;

struct Taps {
  double t[2 * kMaxRadius + 1];
  int R;
};

// ---------------------------------------------------------------------------
// 2D tile kernel: x then y pass through shared memory, one launch per apply.
// Block (32, 8) computes a 32 x TY tile of outputs; the input halo tile
// (32 + 2R) x (TY + 2R) is staged in smem with the input scale applied.
// ---------------------------------------------------------------------------
template <int TY>
__global__ void __launch_bounds__(256) blur2d_tile_kernel(const double* __restrict__ in,
                                                          double* __restrict__ out, int nx,
                                                          int ny, int nz, Taps taps,
                                                          EpiArgs e) {
  if (e.gate && *e.gate == 0) return;
  extern __shared__ double sm[];
  const int R = taps.R;
  const int W = 32 + 2 * R, H = TY + 2 * R;
  double* tin = sm;              // H x W input tile
  double* tx = sm + (size_t)H * W;  // H x 32 x-pass result
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
  // x pass for all H rows of the tile
  for (int ly = threadIdx.y; ly < H; ly += 8) {
    const int gx = x0 + threadIdx.x;
    double acc = 0.0;
    const double* row = tin + (size_t)ly * W + threadIdx.x;
    for (int k = 0; k <= 2 * R; ++k) acc = acc + taps.t[k] * row[k];
    (void)gx;
    tx[ly * 32 + threadIdx.x] = acc;
  }
  __syncthreads();
  for (int ty = threadIdx.y; ty < TY; ty += 8) {
    const int gy = y0 + ty, gx = x0 + threadIdx.x;
    double acc = 0.0;
    for (int k = 0; k <= 2 * R; ++k) acc = acc + taps.t[k] * tx[(ty + k) * 32 + threadIdx.x];
    double v = 0.0;
    const bool ok = gx < nx && gy < ny;
    if (ok) {
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

// ---------------------------------------------------------------------------
// generic single-axis pass (1D, and the z pass of 3D)
// ---------------------------------------------------------------------------
template <int AXIS>
__global__ void blur_pass_kernel(const double* __restrict__ in, double* __restrict__ out,
                                 size_t nx, size_t ny, size_t nz, Taps taps, EpiArgs e,
                                 bool first, bool last) {
  if (e.gate && *e.gate == 0) return;
  const size_t rows = ny * nz;
  const size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y;
  if (row >= rows) return;
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
      acc = acc + taps.t[k] * a;
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

class BlurOp final : public Op {
 public:
  BlurOp(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, const double* taps, int radius)
      : dims_(dims), nx_(nx), ny_(dims >= 2 ? ny : 1), nz_(dims >= 3 ? nz : 1) {
    ctx = c;
    require(radius >= 0 && radius <= kMaxRadius, MLSQR_EINVAL,
            "blur radius must lie in [0, " + std::to_string(kMaxRadius) + "]");
    require(nx_ >= 1 && ny_ >= 1 && nz_ >= 1, MLSQR_EDIM, "blur grid must be non-empty");
    for (int k = 0; k < 2 * radius + 1; ++k) taps_.t[k] = taps[k];
    taps_.R = radius;
    rows = cols = nx_ * ny_ * nz_;
    data_shape = sol_shape = RowShape{nx_, ny_ * nz_};
    if (dims_ == 3) tmp_.alloc(rows);
    if (dims_ >= 2) {
      smem_ = sizeof(double) * ((size_t)(kTY + 2 * radius) * (32 + 2 * radius) + (size_t)(kTY + 2 * radius) * 32);
      if (smem_ > 48 * 1024)
        MLSQR_CUDA(cudaFuncSetAttribute(blur2d_tile_kernel<kTY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_));
    }
  }

  void apply(const double* x, double* y, const Epi& e) override { run(x, y, e); }
  void adjoint(const double* y, double* x, const Epi& e) override { run(y, x, e); }  // A = A^T

 private:
  void run(const double* in, double* out, const Epi& e) {
    TimedRegion tr(ctx, MLSQR_TCLASS_BLUR);
    EpiArgs a = to_args(e);
    const size_t rows_ = ny_ * nz_;
    dim3 blk(32, 8);
    dim3 grd((unsigned)((nx_ + 31) / 32), (unsigned)((rows_ + 7) / 8));
    if (dims_ == 1) {
      blur_pass_kernel<0><<<grd, blk, 0, ctx->stream>>>(in, out, nx_, ny_, nz_, taps_, a, true, true);
      ctx->count();
    } else {
      // 2D tile pass (x then y); for 3D it writes the xy-blurred planes to tmp_
      constexpr int TY = kTY;
      const size_t smem = smem_;
      auto kern = blur2d_tile_kernel<TY>;
      dim3 g2((unsigned)((nx_ + 31) / 32), (unsigned)((ny_ + TY - 1) / TY), (unsigned)nz_);
      if (dims_ == 2) {
        kern<<<g2, blk, smem, ctx->stream>>>(in, out, (int)nx_, (int)ny_, (int)nz_, taps_, a);
        ctx->count();
      } else {
        EpiArgs first = a;
        first.old = nullptr;
        first.seg = nullptr;
        kern<<<g2, blk, smem, ctx->stream>>>(in, tmp_.p, (int)nx_, (int)ny_, (int)nz_, taps_, first);
        EpiArgs last = a;
        last.sx = nullptr;
        blur_pass_kernel<2><<<grd, blk, 0, ctx->stream>>>(tmp_.p, out, nx_, ny_, nz_, taps_, last, false, true);
        ctx->count(2);
      }
    }
    ctx->check_launch();
  }

  static constexpr int kTY = 32;
  int dims_;
  size_t nx_, ny_, nz_;
  size_t smem_ = 0;
  Taps taps_{};
  DevBuf<double> tmp_;
};

Op* make_blur(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, const double* taps, int radius) {
  require(dims >= 1 && dims <= 3, MLSQR_EINVAL, "blur dims must be 1, 2 or 3");
  return new BlurOp(c, dims, nx, ny, nz, taps, radius);
}

}  // namespace mlsqr_b200
