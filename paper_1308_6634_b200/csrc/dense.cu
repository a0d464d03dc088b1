// dense.cu -- K_A' / K_B': the dense (fDOT-like) sensitivity operator and the
// identity operator (DenseOperator / IdentityOperator, linop.cpp:56-84).
//
// A x : one CTA (32 warps) per NR rows.  Each row dot is the canonical
//       reduction over 32-column segments (tree32 per segment, then tree-32
//       levels), so y_i is bit-identical to the oracle's DEVICE-order dot.
// A^T y: one thread per column, rows in 8 fixed chunks, sequential inside a
//       chunk (the reference's per-row axpy order, linop.cpp:78-84), chunk
//       partials added in order -- deterministic and row-shardable.
#include "internal.cuh"
#include "vec.cuh"

namespace mlsqr_b200 {

// ---------------------------------------------------------------------------
// y = A (x*sx) for NR rows per CTA; level-1 partials staged in smem.
// ---------------------------------------------------------------------------
template <int NR>
__global__ void __launch_bounds__(1024) gemv_kernel(const double* __restrict__ A,
                                                    const double* __restrict__ x, size_t rows,
                                                    size_t cols, double* __restrict__ y,
                                                    const double* sx, const int* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ double l1[];  // NR x G1 level-1 partials
  const size_t r0 = (size_t)blockIdx.x * NR;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t nseg = (cols + 31) / 32;
  const size_t G1 = (nseg + 31) / 32;
  const double s = sx ? *sx : 1.0;
  for (size_t g = w; g < G1; g += 32) {
    double keep[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) keep[r] = 0.0;
    for (int k = 0; k < 32; ++k) {
      const size_t col = (g * 32 + k) * 32 + lane;
      double xv = 0.0;
      if (col < cols) {
        xv = x[col];
        if (sx) xv = xv * s;
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        double v = 0.0;
        if (col < cols && r0 + r < rows) v = A[(r0 + r) * cols + col] * xv;
        v = tree32(v);
        v = __shfl_sync(kFull, v, 0);
        if (lane == k) keep[r] = v;
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const double t = tree32(keep[r]);
      if (lane == 0) l1[r * G1 + g] = t;
    }
  }
  __syncthreads();
  // remaining levels over the G1 level-1 partials of each row (serial trees)
  if (threadIdx.x < NR && r0 + threadIdx.x < rows) {
    double* L = l1 + threadIdx.x * G1;
    size_t J = G1;  // level 1 is done; continue while more than one value remains
    while (J > 1) {
      const size_t G = (J + 31) / 32;
      for (size_t q = 0; q < G; ++q) {
        double v[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) v[l] = (q * 32 + l < J) ? L[q * 32 + l] : 0.0;
        L[q] = tree32_serial(v);
      }
      J = G;
    }
    y[r0 + threadIdx.x] = L[0];
  }
}

// ---------------------------------------------------------------------------
// x = A^T (y*sy) with the fused epilogue; one thread per column.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gemvt_kernel(const double* __restrict__ A,
                                                    const double* __restrict__ y, size_t rows,
                                                    size_t cols, double* __restrict__ out,
                                                    EpiArgs e, int chunks) {
  if (e.gate && *e.gate == 0) return;
  const size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  const double s = e.sx ? *e.sx : 1.0;
  const size_t ch = rows / (size_t)chunks;
  double tot = 0.0;
  for (int c = 0; c < chunks; ++c) {
    double acc = 0.0;
    const size_t i0 = (size_t)c * ch, i1 = i0 + ch;
    size_t i = i0;
    for (; i + 4 <= i1; i += 4) {
      const double a0 = A[i * cols + j], a1 = A[(i + 1) * cols + j];
      const double a2 = A[(i + 2) * cols + j], a3 = A[(i + 3) * cols + j];
      double y0 = y[i], y1 = y[i + 1], y2 = y[i + 2], y3 = y[i + 3];
      if (e.sx) { y0 = y0 * s; y1 = y1 * s; y2 = y2 * s; y3 = y3 * s; }
      acc = acc + y0 * a0;
      acc = acc + y1 * a1;
      acc = acc + y2 * a2;
      acc = acc + y3 * a3;
    }
    for (; i < i1; ++i) {
      double yi = y[i];
      if (e.sx) yi = yi * s;
      acc = acc + yi * A[i * cols + j];
    }
    tot = chunks == 1 ? acc : tot + acc;
  }
  out[j] = epilogue(tot, e, j);
}

// row shards: this rank's canonical row chunks of A^T (y*sy), one partial n-vector per chunk
// (the same per-chunk loop as gemvt_kernel), later allgathered and summed in chunk order
__global__ void __launch_bounds__(256) gemvt_part_kernel(const double* __restrict__ A,
                                                         const double* __restrict__ y, size_t rows,
                                                         size_t cols, double* __restrict__ part,
                                                         const double* sx, const int* gate, int chunks) {
  if (gate && *gate == 0) return;
  const size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  const double s = sx ? *sx : 1.0;
  const size_t ch = rows / (size_t)chunks;
  for (int c = 0; c < chunks; ++c) {
    double acc = 0.0;
    const size_t i0 = (size_t)c * ch, i1 = i0 + ch;
    size_t i = i0;
    for (; i + 4 <= i1; i += 4) {
      const double a0 = A[i * cols + j], a1 = A[(i + 1) * cols + j];
      const double a2 = A[(i + 2) * cols + j], a3 = A[(i + 3) * cols + j];
      double y0 = y[i], y1 = y[i + 1], y2 = y[i + 2], y3 = y[i + 3];
      if (sx) { y0 = y0 * s; y1 = y1 * s; y2 = y2 * s; y3 = y3 * s; }
      acc = acc + y0 * a0;
      acc = acc + y1 * a1;
      acc = acc + y2 * a2;
      acc = acc + y3 * a3;
    }
    for (; i < i1; ++i) {
      double yi = y[i];
      if (sx) yi = yi * s;
      acc = acc + yi * A[i * cols + j];
    }
    part[(size_t)c * cols + j] = acc;
  }
}

// the 8 gathered chunk partials summed in chunk order (gemvt_kernel's tot), then the epilogue
__global__ void gemvt_combine_kernel(const double* __restrict__ part, size_t cols, int chunks,
                                     double* __restrict__ out, EpiArgs e) {
  if (e.gate && *e.gate == 0) return;
  const size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double tot = 0.0;
  for (int c = 0; c < chunks; ++c) tot = chunks == 1 ? part[j] : tot + part[(size_t)c * cols + j];
  out[j] = epilogue(tot, e, j);
}

__global__ void epi_vec_kernel(const double* __restrict__ in, double* __restrict__ out, size_t n,
                               EpiArgs e) {
  if (e.gate && *e.gate == 0) return;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = epilogue(in[i], e, i);
}

__global__ void fdot_form_kernel(const double* __restrict__ gs, const double* __restrict__ gd,
                                 size_t nvox, int ndet, size_t rows, size_t row0,
                                 double* __restrict__ A) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t row = blockIdx.y + (size_t)gridDim.y * blockIdx.z;
  if (row >= rows || idx >= nvox) return;
  const size_t s = (row0 + row) / (size_t)ndet, d = (row0 + row) % (size_t)ndet;
  A[row * nvox + idx] = gs[s * nvox + idx] * gd[d * nvox + idx];
}

class DenseOp final : public Op {
 public:
  DenseOp(Ctx* c, size_t r, size_t cl, size_t sol_row_len) {
    ctx = c;
    rows = r;
    cols = cl;
    require(r >= 1 && cl >= 1, MLSQR_EDIM, "operator shape must be at least 1x1");
    if (c->row_sharded()) {
      // rank k holds rows [k m/P, (k+1) m/P): whole canonical A^T chunks and whole 32-row
      // reduction segments, so every result equals the unsharded operator's bit for bit
      const long P = c->comm->size;
      require(c->rows_g > 0 && c->rows_g % 8 == 0 && 8 % P == 0, MLSQR_EINVAL,
              "row shards need m % 8 == 0 and P in {1, 2, 4, 8}");
      require((long)r * P == c->rows_g, MLSQR_EDIM, "local rows must be m / P");
      require((r % 32) == 0, MLSQR_EDIM, "local rows must be a multiple of 32 (whole reduction segments)");
      require(c->row0 == (long)r * c->comm->rank, MLSQR_EINVAL, "row shard offset must be rank * m / P");
      part_.alloc((size_t)(8 / P) * cl);
      gath_.alloc((size_t)8 * cl);
    }
    data_shape = RowShape{rows, 1};
    const size_t L = (sol_row_len && cols % sol_row_len == 0) ? sol_row_len : cols;
    sol_shape = RowShape{L, cols / L};
    a_.alloc(rows * cols);
    tmp_.alloc(rows > cols ? rows : cols);
    const size_t nseg = (cols + 31) / 32, G1 = (nseg + 31) / 32;
    smem_ = sizeof(double) * kNR * (G1 < 1 ? 1 : G1);
    if (smem_ > 48 * 1024)
      MLSQR_CUDA(cudaFuncSetAttribute(gemv_kernel<kNR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_));
  }
  static constexpr int kNR = 4;
  size_t smem_ = 0;
  DevBuf<double> a_;

  int tclass() const override { return MLSQR_TCLASS_DENSE; }

  void apply(const double* x, double* y, const Epi& e) override {
    TimedRegion tr(ctx, MLSQR_TCLASS_DENSE);
    constexpr int NR = kNR;
    const size_t smem = smem_;
    double* dst = e.old ? tmp_.p : y;
    gemv_kernel<NR><<<(unsigned)((rows + NR - 1) / NR), 1024, smem, ctx->stream>>>(
        a_.p, x, rows, cols, dst, e.sx, e.gate);
    ctx->count();
    ctx->check_launch();
    if (e.old || e.seg) {
      Epi e2 = e;
      e2.sx = nullptr;
      axpby_epi(ctx, dst, y, data_shape, e2);
    }
  }

  void adjoint(const double* y, double* x, const Epi& e) override {
    TimedRegion tr(ctx, MLSQR_TCLASS_DENSE);
    EpiArgs a = to_args(e);
    a.seg = nullptr;
    if (ctx->row_sharded()) {
      const int local = 8 / ctx->comm->size;
      gemvt_part_kernel<<<(unsigned)((cols + 255) / 256), 256, 0, ctx->stream>>>(a_.p, y, rows, cols, part_.p, e.sx,
                                                                                 e.gate, local);
      ctx->comm->allgather(part_.p, (size_t)local * cols, gath_.p, ctx->stream);
      gemvt_combine_kernel<<<(unsigned)((cols + 255) / 256), 256, 0, ctx->stream>>>(gath_.p, cols, 8, x, a);
      ctx->count(2);
    } else {
      const int chunks = rows % 8 == 0 ? 8 : 1;
      gemvt_kernel<<<(unsigned)((cols + 255) / 256), 256, 0, ctx->stream>>>(a_.p, y, rows, cols, x, a, chunks);
      ctx->count();
    }
    ctx->check_launch();
    if (e.seg) seg_dot(ctx, x, x, sol_shape, e.seg, e.gate);
  }

 private:
  DevBuf<double> tmp_;
  DevBuf<double> part_, gath_;  // row shards: local chunk partials, all 8 gathered
};

Op* make_dense(Ctx* c, size_t rows, size_t cols, const double* a, bool a_on_device,
               size_t sol_row_len) {
  auto* op = new DenseOp(c, rows, cols, sol_row_len);
  try {
    MLSQR_CUDA(cudaMemcpyAsync(op->a_.p, a, sizeof(double) * rows * cols,
                               a_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                               c->stream));
    MLSQR_CUDA(cudaStreamSynchronize(c->stream));
  } catch (...) {
    delete op;
    throw;
  }
  return op;
}

Op* make_dense_fdot(Ctx* c, size_t nvox, int nsrc, int ndet, const double* gs, const double* gd,
                    size_t sol_row_len) {
  size_t rows = (size_t)nsrc * (size_t)ndet, row0 = 0;
  if (c->row_sharded()) {  // this rank forms only its rows of the global (s, d) row space
    require(c->rows_g == (long)rows, MLSQR_EDIM, "row-shard context rows != nsrc * ndet");
    rows /= (size_t)c->comm->size;
    row0 = (size_t)c->row0;
  }
  auto* op = new DenseOp(c, rows, nvox, sol_row_len);
  try {
    DevBuf<double> dgs((size_t)nsrc * nvox), dgd((size_t)ndet * nvox);
    MLSQR_CUDA(cudaMemcpyAsync(dgs.p, gs, sizeof(double) * nsrc * nvox, cudaMemcpyHostToDevice, c->stream));
    MLSQR_CUDA(cudaMemcpyAsync(dgd.p, gd, sizeof(double) * ndet * nvox, cudaMemcpyHostToDevice, c->stream));
    const unsigned gy = (unsigned)(rows < 65535 ? rows : 65535);
    const unsigned gz = (unsigned)((rows + gy - 1) / gy);
    dim3 grd((unsigned)((nvox + 255) / 256), gy, gz);
    fdot_form_kernel<<<grd, 256, 0, c->stream>>>(dgs.p, dgd.p, nvox, ndet, rows, row0, op->a_.p);
    c->count();
    c->check_launch();
    MLSQR_CUDA(cudaStreamSynchronize(c->stream));
  } catch (...) {
    delete op;
    throw;
  }
  return op;
}

class IdentityOp final : public Op {
 public:
  IdentityOp(Ctx* c, size_t n, size_t row_len) {
    ctx = c;
    rows = cols = n;
    require(n >= 1, MLSQR_EDIM, "operator shape must be at least 1x1");
    const size_t L = (row_len && n % row_len == 0) ? row_len : n;
    data_shape = sol_shape = RowShape{L, n / L};
  }
  void apply(const double* x, double* y, const Epi& e) override { axpby_epi(ctx, x, y, data_shape, e); }
  void adjoint(const double* y, double* x, const Epi& e) override { axpby_epi(ctx, y, x, sol_shape, e); }
};

Op* make_identity(Ctx* c, size_t n, size_t row_len) { return new IdentityOp(c, n, row_len); }

}  // namespace mlsqr_b200
