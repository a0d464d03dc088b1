// dense.cu -- K_A' / K_B': the dense (fDOT-like) sensitivity operator and the
// identity operator (DenseOperator / IdentityOperator, linop.cpp:56-84).
//
// A x : a warp per (row, column part); each row dot is the canonical reduction
//       over 32-column segments (tree32 per segment, then tree-32 levels), so y_i
//       is bit-identical to the oracle's DEVICE-order dot.
// A^T y: one thread per column, rows in 8 fixed chunks, sequential inside a
//       chunk (the reference's per-row axpy order, linop.cpp:78-84), chunk
//       partials added in order -- deterministic and row-shardable.
#include <cudaTypedefs.h>

#include <cmath>
#include <mutex>

#include "internal.cuh"
#include "vec.cuh"

namespace mlsqr_b200 {

#include "tma.cuh"

// ---------------------------------------------------------------------------
// y = A (x*sx) in the canonical order with ~5 instructions per element instead of ~20:
// a CTA owns 8 rows x one column part and walks its 1024-column groups in lockstep.
// Per group the x slice and each warp's row slice are loaded coalesced (16-byte loads)
// into shared memory laid out as 32 segments of 34 doubles; lane l then reads segment l
// with conflict-free 16-byte loads, forms its 32 products and reduces them with
// tree32_serial (the same pairing as a 32-lane shuffle tree), and the warp trees the 32
// segment partials (level 1) into a global [rows x G1] buffer.  gemv_top_kernel runs the
// remaining tree-32 levels of each row.
// ---------------------------------------------------------------------------
constexpr int kGemvWarps = 8;
constexpr int kSegPitch = 34;                  // padded segment pitch (doubles)
constexpr int kGrpDoubles = 32 * kSegPitch;    // one 1024-column group

__global__ void __launch_bounds__(256, 2) gemv_l1_kernel(const double* __restrict__ A,
                                                         const double* __restrict__ x, size_t rows,
                                                         size_t cols, int parts, double* __restrict__ l1,
                                                         const double* sx, const int* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) double gsm[];
  double* xs = gsm;                       // [kGrpDoubles]
  double* as = gsm + kGrpDoubles;         // [kGemvWarps][kGrpDoubles]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t rg = blockIdx.x / (size_t)parts, part = blockIdx.x % (size_t)parts;
  const size_t row = rg * kGemvWarps + w;
  const bool live = row < rows;
  const size_t nseg = (cols + 31) / 32, G1 = (nseg + 31) / 32;
  const size_t gp = (G1 + parts - 1) / parts;
  const size_t g0 = part * gp, g1 = g0 + gp < G1 ? g0 + gp : G1;
  const double s = sx ? *sx : 1.0;
  const double* __restrict__ Ar = A + (live ? row : 0) * cols;
  const bool vec = (cols % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(x) % 16 == 0);
  // element e (0..1023) of a group sits at segment e / 32, slot e % 32
  auto sidx = [](int e) { return (e >> 5) * kSegPitch + (e & 31); };
  for (size_t g = g0; g < g1; ++g) {
    const size_t base = g * 1024;
    const bool full = vec && base + 1024 <= cols;
    __syncthreads();  // the previous group's readers are done
    if (full) {
      {  // x slice: 512 pairs over 256 threads
        const int e = 2 * (int)threadIdx.x;
        const double2 v0 = __ldg(reinterpret_cast<const double2*>(x + base + e));
        const double2 v1 = __ldg(reinterpret_cast<const double2*>(x + base + 512 + e));
        *reinterpret_cast<double2*>(xs + sidx(e)) = v0;
        *reinterpret_cast<double2*>(xs + sidx(512 + e)) = v1;
      }
      if (live) {
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          const int e = 64 * b + 2 * lane;
          *reinterpret_cast<double2*>(as + w * kGrpDoubles + sidx(e)) = *reinterpret_cast<const double2*>(Ar + base + e);
        }
      }
    } else {
      for (int e = threadIdx.x; e < 1024; e += 32 * kGemvWarps) xs[sidx(e)] = base + e < cols ? x[base + e] : 0.0;
      if (live)
        for (int e = lane; e < 1024; e += 32) as[w * kGrpDoubles + sidx(e)] = base + e < cols ? Ar[base + e] : 0.0;
    }
    __syncthreads();
    if (live) {
      const double* ap = as + w * kGrpDoubles + lane * kSegPitch;
      const double* xp = xs + lane * kSegPitch;
      double p[32];
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const double2 av = *reinterpret_cast<const double2*>(ap + j);
        double2 xv = *reinterpret_cast<const double2*>(xp + j);
        if (sx) {
          xv.x = xv.x * s;
          xv.y = xv.y * s;
        }
        p[j] = av.x * xv.x;
        p[j + 1] = av.y * xv.y;
      }
      // zero extension past cols: those products are 0 * 0 = +0 (staged zeros)
      const double t = tree32(tree32_serial(p));  // segment partial, then level 1 across the group
      if (lane == 0) l1[row * G1 + g] = t;
    }
  }
}

// The same level-1 kernel fed by bulk copies (cp.async.bulk into an mbarrier ring): thread 0 issues,
// per 1024-column group, nine contiguous 8 KB copies (the x slice and the eight row slices) into
// stage (g mod kBulkStages), kBulkStages - 1 groups ahead of the group being reduced, so the
// compute warps issue no global loads or staging stores at all.  The slices sit UNPADDED in shared
// memory; lane l still owns segment l but walks its sixteen double2 pairs rotated by l
// (pair (jj + l) mod 16 at step jj: conflict-free 16-byte loads).  tree32_serial's pairing is
// invariant under that rotation -- v[i] meets v[i + 16], then sums i and i + 8 of the sixteen, ...
// and IEEE addition commutes -- so the pair partners always sit at STATIC register slots (jj and
// jj - 8, then k and k + 4, ...) and the segment partial is bit-identical to tree32_serial's.
// Used when the operator has whole 8-row groups and whole 1024-column groups, 16-byte aligned;
// anything else runs gemv_l1_kernel (MLSQR_GEMV_BULK=0 forces it).
constexpr int kBulkStages = 3;
constexpr int kBulkStage = 1024 * (1 + kGemvWarps);  // doubles per stage: x, then the 8 rows
constexpr size_t kBulkSmem = sizeof(double) * kBulkStages * kBulkStage + 8 * kBulkStages;

__device__ __forceinline__ void bulk_load(double* dst, const double* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(256, 1) gemv_l1_bulk_kernel(const double* __restrict__ A,
                                                              const double* __restrict__ x, size_t rows,
                                                              size_t cols, int parts, double* __restrict__ l1,
                                                              const double* sx, const int* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ __align__(128) double gsm[];
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(gsm + kBulkStages * kBulkStage);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t rg = blockIdx.x / (size_t)parts, part = blockIdx.x % (size_t)parts;
  const size_t row0 = rg * kGemvWarps;
  const size_t G1 = cols / 1024;
  const size_t gp = (G1 + parts - 1) / parts;
  const size_t g0 = part * gp, g1 = g0 + gp < G1 ? g0 + gp : G1;
  const double s = sx ? *sx : 1.0;
  auto issue = [&](size_t g) {  // thread 0 only
    if (g >= g1) return;
    const unsigned st = (unsigned)((g - g0) % kBulkStages);
    double* d = gsm + (size_t)st * kBulkStage;
    mbar_arrive_expect(bars + st, 8192u * (1 + kGemvWarps));
    bulk_load(d, x + g * 1024, 8192u, bars + st);
#pragma unroll
    for (int r = 0; r < kGemvWarps; ++r) bulk_load(d + 1024 * (1 + r), A + (row0 + r) * cols + g * 1024, 8192u, bars + st);
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < kBulkStages; ++k) mbar_init(bars + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < kBulkStages - 1; ++k) issue(g0 + k);
  for (size_t g = g0; g < g1; ++g) {
    const unsigned it = (unsigned)(g - g0), st = it % kBulkStages;
    // the stage refilled now was read in the previous iteration: everyone is past it
    __syncthreads();
    if (threadIdx.x == 0) issue(g + kBulkStages - 1);
    mbar_wait(bars + st, (it / kBulkStages) & 1u);
    const double2* ap = reinterpret_cast<const double2*>(gsm + (size_t)st * kBulkStage + 1024 * (1 + w) + 32 * lane);
    const double2* xp = reinterpret_cast<const double2*>(gsm + (size_t)st * kBulkStage + 32 * lane);
    double2 P[8], T[8];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const int q = (jj + lane) & 15;
      const double2 av = ap[q];
      double2 xv = xp[q];
      if (sx) {
        xv.x = xv.x * s;
        xv.y = xv.y * s;
      }
      const double2 pr = make_double2(av.x * xv.x, av.y * xv.y);
      if (jj < 8) {
        P[jj] = pr;
      } else {  // tree32_serial level 1: v[i] + v[i + 16]
        T[jj - 8] = make_double2(P[jj - 8].x + pr.x, P[jj - 8].y + pr.y);
      }
    }
    // levels 2..5 (sums i, i + 8 of 16; i, i + 4 of 8; i, i + 2 of 4; 0, 1)
    double2 U[4], V[2];
#pragma unroll
    for (int k = 0; k < 4; ++k) U[k] = make_double2(T[k].x + T[k + 4].x, T[k].y + T[k + 4].y);
#pragma unroll
    for (int k = 0; k < 2; ++k) V[k] = make_double2(U[k].x + U[k + 2].x, U[k].y + U[k + 2].y);
    const double2 Z = make_double2(V[0].x + V[1].x, V[0].y + V[1].y);
    const double t = tree32(Z.x + Z.y);  // level 1 across the group's 32 segments
    if (lane == 0) l1[(row0 + w) * G1 + g] = t;
  }
}

// levels >= 2 of each row's canonical tree over its G1 level-1 partials
__global__ void gemv_top_kernel(double* __restrict__ l1, size_t rows, size_t G1, double* __restrict__ y,
                                const int* gate) {
  if (gate && *gate == 0) return;
  const size_t row = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  double* L = l1 + row * G1;
  size_t J = G1;
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
  y[row] = L[0];
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
    l1_.alloc(rows * (((cols + 31) / 32 + 31) / 32));
    // set outside any graph capture (the first A x may run inside the captured LSQR iteration)
    MLSQR_CUDA(cudaFuncSetAttribute(gemv_l1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    MLSQR_CUDA(cudaFuncSetAttribute(gemv_l1_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBulkSmem));
  }
  static constexpr int kSmem = sizeof(double) * kGrpDoubles * (1 + kGemvWarps);
  DevBuf<double> a_;

  int tclass() const override { return MLSQR_TCLASS_DENSE; }

  void apply(const double* x, double* y, const Epi& e) override {
    TimedRegion tr(ctx, MLSQR_TCLASS_DENSE);
    double* dst = e.old ? tmp_.p : y;
    const size_t nseg = (cols + 31) / 32, G1 = (nseg + 31) / 32;
    // column parts per 8-row group: enough CTAs for ~7 waves of 2 CTAs per SM
    const size_t groups = (rows + kGemvWarps - 1) / kGemvWarps;
    const size_t want = (size_t)ctx->sm_count * 2 * 7;
    size_t parts = (want + groups - 1) / groups;
    if (parts < 1) parts = 1;
    if (parts > G1) parts = G1;
    static const bool bulk_on = !(getenv("MLSQR_GEMV_BULK") && getenv("MLSQR_GEMV_BULK")[0] == '0');
    const bool bulk = bulk_on && rows % kGemvWarps == 0 && cols % 1024 == 0 &&
                      reinterpret_cast<uintptr_t>(a_.p) % 16 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0;
    if (bulk) {
      // one CTA per SM: the column split that fills whole waves best, with at least ~24 waves of
      // short CTAs where the matrix allows (C4: 8 parts 396 it/s, 2 parts 389)
      double best = -1.0;
      for (size_t p = 1; p <= 16 && p <= G1; ++p) {
        const double w = (double)(groups * p) / ctx->sm_count;
        const double eff = w / std::ceil(w) * (w >= 24.0 ? 1.0 : 0.9 + 0.1 * w / 24.0) * (G1 % p == 0 ? 1.0 : 0.98);
        if (eff > best + 1e-9) {
          best = eff;
          parts = p;
        }
      }
    }
    static const long parts_env = getenv("MLSQR_GEMV_PARTS") ? atol(getenv("MLSQR_GEMV_PARTS")) : 0;
    if (parts_env > 0 && (size_t)parts_env <= G1) parts = (size_t)parts_env;
    const size_t ctas = groups * parts;
    if (bulk)
      gemv_l1_bulk_kernel<<<(unsigned)ctas, 32 * kGemvWarps, kBulkSmem, ctx->stream>>>(a_.p, x, rows, cols, (int)parts,
                                                                                      l1_.p, e.sx, e.gate);
    else
      gemv_l1_kernel<<<(unsigned)ctas, 32 * kGemvWarps, kSmem, ctx->stream>>>(a_.p, x, rows, cols, (int)parts, l1_.p,
                                                                         e.sx, e.gate);
    gemv_top_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, ctx->stream>>>(l1_.p, rows, G1, dst, e.gate);
    ctx->count(2);
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
      {
        TimedRegion tc(ctx, MLSQR_TCLASS_COLL);
        ctx->comm->allgather(part_.p, (size_t)local * cols, gath_.p, ctx->stream);
      }
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
 public:
  DevBuf<double> l1_;           // [rows x G1] level-1 partials of A x
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
