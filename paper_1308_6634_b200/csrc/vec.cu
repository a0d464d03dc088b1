// vec.cu -- canonical reductions and fused BLAS-1 passes (kernels.hpp:15-31
// replaced).  Every dot / nrm2 of the reference (kernels_scalar.cpp:7-23)
// becomes (1) per-32-element segment partials produced inside the kernel that
// writes the vector, then (2) tree-32 levels over the partials, all on the
// device with a fixed shape -> run-to-run bitwise deterministic, no atomics.
#include "internal.cuh"
#include "vec.cuh"

namespace mlsqr_b200 {

// ---------------------------------------------------------------------------
// segment partials of x .* y over a row shape: block (32, 8) = 8 row segments
// ---------------------------------------------------------------------------
__global__ void seg_dot_kernel(const double* __restrict__ x, const double* __restrict__ y,
                               size_t len, size_t rows, size_t chunks, double* __restrict__ seg,
                               const int* gate) {
  if (gate && *gate == 0) return;
  // row-stride loop: gridDim.y is capped at 65535 (row_grid); a warp is one row segment, so
  // every lane of a warp takes the same trip count
  for (size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += (size_t)gridDim.y * blockDim.y) {
    const size_t xi = (size_t)blockIdx.x * 32 + threadIdx.x;
    double v = 0.0;
    if (xi < len) {
      const size_t i = row * len + xi;
      v = x[i] * y[i];
    }
    v = tree32(v);
    if (threadIdx.x == 0) seg[row * chunks + blockIdx.x] = v;
  }
}

void seg_dot(Ctx* c, const double* x, const double* y, RowShape s, double* seg, const int* gate) {
  if (s.n() == 0) return;
  dim3 blk(32, 8), grd((unsigned)s.chunks(), row_grid(s.rows));
  seg_dot_kernel<<<grd, blk, 0, c->stream>>>(x, y, s.len, s.rows, s.chunks(), seg, gate);
  c->count();
  c->check_launch();
}

// ---------------------------------------------------------------------------
// out = x*sx + coef*(old*so)  (+ segment partials of out^2)
// ---------------------------------------------------------------------------
__global__ void axpby_epi_kernel(const double* __restrict__ x, double* __restrict__ out,
                                 size_t len, size_t rows, size_t chunks, EpiArgs e) {
  if (e.gate && *e.gate == 0) return;
  for (size_t row = (size_t)blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += (size_t)gridDim.y * blockDim.y) {
    const size_t xi = (size_t)blockIdx.x * 32 + threadIdx.x;
    double v = 0.0;
    if (xi < len) {
      const size_t i = row * len + xi;
      double a = x[i];
      if (e.sx) a = a * *e.sx;
      v = epilogue(a, e, i);
      out[i] = v;
    }
    if (e.seg) {
      const double s = tree32(v * v);
      if (threadIdx.x == 0) e.seg[row * chunks + blockIdx.x] = s;
    }
  }
}

void axpby_epi(Ctx* c, const double* x, double* out, RowShape s, const Epi& e) {
  if (s.n() == 0) return;
  dim3 blk(32, 8), grd((unsigned)s.chunks(), row_grid(s.rows));
  axpby_epi_kernel<<<grd, blk, 0, c->stream>>>(x, out, s.len, s.rows, s.chunks(), to_args(e));
  c->count();
  c->check_launch();
}

// ---------------------------------------------------------------------------
// tree-32 levels: one block of 1024 threads folds 32768 consecutive inputs
// (3 levels) into one value; inputs past J are +0 padding.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) reduce3_kernel(const double* __restrict__ in, size_t J,
                                                       double* __restrict__ out, const int* gate) {
  if (gate && *gate == 0) return;
  const double r = block_reduce3(in + (size_t)blockIdx.x * 32768,
                                 J > (size_t)blockIdx.x * 32768 ? J - (size_t)blockIdx.x * 32768 : 0);
  if (threadIdx.x == 0) out[blockIdx.x] = r;
}

// Two tree-32 levels per warp: warp k reduces in[1024k .. 1024k + 1023] (zero padded past J) --
// lane l forms level 1 of group 32k + l serially, the warp's shuffle tree level 2 -- into out[k].
// Whole canonical levels in any grouping give the same bits, so a reduction can take two levels
// per pass with one warp per 1024 values instead of three per pass with one 1024-thread block per
// 32768 (which leaves all but a few SMs idle on small vectors).
__global__ void __launch_bounds__(256) reduce2_kernel(const double* __restrict__ in, size_t J, size_t K,
                                                      double* __restrict__ out, const int* gate) {
  if (gate && *gate == 0) return;
  const size_t k = (size_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (k >= K) return;  // whole warp
  const int lane = threadIdx.x & 31;
  const size_t base = k * 1024 + (size_t)lane * 32;
  double v[32];
  if (base + 32 <= J && !(reinterpret_cast<uintptr_t>(in + base) & 15)) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const double2 q = *reinterpret_cast<const double2*>(in + base + 2 * j);
      v[2 * j] = q.x;
      v[2 * j + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = base + j < J ? in[base + j] : 0.0;
  }
  const double r = tree32(tree32_serial(v));
  if (lane == 0) out[k] = r;
}

void reduce2_pass(Ctx* c, const double* in, size_t J, size_t K, double* out, const int* gate) {
  reduce2_kernel<<<(unsigned)((K + 7) / 8), 256, 0, c->stream>>>(in, J, K, out, gate);
  c->count();
}

size_t reduce_scratch_size(size_t nseg) {
  size_t tot = 0;
  while (nseg > 1024) {
    nseg = (nseg + 1023) / 1024;
    tot += nseg;
  }
  // (covers the block-aligned distributed path's nseg / 32768 level-3 partials too)
  return tot + 1;
}

const double* reduce_segments_to_warp(Ctx* c, const double* seg, size_t nseg, double* scratch, const int* gate,
                                      size_t* J_out) {
  const double* cur = seg;
  size_t J = nseg;
  double* s = scratch;
  while (J > 1024) {
    const size_t K = (J + 1023) / 1024;
    reduce2_kernel<<<(unsigned)((K + 7) / 8), 256, 0, c->stream>>>(cur, J, K, s, gate);
    c->count();
    c->check_launch();
    cur = s;
    s += K;
    J = K;
  }
  *J_out = J;
  return cur;
}

void reduce_segments(Ctx* c, const double* seg, size_t nseg, double* scratch, double* out,
                     const int* gate) {
  const double* cur = seg;
  size_t J = nseg;
  double* s = scratch;
  for (;;) {
    const size_t K = (J + 1023) / 1024;
    double* dst = K == 1 ? out : s;
    reduce2_kernel<<<(unsigned)((K + 7) / 8), 256, 0, c->stream>>>(cur, J, K, dst, gate);
    c->count();
    c->check_launch();
    if (K == 1) break;
    cur = s;
    s += K;
    J = K;
  }
}

// ---------------------------------------------------------------------------
// z-slab decomposition helpers
// ---------------------------------------------------------------------------
void halo_planes(Ctx* c, double* v, size_t plane, long nz_loc, int k) { halo_planes(c, v, plane, nz_loc, k, c->stream); }

void halo_planes(Ctx* c, double* v, size_t plane, long nz_loc, int k, cudaStream_t s) {
  if (!c->sharded() || k <= 0) return;
  require(nz_loc >= k, MLSQR_EDIM, "z slab thinner than the halo it must provide");
  const size_t cnt = plane * (size_t)k;
  TimedRegion th(c, MLSQR_TCLASS_HALO, s);
  c->comm->halo(v, v + (size_t)(nz_loc - k) * plane, v - cnt, v + (size_t)nz_loc * plane, cnt, s);
}

size_t dist_gather_size(Ctx* c, size_t nseg) {
  const size_t P = c->comm ? (size_t)c->comm->size : 1;
  return (nseg % 32768 == 0 ? nseg / 32768 : nseg) * P;
}

void reduce_segments_dist(Ctx* c, const double* seg, size_t nseg, double* scratch, double* gathered,
                          double* out, const int* gate) {
  reduce_segments_dist(c, seg, nseg, scratch, gathered, out, gate, c->sharded());
}

const double* dist_gather_partials(Ctx* c, const double* seg, size_t nseg, double* scratch, double* gathered,
                                   const int* gate, size_t* count) {
  const size_t P = (size_t)c->comm->size;
  if (nseg % 32768 == 0) {
    // this rank's segments are whole 32768-blocks of the global list: levels 1-3 locally
    const size_t K = nseg / 32768;
    reduce3_kernel<<<(unsigned)K, 1024, 0, c->stream>>>(seg, nseg, scratch, gate);
    c->count();
    c->check_launch();
    {
      TimedRegion tc(c, MLSQR_TCLASS_COLL);
      c->comm->allgather(scratch, K, gathered, c->stream);
    }
    *count = K * P;
  } else {
    {
      TimedRegion tc(c, MLSQR_TCLASS_COLL);
      c->comm->allgather(seg, nseg, gathered, c->stream);
    }
    *count = nseg * P;
  }
  return gathered;
}

void reduce_segments_dist(Ctx* c, const double* seg, size_t nseg, double* scratch, double* gathered,
                          double* out, const int* gate, bool dist) {
  if (!dist || !c->data_distributed()) {
    reduce_segments(c, seg, nseg, scratch, out, gate);
    return;
  }
  size_t J = 0;
  const double* g = dist_gather_partials(c, seg, nseg, scratch, gathered, gate, &J);
  reduce_segments(c, g, J, scratch, out, gate);
}

}  // namespace mlsqr_b200
