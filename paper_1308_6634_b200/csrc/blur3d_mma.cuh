// blur3d_mma.cuh -- the fused 3D blur with its x and y passes on the FP64 tensor cores
// (included by blur.cu after blur3d_pipe.cuh, whose TMA / mbarrier helpers it reuses).
//
// Same canonical DEVICE order as blur3d_pipe (per output an ascending fma chain along x, then y,
// then z), but the x and y passes are banded-Toeplitz GEMMs issued as `mma.sync.m8n8k4.f64`:
// tools/dmma_probe.cu shows the FP64 MMA rounds exactly like fma(a3,b3,fma(a2,b2,fma(a1,b1,
// fma(a0,b0,c)))), i.e. an ascending fma chain over k, so a k-loop over the source window in
// ascending order reproduces the scalar chain bit for bit (taps outside an output's band are
// zero: fma(0, x, acc) == acc, up to the sign of an exact zero).
//
//  x pass (plane p+1):  X[r][o] = sum_s In[r][s] T[s][o],   T[s][o] = t[s - o]   (H x 32 outputs)
//  y pass (plane p):    Y[r][o] = sum_u T'[r][u] X[u][o],   T'[r][u] = t[u - r]  (32 x 32 outputs)
// Both use the same per-lane tap fragments tq[q] = t[4q + (lane & 3) - (lane >> 2)] (zero
// outside [0, 2R]).  An m8n8 output tile takes ceil((8 + 2R) / 4) k-steps.
//  z pass: running accumulators; each thread owns the two outputs of its y-pass fragment,
//  Y[r0 + lane/4][o0 + 2 (lane % 4) + {0, 1}], of warp w's tile (r0, o0) = (8 (w / 4), 8 (w % 4)),
//  so every value stays in the registers of the thread that sums it.
//
// Schedule (FP64-pipe and shared-memory bound, tools/dmma_mix_probe.cu: DMMA and DFMA share one
// 64 FMA/cycle/SM pipe; a DMMA holds it 4 SM cycles):
//  * a continuous TMA ring over all of a CTA's items: ring slot r holds input plane q (the r-th of
//    the CTA's plane sequence) and the old-vector tile of output plane q - R - 1, so the phase that
//    runs the x pass of q also emits that output and frees the whole slot.  Slot r is issued right
//    after the barrier that ends the phase consuming slot r - NSTAGE, i.e. NSTAGE - 1 phases ahead
//    of its use, across item boundaries.  One predicated thread issues it (no branch, so no reconvergence
//    barrier in the other warps); the z coordinate of a plane outside the (global) grid is moved
//    out of the tensor map's bounds, so the hardware zero-fills it and no pass tests planes;
//  * phase p loads the y-pass fragments of plane p (published by the last barrier) before it
//    writes the x-pass results of plane p+1, so the y chain and the x chains interleave;
//  * every thread waits on the slot's mbarrier itself (no single-warp poll + broadcast);
//  * the epilogue variants (old vector / |out|^2 partials) are template parameters.
// Shared-memory pitches are chosen for conflict-free 8-byte fragment loads: a half-warp reads
// 4 rows x 4 (x pass) or 4 rows x 4 columns (y pass), so row pitches are = 4 (mod 16) doubles.

template <int R>
struct B3M {
  static constexpr int NT = 2 * R + 1;
  static constexpr int TX = 32, TY = 32;
  static constexpr int THREADS = 256;  // 8 warps x 4 outputs per thread: registers for the z state
  static constexpr int W = TX + 2 * R;
  static constexpr int H = TY + 2 * R;
  static constexpr int XOFF = R & 1;           // TMA boxes start at an even x (see B3P)
  static constexpr int P = ((W + XOFF + 11) / 16) * 16 + 4;  // smallest pitch >= W + XOFF, = 4 mod 16
  static constexpr int KS = (8 + 2 * R + 3) / 4;               // k-steps per 8x8 tile
  static constexpr int MT = (H + 7) / 8;                       // x-pass row tiles
  static constexpr int XTILES = MT * 4;
  static constexpr int XT = (XTILES + 7) / 8;                  // x-pass tiles per warp
  static constexpr int XP = 36;                                // xs pitch (= 4 mod 16)
  static constexpr int SQP = 34;
  static constexpr int OP = 32;
  static constexpr int NSTAGE = 4;
  static constexpr int TREE_WARP = 7;
  // the x pass of the last row tile reads up to 8 * MT - H rows past the tile: keep them inside
  static constexpr int IN_SLOT = ((8 * MT) * P + 15) / 16 * 16;
  static constexpr int OLD_DOUBLES = TX * TY;
  static constexpr int XS_DOUBLES = H * XP;
  static constexpr int SQ_DOUBLES = TY * SQP;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)NSTAGE * IN_SLOT + (size_t)NSTAGE * OLD_DOUBLES +
                                                   2 * XS_DOUBLES + 2 * SQ_DOUBLES) +
                                 NSTAGE * sizeof(unsigned long long);
  static constexpr unsigned IN_BYTES = H * P * 8u;
  static constexpr unsigned OLD_BYTES = TX * TY * 8u;
  static_assert(P % 2 == 0 && P >= W + XOFF && P <= 256, "TMA box width");
  static_assert(XOFF + 24 + 4 * KS <= P, "x-pass window inside the row");
  static_assert(8 * 3 + 4 * KS <= H, "y-pass window inside the x results (even R)");
  static_assert(XT <= 4, "x-pass tiles per warp");
  static_assert(NSTAGE == 4, "ring arithmetic assumes 4 slots");
};

// (not volatile: a pure function of its operands, so independent chains may interleave)
__device__ __forceinline__ void dmma8844(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// thread `on` arms the slot's mbarrier and issues its TMA loads; predicated, no branch
__device__ __forceinline__ void tma_slot_issue(bool on, bool old_on, unsigned long long* bar, unsigned bytes,
                                               double* dst_in, const CUtensorMap* mi, int c0, int c1, int c2,
                                               double* dst_old, const CUtensorMap* mo, int o0, int o1, int o2) {
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.u32 p, %0, 0;\n setp.ne.u32 q, %1, 0;\n"
      " @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
      " @p cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%4], [%5, {%6, %7, %8}], [%2];\n"
      " @q cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%9], [%10, {%11, %12, %13}], [%2];\n"
      "}\n" ::"r"((unsigned)on),
      "r"((unsigned)(on && old_on)), "r"(smem_u32(bar)), "r"(bytes), "r"(smem_u32(dst_in)),
      "l"(reinterpret_cast<unsigned long long>(mi)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(dst_old)),
      "l"(reinterpret_cast<unsigned long long>(mo)), "r"(o0), "r"(o1), "r"(o2)
      : "memory");
}

// a persistent CTA's work item: z chunk item / tiles of column tile item % tiles
struct B3Item {
  int z0, z1, x0, y0, bx;
  __device__ __forceinline__ void set(int item, int tiles, int tiles_x, int zchunk, int nz) {
    const int t = item % tiles;
    z0 = (item / tiles) * zchunk;
    z1 = min(nz, z0 + zchunk);
    bx = t % tiles_x;
    x0 = bx * 32;
    y0 = (t / tiles_x) * 32;
  }
};

// Per item (outputs z0..z1-1) the phases p = zlo - 1 .. zhi + 1 (zlo = z0 - R, zhi = z1 + R - 1) run
// the x pass of plane p+1 and the y / z passes of plane p, and emit output p - R; ring slots carry
// planes zlo .. zhi + 2 (the last two are zero-filled tails).  The first phase's y pass reads the
// previous item's x results: it only feeds accumulators of outputs below z0, which are restarted
// (fma(t[0], y, 0)) before they are used.
template <int R, bool OLD, bool SEG>
__global__ void __launch_bounds__(256, 1) blur3d_mma(const double* __restrict__ in, double* __restrict__ out,
                                                     int nx, int ny, int nz, int tiles_x, int tiles, int zchunk,
                                                     int items, int zoff, int nzg, int zshift, Taps taps, EpiArgs e,
                                                     const __grid_constant__ CUtensorMap map_in,
                                                     const __grid_constant__ CUtensorMap map_old) {
  using C = B3M<R>;
  if (e.gate && *e.gate == 0) return;
  if ((int)blockIdx.x >= items) return;
  extern __shared__ __align__(128) double sm[];
  double* tin = sm;                                       // [NSTAGE][IN_SLOT]  rows of pitch P
  double* olds = tin + C::NSTAGE * C::IN_SLOT;            // [NSTAGE][TY][TX]
  double* xs = olds + C::NSTAGE * C::OLD_DOUBLES;         // [2][H][XP]
  double* sq = xs + 2 * C::XS_DOUBLES;                    // [2][TY][SQP]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sq + 2 * C::SQ_DOUBLES);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const size_t nxy = (size_t)nx * ny;
  const double sx = e.sx ? *e.sx : 1.0;   // x * 1.0 == x: no scale is exact
  const double so = OLD && e.so ? *e.so : 1.0;
  const double coef = OLD ? *e.coef : 0.0;
  const size_t chunks = (size_t)(nx + 31) / 32;
  // tap fragments: t[4q + lane%4 - lane/4], zero outside the band
  double tq[C::KS];
#pragma unroll
  for (int q = 0; q < C::KS; ++q) {
    const int i = 4 * q + (lane & 3) - (lane >> 2);
    tq[q] = (i >= 0 && i <= 2 * R) ? taps.t[i <= R ? i : 2 * R - i] : 0.0;
  }
  // y tiles of warp w: row tile w/2, column tiles 2 (w%2) + {0, 1}; this thread's outputs are
  // row yr, columns yc + {0, 1} and yc + 8 + {0, 1}
  const int yr = 8 * (warp >> 1) + (lane >> 2), yc = 16 * (warp & 1) + 2 * (lane & 3);
  const int yb_off = (8 * (warp >> 1) + (lane & 3)) * C::XP + 16 * (warp & 1) + (lane >> 2);
  // x tiles of warp w: w + 8 i -> row tile w/4 + 2 i, column tile w%4
  const int xa_off = (8 * (warp >> 2) + (lane >> 2)) * C::P + C::XOFF + 8 * (warp & 3) + (lane & 3);
  const int xd_off = (8 * (warp >> 2) + (lane >> 2)) * C::XP + 8 * (warp & 3) + 2 * (lane & 3);
  // tile i of this warp exists (warp-uniform) and this lane's row of it lies inside the H rows
  bool xhas[C::XT], xrow_ok[C::XT];
#pragma unroll
  for (int i = 0; i < C::XT; ++i) {
    xhas[i] = warp + 8 * i < C::XTILES;
    xrow_ok[i] = 8 * ((warp >> 2) + 2 * i) + (lane >> 2) < C::H;
  }

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < C::NSTAGE; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ---- issue cursor (warp 0 only; lane 0's issues take effect)
  int ic_item = blockIdx.x, ic_q = 0;
  unsigned issued = 0;
  B3Item ic;
  auto issue_next = [&]() {
    if (ic_item >= items) return;
    const int zhi = ic.z1 + R - 1;
    const int zo = ic_q - R - 1;  // output whose epilogue runs in the phase consuming this slot
    const bool real = ic_q <= zhi && ic_q + zoff >= 0 && ic_q + zoff < nzg;
    const bool lold = OLD && zo >= ic.z0 && zo < ic.z1;
    const unsigned st = issued & (C::NSTAGE - 1);
    // a plane outside the grid (or a pipeline tail) is loaded from far outside the tensor map:
    // the hardware zero-fills the whole box and still completes IN_BYTES
    const int zc = real ? ic_q + zshift : -(1 << 20);
    tma_slot_issue(lane == 0, lold, bars + st, C::IN_BYTES + (lold ? C::OLD_BYTES : 0u), tin + st * C::IN_SLOT,
                   &map_in, ic.x0 - R - C::XOFF, ic.y0 - R, zc, olds + st * C::OLD_DOUBLES, &map_old, ic.x0,
                   ic.y0, zo);
    ++issued;
    if (++ic_q > zhi + 2) {
      ic_item += gridDim.x;
      if (ic_item < items) {
        ic.set(ic_item, tiles, tiles_x, zchunk, nz);
        ic_q = ic.z0 - R;
      }
    }
  };
  if (warp == 0) {
    ic.set(ic_item, tiles, tiles_x, zchunk, nz);
    ic_q = ic.z0 - R;
#pragma unroll 1
    for (int s = 0; s < C::NSTAGE; ++s) issue_next();
  }

  double acc[4][C::NT];
  unsigned consumed = 0;  // ring slots of earlier items
#pragma unroll 1
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    B3Item it;
    it.set(item, tiles, tiles_x, zchunk, nz);
    const int z0 = it.z0, z1 = it.z1;
    const int zlo = z0 - R, zhi = z1 + R - 1;
    const int gx = it.x0 + yc, gy = it.y0 + yr;
    const bool rowok = gy < ny;
    const bool ok0 = rowok && gx < nx, ok1 = rowok && gx + 1 < nx, ok2 = rowok && gx + 8 < nx,
               ok3 = rowok && gx + 9 < nx;
    double* const obase = out + (size_t)gy * nx + gx;
    const unsigned rb = consumed - (unsigned)zlo;  // ring slot of plane q: rb + q
#pragma unroll 1
    for (int pb = zlo - 1; pb <= zhi + 1; pb += C::NT) {
#pragma unroll
      for (int u = 0; u < C::NT; ++u) {
        const int p = pb + u;
        if (p <= zhi + 1) {  // block-uniform
          const unsigned r1 = rb + (unsigned)(p + 1);  // slot: plane p+1, old tile of output p - R
          const int zo = p - R;
          const bool emit = zo >= z0 && zo < z1;  // block-uniform
          // y-pass B fragments of plane p (x results published by the last barrier)
          const double* xb = xs + (p & 1) * C::XS_DOUBLES + yb_off;
          double yb0[C::KS], yb1[C::KS];
#pragma unroll
          for (int q = 0; q < C::KS; ++q) {
            yb0[q] = xb[4 * q * C::XP];
            yb1[q] = xb[4 * q * C::XP + 8];
          }
          // plane p+1 (and the old tile of output zo) has landed
          mbar_wait(bars + (r1 & 3), (r1 >> 2) & 1u);
          const double* tile = tin + (r1 & 3) * C::IN_SLOT + xa_off;
          double xa[C::XT][C::KS];
#pragma unroll
          for (int i = 0; i < C::XT; ++i)
#pragma unroll
            for (int q = 0; q < C::KS; ++q) xa[i][q] = xhas[i] ? tile[16 * i * C::P + 4 * q] * sx : 0.0;
          double2 o0 = make_double2(0.0, 0.0), o1 = o0;
          if (OLD && emit) {
            const double* po = olds + (r1 & 3) * C::OLD_DOUBLES + yr * C::OP + yc;
            o0 = *reinterpret_cast<const double2*>(po);
            o1 = *reinterpret_cast<const double2*>(po + 8);
          }
          // two y chains (plane p) and XT x chains (plane p+1), interleaved
          double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
          double d[C::XT][2];
#pragma unroll
          for (int i = 0; i < C::XT; ++i) d[i][0] = d[i][1] = 0.0;
#pragma unroll
          for (int q = 0; q < C::KS; ++q) {
            dmma8844(y0, y1, tq[q], yb0[q]);
            dmma8844(y2, y3, tq[q], yb1[q]);
#pragma unroll
            for (int i = 0; i < C::XT; ++i)
              if (xhas[i]) dmma8844(d[i][0], d[i][1], xa[i][q], tq[q]);
          }
          double* xw = xs + ((p + 1) & 1) * C::XS_DOUBLES + xd_off;
#pragma unroll
          for (int i = 0; i < C::XT; ++i)
            if (xhas[i] && xrow_ok[i]) *reinterpret_cast<double2*>(xw + 16 * i * C::XP) = make_double2(d[i][0], d[i][1]);
          // ---- z pass: output zo' = p - R + j takes tap 2R - j
          const double yv[4] = {y0, y1, y2, y3};
#pragma unroll
          for (int j = 0; j < C::NT; ++j) {
            const int s = (u + j) % C::NT;
            const double t = taps.t[(2 * R - j) <= R ? 2 * R - j : j];
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[c][s] = fma(t, yv[c], j == C::NT - 1 ? 0.0 : acc[c][s]);
          }
          if (emit) {
            double v0 = ok0 ? acc[0][u] : 0.0, v1 = ok1 ? acc[1][u] : 0.0;
            double v2 = ok2 ? acc[2][u] : 0.0, v3 = ok3 ? acc[3][u] : 0.0;
            if (OLD) {
              if (ok0) v0 = v0 + coef * (o0.x * so);
              if (ok1) v1 = v1 + coef * (o0.y * so);
              if (ok2) v2 = v2 + coef * (o1.x * so);
              if (ok3) v3 = v3 + coef * (o1.y * so);
            }
            double* orow = obase + (size_t)zo * nxy;
            if (ok1) {
              *reinterpret_cast<double2*>(orow) = make_double2(v0, v1);
            } else if (ok0) {
              orow[0] = v0;
            }
            if (ok3) {
              *reinterpret_cast<double2*>(orow + 8) = make_double2(v2, v3);
            } else if (ok2) {
              orow[8] = v2;
            }
            if (SEG) {
              double* ps = sq + (zo & 1) * C::SQ_DOUBLES + yr * C::SQP + yc;
              *reinterpret_cast<double2*>(ps) = make_double2(v0 * v0, v1 * v1);
              *reinterpret_cast<double2*>(ps + 8) = make_double2(v2 * v2, v3 * v3);
            }
          }
          // canonical segment partials of the plane completed in the previous phase
          if (SEG) {
            const int zt = zo - 1;
            if (warp == C::TREE_WARP && zt >= z0 && zt < z1) {
              const int gyt = it.y0 + lane;
              if (gyt < ny) {
                const double* rr = sq + (zt & 1) * C::SQ_DOUBLES + lane * C::SQP;
                double v[32];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                  const double2 qv = *reinterpret_cast<const double2*>(rr + 2 * j);
                  v[2 * j] = qv.x;
                  v[2 * j + 1] = qv.y;
                }
                e.seg[((size_t)zt * ny + gyt) * chunks + it.bx] = tree32_serial(v);
              }
            }
          }
          __syncthreads();  // x results of p+1 and |out|^2 of zo published; slot r1 is free
          if (warp == 0) issue_next();  // slot r1 + NSTAGE
        }
      }
    }
    consumed += (unsigned)(zhi + 2 - zlo + 1);
  }
}

// MMA variant of launch_b3 (same persistent schedule); false when TMA cannot address the grid
template <int R>
static bool launch_b3m(Ctx* c, const double* in, double* out, int nx, int ny, int nz, const Taps& t,
                       const EpiArgs& a) {
  using C = B3M<R>;
  static std::once_flag attr;
  std::call_once(attr, [] {
    MLSQR_CUDA(cudaFuncSetAttribute(blur3d_mma<R, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    MLSQR_CUDA(cudaFuncSetAttribute(blur3d_mma<R, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    MLSQR_CUDA(cudaFuncSetAttribute(blur3d_mma<R, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    MLSQR_CUDA(cudaFuncSetAttribute(blur3d_mma<R, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  });
  const int tiles_x = (nx + C::TX - 1) / C::TX, tiles_y = (ny + C::TY - 1) / C::TY;
  const int tiles = tiles_x * tiles_y;
  int zck = nz;
  long best = -1;
  for (int zc = 1; zc <= nz; ++zc) {
    const long items = (long)tiles * ((nz + zc - 1) / zc);
    const long g = items < c->sm_count ? items : c->sm_count;
    const long cost = (items + g - 1) / g * (zc + 2 * R + 2);
    if (best < 0 || cost < best) {
      best = cost;
      zck = zc;
    }
  }
  const int items = tiles * ((nz + zck - 1) / zck);
  const unsigned grid = (unsigned)(items < c->sm_count ? items : c->sm_count);
  const bool sh = c->sharded();
  const int zoff = sh ? (int)c->zoff : 0, nzg = sh ? (int)c->nzg : nz;
  const int zshift = sh ? R : 0;
  CUtensorMap mi{}, mo{};
  bool tma = tensor_map3d(&mi, in - (size_t)zshift * nx * ny, nx, ny, nz + 2 * zshift, C::P, C::H);
  if (tma && a.old) tma = tensor_map3d(&mo, a.old, nx, ny, nz, C::TX, C::TY);
  if (!tma) return false;
  auto k = a.old ? (a.seg ? blur3d_mma<R, true, true> : blur3d_mma<R, true, false>)
                 : (a.seg ? blur3d_mma<R, false, true> : blur3d_mma<R, false, false>);
  k<<<grid, C::THREADS, C::SMEM, c->stream>>>(in, out, nx, ny, nz, tiles_x, tiles, zck, items, zoff, nzg, zshift, t, a,
                                              mi, mo);
  c->count();
  return true;
}
