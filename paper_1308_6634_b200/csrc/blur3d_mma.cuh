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
  static constexpr int XWARPS = 4;                 // warpgroup 0: x pass (producer)
  static constexpr int YWARPS = 8;                 // warpgroups 1-2: y / z passes + epilogue (consumers)
  static constexpr int THREADS = 32 * (XWARPS + YWARPS);
  // setmaxnreg split of the launch allocation (384 x 168 = 64512): 128 x 88 + 256 x 208 = 64512 --
  // an increase beyond what the decrease released would block forever
  static constexpr int XREGS = 88, YREGS = 208;
  static constexpr int W = TX + 2 * R;
  static constexpr int H = TY + 2 * R;
  static constexpr int XOFF = R & 1;           // TMA boxes start at an even x (see B3P)
  static constexpr int P = ((W + XOFF + 11) / 16) * 16 + 4;  // smallest pitch >= W + XOFF, = 4 mod 16
  static constexpr int KS = (8 + 2 * R + 3) / 4;               // k-steps per 8x8 tile
  static constexpr int MT = (H + 7) / 8;                       // x-pass row tiles (per x warp)
  static constexpr int XP = 36;                                // xs pitch (= 4 mod 16)
  static constexpr int SQP = 34;
  static constexpr int OP = 32;
  static constexpr int NIN = 4;    // input-plane ring (TMA, x warps)
  static constexpr int NOLD = 4;   // old-tile ring (TMA, y warps)
  static constexpr int NXS = 3;    // x-result ring (x warps -> y warps)
  static constexpr int TREE_WARP = XWARPS + YWARPS - 1;
  // the x pass of the last row tile reads up to 8 * MT - H rows past the tile: keep them inside
  static constexpr int IN_SLOT = ((8 * MT) * P + 15) / 16 * 16;
  static constexpr int OLD_DOUBLES = TX * TY;
  static constexpr int XS_DOUBLES = H * XP;
  static constexpr int SQ_DOUBLES = TY * SQP;
  static constexpr int NBARS = NIN + NOLD + 2 * NXS;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)NIN * IN_SLOT + (size_t)NOLD * OLD_DOUBLES +
                                                   (size_t)NXS * XS_DOUBLES + 2 * SQ_DOUBLES) +
                                 NBARS * sizeof(unsigned long long);
  static constexpr unsigned IN_BYTES = H * P * 8u;
  static constexpr unsigned OLD_BYTES = TX * TY * 8u;
  static_assert(P % 2 == 0 && P >= W + XOFF && P <= 256, "TMA box width");
  static_assert(XOFF + 24 + 4 * KS <= P, "x-pass window inside the row");
  static_assert(8 * 3 + 4 * KS <= H, "y-pass window inside the x results (even R)");
  static_assert(MT <= 6, "x-pass chains per x warp");
  static_assert(XREGS * 32 * XWARPS + YREGS * 32 * YWARPS <= (65536 / THREADS / 8 * 8) * THREADS, "register split");
};

// (not volatile: a pure function of its operands, so independent chains may interleave)
__device__ __forceinline__ void dmma8844(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// thread `on` arms the mbarrier and issues one TMA box load into it; predicated, no branch
__device__ __forceinline__ void tma_issue_pred(bool on, unsigned long long* bar, unsigned bytes, double* dst,
                                               const CUtensorMap* m, int c0, int c1, int c2) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %0, 0;\n"
      " @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %2;\n"
      " @p cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%3], [%4, {%5, %6, %7}], [%1];\n"
      "}\n" ::"r"((unsigned)on),
      "r"(smem_u32(bar)), "r"(bytes), "r"(smem_u32(dst)), "l"(reinterpret_cast<unsigned long long>(m)), "r"(c0),
      "r"(c1), "r"(c2)
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

// Sequential cursor over a CTA's items and, per item, planes [lo(item), hi(item)] (TMA issue order)
struct B3Cursor {
  int item, q, hi;
  B3Item it;
};

// Warp-specialised: warpgroup 0 (4 warps) runs the x pass of every input plane of the CTA's items
// (one column tile per warp, MT row-tile DMMA chains) into a ring of NXS x-result buffers; warpgroups
// 1-2 (8 warps, 4 outputs per thread) run the y pass, the z accumulators and the epilogue of the
// same planes.  The two sides meet only at the x-result ring (full / empty mbarriers), so the x warps
// stream up to NXS planes ahead and the shared FP64 pipe is fed from both sides at once.  Each side
// refills its own TMA ring after a named barrier of that side: input planes (x warp 0), old-vector
// tiles of the outputs (y warp 0).  Per item, planes zlo = z0 - R .. zhi = z1 + R - 1; plane p's y / z
// step emits output p - R when it lies in [z0, z1).  A plane outside the (global) grid is loaded from
// far outside the tensor map: the hardware zero-fills the box.
template <int R, bool OLD, bool SEG>
__global__ void __launch_bounds__(B3M<R>::THREADS, 1)
    blur3d_mma(const double* __restrict__ in, double* __restrict__ out, int nx, int ny, int nz, int tiles_x,
               int tiles, int zchunk, int items, int zoff, int nzg, int zshift, Taps taps, EpiArgs e,
               const __grid_constant__ CUtensorMap map_in, const __grid_constant__ CUtensorMap map_old) {
  using C = B3M<R>;
  if (e.gate && *e.gate == 0) return;
  if ((int)blockIdx.x >= items) return;
  extern __shared__ __align__(128) double sm[];
  double* tin = sm;                                // [NIN][IN_SLOT]  rows of pitch P
  double* olds = tin + C::NIN * C::IN_SLOT;        // [NOLD][TY][TX]
  double* xs = olds + C::NOLD * C::OLD_DOUBLES;    // [NXS][H][XP]
  double* sq = xs + C::NXS * C::XS_DOUBLES;        // [2][TY][SQP]
  unsigned long long* tfull = reinterpret_cast<unsigned long long*>(sq + 2 * C::SQ_DOUBLES);
  unsigned long long* ofull = tfull + C::NIN;
  unsigned long long* xfull = ofull + C::NOLD;
  unsigned long long* xempty = xfull + C::NXS;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < C::NIN; ++s) mbar_init(tfull + s, 1);
#pragma unroll
    for (int s = 0; s < C::NOLD; ++s) mbar_init(ofull + s, 1);
#pragma unroll
    for (int s = 0; s < C::NXS; ++s) {
      mbar_init(xfull + s, 32 * C::XWARPS);
      mbar_init(xempty + s, 32 * C::YWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // tap fragments: t[4q + lane%4 - lane/4], zero outside the band
  double tq[C::KS];
#pragma unroll
  for (int q = 0; q < C::KS; ++q) {
    const int i = 4 * q + (lane & 3) - (lane >> 2);
    tq[q] = (i >= 0 && i <= 2 * R) ? taps.t[i <= R ? i : 2 * R - i] : 0.0;
  }

  if (warp < C::XWARPS) {
    // =================== x warps: X[r][o] for all H rows of column tile `warp`
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::XREGS));
    const double sx = e.sx ? *e.sx : 1.0;  // x * 1.0 == x: no scale is exact
    const int xa_off = (lane >> 2) * C::P + C::XOFF + 8 * warp + (lane & 3);
    const int xd_off = (lane >> 2) * C::XP + 8 * warp + 2 * (lane & 3);
    // input-plane issue cursor (warp 0, lane 0's issues take effect)
    B3Cursor ic;
    unsigned issued = 0;
    auto issue_in = [&]() {
      if (ic.item >= items) return;
      const int q = ic.q;
      const bool real = q + zoff >= 0 && q + zoff < nzg;
      const unsigned st = issued % C::NIN;
      tma_issue_pred(lane == 0, tfull + st, C::IN_BYTES, tin + st * C::IN_SLOT, &map_in, ic.it.x0 - R - C::XOFF,
                     ic.it.y0 - R, real ? q + zshift : -(1 << 20));
      ++issued;
      if (++ic.q > ic.hi) {
        ic.item += gridDim.x;
        if (ic.item < items) {
          ic.it.set(ic.item, tiles, tiles_x, zchunk, nz);
          ic.q = ic.it.z0 - R;
          ic.hi = ic.it.z1 + R - 1;
        }
      }
    };
    if (warp == 0) {
      ic.item = blockIdx.x;
      ic.it.set(ic.item, tiles, tiles_x, zchunk, nz);
      ic.q = ic.it.z0 - R;
      ic.hi = ic.it.z1 + R - 1;
#pragma unroll 1
      for (int s = 0; s < C::NIN; ++s) issue_in();
    }
    unsigned k = 0;  // planes done (input slots and x-result buffers, in sequence)
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      B3Item it;
      it.set(item, tiles, tiles_x, zchunk, nz);
      const int nplanes = it.z1 - it.z0 + 2 * R;
#pragma unroll 1
      for (int j = 0; j < nplanes; ++j, ++k) {
        const unsigned si = k % C::NIN, sb = k % C::NXS;
        mbar_wait(tfull + si, (k / C::NIN) & 1u);
        mbar_wait(xempty + sb, ((k / C::NXS) & 1u) ^ 1u);  // first pass: free
        const double* tile = tin + si * C::IN_SLOT + xa_off;
        double d[C::MT][2];
#pragma unroll
        for (int i = 0; i < C::MT; ++i) d[i][0] = d[i][1] = 0.0;
#pragma unroll
        for (int q = 0; q < C::KS; ++q) {
          double a[C::MT];
#pragma unroll
          for (int i = 0; i < C::MT; ++i) a[i] = tile[8 * i * C::P + 4 * q] * sx;
#pragma unroll
          for (int i = 0; i < C::MT; ++i) dmma8844(d[i][0], d[i][1], a[i], tq[q]);
        }
        double* xw = xs + sb * C::XS_DOUBLES + xd_off;
#pragma unroll
        for (int i = 0; i < C::MT; ++i)
          if (8 * i + (lane >> 2) < C::H) *reinterpret_cast<double2*>(xw + 8 * i * C::XP) = make_double2(d[i][0], d[i][1]);
        mbar_arrive(xfull + sb);
        named_bar(1, 32 * C::XWARPS);  // every x warp is done with input slot si
        if (warp == 0) issue_in();
      }
    }
  } else {
    // =================== y warps: Y = T' X, z accumulators, epilogue, |out|^2 partials
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::YREGS));
    const int yw = warp - C::XWARPS;
    const size_t nxy = (size_t)nx * ny;
    const size_t chunks = (size_t)(nx + 31) / 32;
    const double so = OLD && e.so ? *e.so : 1.0;
    const double coef = OLD ? *e.coef : 0.0;
    // y tiles of warp yw: row tile yw/2, column tiles 2 (yw%2) + {0, 1}; this thread's outputs are
    // row yr, columns yc + {0, 1} and yc + 8 + {0, 1}
    const int yr = 8 * (yw >> 1) + (lane >> 2), yc = 16 * (yw & 1) + 2 * (lane & 3);
    const int yb_off = (8 * (yw >> 1) + (lane & 3)) * C::XP + 16 * (yw & 1) + (lane >> 2);
    // old-tile issue cursor over the CTA's outputs (y warp 0, lane 0)
    B3Cursor oc;
    unsigned oissued = 0;
    auto issue_old = [&]() {
      if (!OLD || oc.item >= items) return;
      const unsigned st = oissued % C::NOLD;
      tma_issue_pred(lane == 0, ofull + st, C::OLD_BYTES, olds + st * C::OLD_DOUBLES, &map_old, oc.it.x0, oc.it.y0,
                     oc.q);
      ++oissued;
      if (++oc.q > oc.hi) {
        oc.item += gridDim.x;
        if (oc.item < items) {
          oc.it.set(oc.item, tiles, tiles_x, zchunk, nz);
          oc.q = oc.it.z0;
          oc.hi = oc.it.z1 - 1;
        }
      }
    };
    if (OLD && yw == 0) {
      oc.item = blockIdx.x;
      oc.it.set(oc.item, tiles, tiles_x, zchunk, nz);
      oc.q = oc.it.z0;
      oc.hi = oc.it.z1 - 1;
#pragma unroll 1
      for (int s = 0; s < C::NOLD; ++s) issue_old();
    }
    double acc[4][C::NT];
    unsigned k = 0;   // planes consumed (x-result buffers)
    unsigned ko = 0;  // outputs emitted (old-tile slots)
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
      auto tree = [&](int zt) {  // canonical segment partials of output plane zt (tree warp)
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
      };
#pragma unroll 1
      for (int pb = zlo; pb <= zhi; pb += C::NT) {
#pragma unroll
        for (int u = 0; u < C::NT; ++u) {
          const int p = pb + u;
          if (p <= zhi) {  // block-uniform
            const unsigned sb = k % C::NXS;
            mbar_wait(xfull + sb, (k / C::NXS) & 1u);
            const double* xb = xs + sb * C::XS_DOUBLES + yb_off;
            double b0[C::KS], b1[C::KS];
#pragma unroll
            for (int q = 0; q < C::KS; ++q) {
              b0[q] = xb[4 * q * C::XP];
              b1[q] = xb[4 * q * C::XP + 8];
            }
            double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
#pragma unroll
            for (int q = 0; q < C::KS; ++q) {
              dmma8844(y0, y1, tq[q], b0[q]);
              dmma8844(y2, y3, tq[q], b1[q]);
            }
            mbar_arrive(xempty + sb);  // the fragments are consumed (the DMMAs read them)
            ++k;
            // ---- z pass: output zo' = p - R + j takes tap 2R - j; slot (u + j) % NT
            const double yv[4] = {y0, y1, y2, y3};
#pragma unroll
            for (int j = 0; j < C::NT; ++j) {
              const int s = (u + j) % C::NT;
              const double t = taps.t[(2 * R - j) <= R ? 2 * R - j : j];
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[c][s] = fma(t, yv[c], j == C::NT - 1 ? 0.0 : acc[c][s]);
            }
            const int zo = p - R;
            const bool emit = zo >= z0;  // (zo <= zhi - R = z1 - 1 always)
            if (emit) {
              double v0 = ok0 ? acc[0][u] : 0.0, v1 = ok1 ? acc[1][u] : 0.0;
              double v2 = ok2 ? acc[2][u] : 0.0, v3 = ok3 ? acc[3][u] : 0.0;
              if (OLD) {
                const unsigned so_ = ko % C::NOLD;
                mbar_wait(ofull + so_, (ko / C::NOLD) & 1u);
                const double* po = olds + so_ * C::OLD_DOUBLES + yr * C::OP + yc;
                const double2 o0 = *reinterpret_cast<const double2*>(po);
                const double2 o1 = *reinterpret_cast<const double2*>(po + 8);
                if (ok0) v0 = v0 + coef * (o0.x * so);
                if (ok1) v1 = v1 + coef * (o0.y * so);
                if (ok2) v2 = v2 + coef * (o1.x * so);
                if (ok3) v3 = v3 + coef * (o1.y * so);
              }
              ++ko;
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
            if (SEG && warp == C::TREE_WARP && zo - 1 >= z0) tree(zo - 1);
            if (SEG || OLD) named_bar(2, 32 * C::YWARPS);  // |out|^2 of zo published; old slot free
            if (OLD && emit && yw == 0) issue_old();
          }
        }
      }
      if (SEG) {  // the last output plane's partials
        if (warp == C::TREE_WARP) tree(z1 - 1);
        named_bar(2, 32 * C::YWARPS);
      }
    }
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
    const long cost = (items + g - 1) / g * (zc + 2 * R);
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
