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

#ifndef MLSQR_B3M_NIN
#define MLSQR_B3M_NIN 4
#endif
#ifndef MLSQR_B3M_NXS
#define MLSQR_B3M_NXS 3
#endif

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
  static constexpr int NIN = MLSQR_B3M_NIN;  // input-plane ring (TMA, x warps)
  static constexpr int NXS = MLSQR_B3M_NXS;  // x-result ring (x warps -> y warps)
  // the x pass of the last row tile reads up to 8 * MT - H rows past the tile: keep them inside
  static constexpr int IN_SLOT = ((8 * MT) * P + 15) / 16 * 16;
  static constexpr int XS_DOUBLES = H * XP;
  static constexpr int NBARS = NIN + 2 * NXS;
  static constexpr size_t SMEM =
      sizeof(double) * ((size_t)NIN * IN_SLOT + (size_t)NXS * XS_DOUBLES) + NBARS * sizeof(unsigned long long);
  static constexpr unsigned IN_BYTES = H * P * 8u;
  static_assert(P % 2 == 0 && P >= W + XOFF && P <= 256, "TMA box width");
  static_assert(XOFF + 24 + 4 * KS <= P, "x-pass window inside the row");
  static_assert(TY == 4 * YWARPS && TX == 32, "y warps: lane = tile column, 4 tile rows per warp");
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
               const __grid_constant__ CUtensorMap map_in) {
  using C = B3M<R>;
  if (e.gate && *e.gate == 0) return;
  if ((int)blockIdx.x >= items) return;
  extern __shared__ __align__(128) double sm[];
  double* tin = sm;                                // [NIN][IN_SLOT]  rows of pitch P
  double* xs = tin + C::NIN * C::IN_SLOT;          // [NXS][H][XP]
  unsigned long long* tfull = reinterpret_cast<unsigned long long*>(xs + C::NXS * C::XS_DOUBLES);
  unsigned long long* xfull = tfull + C::NIN;
  unsigned long long* xempty = xfull + C::NXS;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < C::NIN; ++s) mbar_init(tfull + s, 1);
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
    B3Cursor ic{};
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
    unsigned si = 0, pi = 0, sb = 0, pb = 1;  // ring positions (slot, parity) of the next plane; x-result
                                              // slots start free (parity 1 passes on a fresh barrier)
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      B3Item it;
      it.set(item, tiles, tiles_x, zchunk, nz);
      const int nplanes = it.z1 - it.z0 + 2 * R;
#pragma unroll 1
      for (int j = 0; j < nplanes; ++j) {
        mbar_wait(tfull + si, pi);
        mbar_wait(xempty + sb, pb);
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
        if (++si == C::NIN) {
          si = 0;
          pi ^= 1u;
        }
        if (++sb == C::NXS) {
          sb = 0;
          pb ^= 1u;
        }
        named_bar(1, 32 * C::XWARPS);  // every x warp is done with the input slot
        if (warp == 0) issue_in();
      }
    }
  } else {
    // =================== y warps: lane = tile column, warp yw = tile rows 4 yw .. 4 yw + 3
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::YREGS));
    const int yw = warp - C::XWARPS;
    const size_t nxy = (size_t)nx * ny;
    const size_t chunks = (size_t)(nx + 31) / 32;
    const double so = OLD && e.so ? *e.so : 1.0;
    const double coef = OLD ? *e.coef : 0.0;
    const int r0 = 4 * yw;
    // butterfly row-segment tree (SEG): the row this lane's final value belongs to
    const int trow = r0 + ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1);
    double acc[4][C::NT];
    unsigned sb = 0, ph = 0;  // x-result ring position (slot, parity) of the next plane
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      B3Item it;
      it.set(item, tiles, tiles_x, zchunk, nz);
      const int z0 = it.z0, z1 = it.z1;
      const int zlo = z0 - R, zhi = z1 + R - 1;
      const int gx = it.x0 + lane, gy = it.y0 + r0;
      const bool colok = gx < nx;
      bool ok[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) ok[c] = colok && gy + c < ny;
      // running pointers: the next output plane's row gy, the next old plane to load, the next
      // segment partial of this lane's tree row
      const size_t first = ((size_t)z0 * ny + gy) * nx + gx;
      double* orow = out + first;
      const double* oold = OLD ? e.old + first : nullptr;
      double* segp = SEG ? e.seg + ((size_t)z0 * ny + it.y0 + trow) * chunks + it.bx : nullptr;
      const size_t segstep = (size_t)ny * chunks;
      const bool segok = it.y0 + trow < ny && (lane & 7) == 0;
      // old-vector values of the next output plane, loaded one plane ahead
      double on[4] = {0.0, 0.0, 0.0, 0.0};
      auto load_old = [&]() {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (ok[c]) on[c] = __ldcg(oold + (size_t)c * nx);
        oold += nxy;
      };
      if (OLD) load_old();
#pragma unroll 1
      for (int pb = zlo; pb <= zhi; pb += C::NT) {
#pragma unroll
        for (int u = 0; u < C::NT; ++u) {
          const int p = pb + u;
          if (p <= zhi) {  // warp-uniform
            mbar_wait(xfull + sb, ph);
            const double* xb = xs + sb * C::XS_DOUBLES + r0 * C::XP + lane;
            double b[4 + 2 * R];
#pragma unroll
            for (int j = 0; j < 4 + 2 * R; ++j) b[j] = xb[j * C::XP];
            mbar_arrive(xempty + sb);  // the x results are in registers
            if (++sb == C::NXS) {
              sb = 0;
              ph ^= 1u;
            }
            // ---- y pass: ascending fma chain over the 2R+1 rows of each output
            double yv[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              yv[c] = 0.0;
#pragma unroll
              for (int s = 0; s < C::NT; ++s) yv[c] = fma(taps.t[s <= R ? s : 2 * R - s], b[c + s], yv[c]);
            }
            // ---- z pass: output zo' = p - R + j takes tap 2R - j; slot (u + j) % NT
#pragma unroll
            for (int j = 0; j < C::NT; ++j) {
              const int s = (u + j) % C::NT;
              const double t = taps.t[(2 * R - j) <= R ? 2 * R - j : j];
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[c][s] = fma(t, yv[c], j == C::NT - 1 ? 0.0 : acc[c][s]);
            }
            const int zo = p - R;
            if (zo >= z0) {  // (zo <= zhi - R = z1 - 1 always)
              double v[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) v[c] = ok[c] ? acc[c][u] : 0.0;
              if (OLD) {
                double o[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) o[c] = on[c];
                if (zo + 1 < z1) load_old();
#pragma unroll
                for (int c = 0; c < 4; ++c)
                  if (ok[c]) v[c] = v[c] + coef * (o[c] * so);
              }
#pragma unroll
              for (int c = 0; c < 4; ++c)
                if (ok[c]) orow[(size_t)c * nx] = v[c];
              orow += nxy;
              if (SEG) {
                // tree32 of each row's 32 squares (v[l] += v[l + off], off = 16 .. 1) as a
                // butterfly: every level halves the live values per lane, the pairs are tree32's
                const bool hi16 = lane & 16, hi8 = lane & 8;
                const double q0 = v[0] * v[0], q1 = v[1] * v[1], q2 = v[2] * v[2], q3 = v[3] * v[3];
                // level 16: lanes < 16 keep rows 0 / 2, lanes >= 16 rows 1 / 3
                const double a = (hi16 ? q1 : q0) + __shfl_xor_sync(0xffffffffu, hi16 ? q0 : q1, 16);
                const double c2 = (hi16 ? q3 : q2) + __shfl_xor_sync(0xffffffffu, hi16 ? q2 : q3, 16);
                // level 8: lanes with bit 3 clear keep a's row, the others c2's row
                double w = (hi8 ? c2 : a) + __shfl_xor_sync(0xffffffffu, hi8 ? a : c2, 8);
                w = w + __shfl_xor_sync(0xffffffffu, w, 4);
                w = w + __shfl_xor_sync(0xffffffffu, w, 2);
                w = w + __shfl_xor_sync(0xffffffffu, w, 1);
                if (segok) *segp = w;
                segp += segstep;
              }
            }
          }
        }
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
  CUtensorMap mi{};
  if (!tensor_map3d(&mi, in - (size_t)zshift * nx * ny, nx, ny, nz + 2 * zshift, C::P, C::H)) return false;
  auto k = a.old ? (a.seg ? blur3d_mma<R, true, true> : blur3d_mma<R, true, false>)
                 : (a.seg ? blur3d_mma<R, false, true> : blur3d_mma<R, false, false>);
  k<<<grid, C::THREADS, C::SMEM, c->stream>>>(in, out, nx, ny, nz, tiles_x, tiles, zck, items, zoff, nzg, zshift, t, a,
                                              mi);
  c->count();
  return true;
}
