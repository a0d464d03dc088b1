// blur3d_mma.cuh -- the fused 3D blur: x pass on the FP64 tensor cores, y / z passes and the
// LSQR epilogue on the FP64 CUDA cores (included by blur.cu after blur3d_pipe.cuh, whose TMA /
// mbarrier helpers it reuses).
//
// Canonical DEVICE order (the oracle's): per output an ascending fma chain along x, then y, then z.
//  x pass: banded-Toeplitz GEMM X[r][o] = sum_s In[r][s] T[s][o], T[s][o] = t[s - o], issued as
//    `mma.sync.m8n8k4.f64` with tap fragments tq[q] = t[4q + lane%4 - lane/4] (zero outside [0, 2R]);
//    tools/dmma_probe.cu shows the FP64 MMA rounds exactly like an ascending fma chain over k, so
//    the k-loop over the source window reproduces the scalar chain bit for bit.
//  y pass: 2R+1-long DFMA chains down a column (lane = tile column), the DMMA's band would waste a
//    third of the pipe there;  z pass: 2R+1 running accumulators per output (independent DFMAs).
//
// Warp roles (tools/dmma_mix_probe.cu: DMMA and DFMA share one 64 FMA/cycle/SM pipe, so the
// roles are sized to keep it fed from every SMSP):
//  * x warps, XG groups of four taking alternate planes: TMA ring of input planes (TMA zero-fills
//    the box outside the grid; a plane outside the global grid is loaded from far outside the
//    tensor map), DMMA x pass into an x-result ring (full / empty mbarriers).  Group warp w does
//    row tiles MTH (w / 2) + {0 .. MTH-1} and column tiles 2 (w % 2) + {0, 1}, whose A fragments
//    overlap in KS - 2 of KS k-steps;
//  * y warps (4 tile rows each): y pass and z accumulators; each z-complete output plane goes to an
//    output ring;
//  * epilogue warps (8 tile rows each): out = v + coef (old so) with the old vector streamed into
//    each thread's own shared-memory slots by cp.async three planes ahead, the stores, and the
//    |out|^2 row-segment partials as a register butterfly (tree32's pairs, no shared memory).
// Only the rings couple the roles, so a role waits for another only when a ring runs empty / full.
// Shared-memory pitches are chosen for conflict-free 8-byte fragment loads: a half-warp reads
// 4 rows x 4 doubles (x pass), so the input row pitch is = 4 (mod 16) doubles.

#ifndef MLSQR_B3M_XG
#define MLSQR_B3M_XG 2
#endif
#ifndef MLSQR_B3M_NIN
#define MLSQR_B3M_NIN 4
#endif
#ifndef MLSQR_B3M_NXS
#define MLSQR_B3M_NXS 4
#endif

template <int R>
struct B3M {
  static constexpr int NT = 2 * R + 1;
  static constexpr int TX = 32, TY = 32;
  static constexpr int XG = MLSQR_B3M_XG;          // x groups (4 warps each) taking alternate planes
  static constexpr int XWARPS = 4 * XG;            // x pass
  static constexpr int YR = 4;                     // tile rows per y warp (outputs per y thread)
  static constexpr int YWARPS = TY / YR;           // y and z passes
  static constexpr int ER = 8;                     // tile rows per epilogue warp
  static constexpr int EWARPS = TY / ER;           // epilogue: old vector, stores, |out|^2 segment trees
  static constexpr int THREADS = 32 * (XWARPS + YWARPS + EWARPS);
  // setmaxnreg split of the launch allocation (XG 1: 512 x 128 = 65536, XG 2: 640 x 96 = 61440):
  // an increase beyond what the decreases released would block forever
  static constexpr int XREGS = XG == 1 ? 88 : 80, EREGS = XG == 1 ? 80 : 72;
  static constexpr int YREGS = XG == 1 ? 168 : 120;
  static constexpr int W = TX + 2 * R;
  static constexpr int H = TY + 2 * R;
  static constexpr int XOFF = R & 1;           // TMA boxes start at an even x (see B3P)
  static constexpr int P = ((W + XOFF + 11) / 16) * 16 + 4;  // smallest pitch >= W + XOFF, = 4 mod 16
  static constexpr int KS = (8 + 2 * R + 3) / 4;               // k-steps per 8x8 tile
  static constexpr int MT = (H + 7) / 8;                       // x-pass row tiles (per x warp)
  static constexpr int XP = 40;  // xs pitch: = 8 mod 16, so the x warps' STS.128 rows land on disjoint banks
  static constexpr int NIN = MLSQR_B3M_NIN;  // input-plane ring (TMA, x warps)
  static constexpr int NXS = MLSQR_B3M_NXS;  // x-result ring (x warps -> y warps)
  // the x pass of the last row tile reads up to 8 * MT - H rows past the tile: keep them inside
  static constexpr int IN_SLOT = ((8 * MT) * P + 15) / 16 * 16;
  static constexpr int XS_DOUBLES = H * XP;
  static constexpr int NV = 4;                                 // z-complete output ring (y -> epilogue warps)
  static constexpr int V_DOUBLES = TY * TX;
  static constexpr int NOLD = 4;  // epilogue threads' own old-vector slots (cp.async, NOLD - 1 planes ahead)
  static constexpr int OLD_DOUBLES = NOLD * TY * TX;
  static constexpr int NBARS = NIN + 2 * NXS + 2 * NV;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)NIN * IN_SLOT + (size_t)NXS * XS_DOUBLES +
                                                   (size_t)NV * V_DOUBLES + OLD_DOUBLES) +
                                 NBARS * sizeof(unsigned long long);
  static constexpr unsigned IN_BYTES = H * P * 8u;
  static_assert(P % 2 == 0 && P >= W + XOFF && P <= 256, "TMA box width");
  static_assert(XOFF + 24 + 4 * KS <= P, "x-pass window inside the row");
  static_assert((XG == 1 || (XG == 2 && NIN % 2 == 0 && NXS % 2 == 0)) && TX == 32 && TY == 32, "roles");
  static_assert(MT <= 6 && KS + 2 <= 7, "x-pass chains and A fragments per x warp");
  static_assert(XREGS * 32 * XWARPS + YREGS * 32 * YWARPS + EREGS * 32 * EWARPS <= (65536 / THREADS / 8 * 8) * THREADS,
                "register split");
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
  // outputs z0 .. z1-1 of the range zb .. ze-1 (ze - zb planes split into zchunk-plane items)
  __device__ __forceinline__ void set(int item, int tiles, int tiles_x, int zchunk, int zb, int ze) {
    const int t = item % tiles;
    z0 = zb + (item / tiles) * zchunk;
    z1 = min(ze, z0 + zchunk);
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
    blur3d_mma(const double* __restrict__ in, double* __restrict__ out, int nx, int ny, int zb, int ze, int tiles_x,
               int tiles, int zchunk, int items, int zoff, int nzg, int zshift, Taps taps, EpiArgs e,
               const __grid_constant__ CUtensorMap map_in) {
  using C = B3M<R>;
  if (e.gate && *e.gate == 0) return;
  if ((int)blockIdx.x >= items) return;
  extern __shared__ __align__(128) double sm[];
  double* tin = sm;                                // [NIN][IN_SLOT]  rows of pitch P
  double* xs = tin + C::NIN * C::IN_SLOT;          // [NXS][H][XP]
  double* vs = xs + C::NXS * C::XS_DOUBLES;        // [NV][TY][TX]  z-complete outputs
  double* olds = vs + C::NV * C::V_DOUBLES;        // [NOLD][ER][EWARPS * 32]  old vector, per thread
  unsigned long long* tfull = reinterpret_cast<unsigned long long*>(olds + C::OLD_DOUBLES);
  unsigned long long* xfull = tfull + C::NIN;
  unsigned long long* xempty = xfull + C::NXS;
  unsigned long long* vfull = xempty + C::NXS;
  unsigned long long* vempty = vfull + C::NV;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < C::NIN; ++s) mbar_init(tfull + s, 1);
#pragma unroll
    for (int s = 0; s < C::NXS; ++s) {
      mbar_init(xfull + s, 128);  // one x group writes a plane
      mbar_init(xempty + s, 32 * C::YWARPS);
    }
#pragma unroll
    for (int s = 0; s < C::NV; ++s) {
      mbar_init(vfull + s, 32 * C::YWARPS);
      mbar_init(vempty + s, 32 * C::EWARPS);
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
    // x warp w: row tiles MTH (w / 2) + {0 .. MTH-1}, column tiles 2 (w % 2) + {0, 1}; the two column
    // tiles share the A fragments of KS - 2 of their KS k-steps (KP = KS + 2 loads per row tile)
    constexpr int MTH = (C::MT + 1) / 2, KP = C::KS + 2;
    const int grp = warp >> 2, role = warp & 3;  // x group, and the warp's tiles within the plane
    const int xg = role >> 1, xh = role & 1;
    const int xa_off = (8 * MTH * xg + (lane >> 2)) * C::P + C::XOFF + 16 * xh + (lane & 3);
    const int xd_off = (8 * MTH * xg + (lane >> 2)) * C::XP + 16 * xh + 2 * (lane & 3);
    // the CTA's plane sequence (all items, planes z0 - R .. z1 + R - 1 each); x group grp runs the
    // planes k = grp (mod XG), its role-0 warp refills their input slots (lane 0's issues take effect)
    B3Cursor ic{};
    auto advance = [&]() {
      if (ic.item >= items) return;
      if (++ic.q > ic.hi) {
        ic.item += gridDim.x;
        if (ic.item < items) {
          ic.it.set(ic.item, tiles, tiles_x, zchunk, zb, ze);
          ic.q = ic.it.z0 - R;
          ic.hi = ic.it.z1 + R - 1;
        }
      }
    };
    auto issue_in = [&](unsigned kq) {  // the cursor's plane, sequence index kq
      if (ic.item >= items) return;
      const int q = ic.q;
      const bool real = q + zoff >= 0 && q + zoff < nzg;
      const unsigned st = kq % C::NIN;
      tma_issue_pred(lane == 0, tfull + st, C::IN_BYTES, tin + st * C::IN_SLOT, &map_in, ic.it.x0 - R - C::XOFF,
                     ic.it.y0 - R, real ? q + zshift : -(1 << 20));
    };
    unsigned kis = grp;  // sequence index of the next plane this group issues
    if (role == 0) {
      ic.item = blockIdx.x;
      ic.it.set(ic.item, tiles, tiles_x, zchunk, zb, ze);
      ic.q = ic.it.z0 - R;
      ic.hi = ic.it.z1 + R - 1;
      if (C::XG == 2 && grp) advance();
#pragma unroll 1
      for (int s = 0; s < C::NIN / C::XG; ++s) {
        issue_in(kis);
        kis += C::XG;
#pragma unroll
        for (int g = 0; g < C::XG; ++g) advance();
      }
    }
    unsigned k = 0;  // sequence index of the current plane
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      B3Item it;
      it.set(item, tiles, tiles_x, zchunk, zb, ze);
      const int nplanes = it.z1 - it.z0 + 2 * R;
#pragma unroll 1
      for (int j = 0; j < nplanes; ++j, ++k) {
        if (C::XG == 2 && (int)(k & 1u) != grp) continue;
        const unsigned si = k % C::NIN, sb = k % C::NXS;
        mbar_wait(tfull + si, (k / C::NIN) & 1u);
        mbar_wait(xempty + sb, ((k / C::NXS) & 1u) ^ 1u);  // x-result slots start free
        const double* tile = tin + si * C::IN_SLOT + xa_off;
        auto live = [&](int i) { return C::MT % 2 == 0 || MTH * xg + i < C::MT; };  // warp-uniform
        double a[MTH][KP];
#pragma unroll
        for (int i = 0; i < MTH; ++i)
          if (live(i)) {
#pragma unroll
            for (int q = 0; q < KP; ++q) a[i][q] = tile[8 * i * C::P + 4 * q] * sx;
          }
        double d[MTH][2][2];
#pragma unroll
        for (int i = 0; i < MTH; ++i) d[i][0][0] = d[i][0][1] = d[i][1][0] = d[i][1][1] = 0.0;
#pragma unroll
        for (int q = 0; q < C::KS; ++q)
#pragma unroll
          for (int i = 0; i < MTH; ++i)
            if (live(i)) {
              dmma8844(d[i][0][0], d[i][0][1], a[i][q], tq[q]);
              dmma8844(d[i][1][0], d[i][1][1], a[i][q + 2], tq[q]);
            }
        double* xw = xs + sb * C::XS_DOUBLES + xd_off;
#pragma unroll
        for (int i = 0; i < MTH; ++i)
          if (live(i) && 8 * (MTH * xg + i) + (lane >> 2) < C::H) {
            *reinterpret_cast<double2*>(xw + 8 * i * C::XP) = make_double2(d[i][0][0], d[i][0][1]);
            *reinterpret_cast<double2*>(xw + 8 * i * C::XP + 8) = make_double2(d[i][1][0], d[i][1][1]);
          }
        mbar_arrive(xfull + sb);
        named_bar(1 + grp, 128);  // the group's four warps are done with the input slot
        if (role == 0) {
          issue_in(kis);
          kis += C::XG;
#pragma unroll
          for (int g = 0; g < C::XG; ++g) advance();
        }
      }
    }
  } else if (warp < C::XWARPS + C::YWARPS) {
    // =================== y warps: lane = tile column, warp yw = tile rows 4 yw .. 4 yw + 3
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::YREGS));
    constexpr int YR = C::YR;
    const int r0 = YR * (warp - C::XWARPS);
    double acc[YR][C::NT];
    unsigned sb = 0, ph = 0;  // x-result ring position (slot, parity) of the next plane
    unsigned vb = 0, vp = 1;  // output ring position of the next output plane (slots start free)
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      B3Item it;
      it.set(item, tiles, tiles_x, zchunk, zb, ze);
      const int z0 = it.z0, z1 = it.z1;
      const int zlo = z0 - R, zhi = z1 + R - 1;
#pragma unroll 1
      for (int pb = zlo; pb <= zhi; pb += C::NT) {
#pragma unroll
        for (int u = 0; u < C::NT; ++u) {
          const int p = pb + u;
          if (p <= zhi) {  // warp-uniform
            mbar_wait(xfull + sb, ph);
            const double* xb = xs + sb * C::XS_DOUBLES + r0 * C::XP + lane;
            double b[YR + 2 * R];
#pragma unroll
            for (int j = 0; j < YR + 2 * R; ++j) b[j] = xb[j * C::XP];
            mbar_arrive(xempty + sb);  // the x results are in registers
            if (++sb == C::NXS) {
              sb = 0;
              ph ^= 1u;
            }
            // ---- y pass: ascending fma chain over the 2R+1 rows of each output
            double yv[YR];
#pragma unroll
            for (int c = 0; c < YR; ++c) {
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
              for (int c = 0; c < YR; ++c) acc[c][s] = fma(t, yv[c], j == C::NT - 1 ? 0.0 : acc[c][s]);
            }
            if (p - R >= z0) {  // output p - R is complete (p - R <= z1 - 1 always): hand it over
              mbar_wait(vempty + vb, vp);
              double* vw = vs + vb * C::V_DOUBLES + r0 * C::TX + lane;
#pragma unroll
              for (int c = 0; c < YR; ++c) vw[c * C::TX] = acc[c][u];
              mbar_arrive(vfull + vb);
              if (++vb == C::NV) {
                vb = 0;
                vp ^= 1u;
              }
            }
          }
        }
      }
    }
  } else {
    // =================== epilogue warps: lane = tile column, warp ew = tile rows 8 ew .. 8 ew + 7
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::EREGS));
    constexpr int ER = C::ER;
    const int r0 = ER * (warp - C::XWARPS - C::YWARPS);
    const size_t nxy = (size_t)nx * ny;
    const size_t chunks = (size_t)(nx + 31) / 32;
    const double so = OLD && e.so ? *e.so : 1.0;
    const double coef = OLD ? *e.coef : 0.0;
    // butterfly row-segment tree (SEG): lane 4m ends with the sum of row r0 + trow, m = lane / 4
    const int m = lane >> 2;
    const int trow = r0 + 2 * (2 * (m & 1) + ((m >> 1) & 1)) + ((m >> 2) & 1);
    unsigned vb = 0, vp = 0;  // output ring position of the next output plane
    constexpr int ET = 32 * C::EWARPS;
    double* const omine = olds + (tid - 32 * (C::XWARPS + C::YWARPS));  // slot s, row c: [(s ER + c) ET]
    unsigned os = 0;  // old slot of the next output plane
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      B3Item it;
      it.set(item, tiles, tiles_x, zchunk, zb, ze);
      const int z0 = it.z0, z1 = it.z1;
      const int gx = it.x0 + lane, gy = it.y0 + r0;
      const bool colok = gx < nx;
      bool ok[ER];
#pragma unroll
      for (int c = 0; c < ER; ++c) ok[c] = colok && gy + c < ny;
      // running pointers: the next output plane's row gy, the next old plane to load, the next
      // segment partial of this lane's tree row
      const size_t first = ((size_t)z0 * ny + gy) * nx + gx;
      double* orow = out + first;
      const double* oold = OLD ? e.old + first : nullptr;
      double* segp = SEG ? e.seg + ((size_t)z0 * ny + it.y0 + trow) * chunks + it.bx : nullptr;
      const size_t segstep = (size_t)ny * chunks;
      const bool segok = it.y0 + trow < ny && (lane & 3) == 0;
      // old-vector values NOLD - 1 planes ahead: cp.async into this thread's own slots, one commit
      // group per output plane (empty past z1), so wait_group<NOLD - 1> completes the current one
      int zl = z0;
      const unsigned os0 = os;
      auto load_old = [&]() {
        if (zl < z1) {
          double* dst = omine + ((os0 + (unsigned)(zl - z0)) % C::NOLD) * ER * ET;
#pragma unroll
          for (int c = 0; c < ER; ++c)
            if (ok[c]) cp_async8(dst + c * ET, oold + (size_t)c * nx, true);
          oold += nxy;
        }
        ++zl;
        cp_async_commit();
      };
      if (OLD)
#pragma unroll
        for (int j = 0; j < C::NOLD - 1; ++j) load_old();
#pragma unroll 1
      for (int zo = z0; zo < z1; ++zo) {
        double o[ER];
        if (OLD) {
          load_old();  // plane zo + NOLD - 1
          cp_async_wait<C::NOLD - 1>();
          const double* src = omine + (os % C::NOLD) * ER * ET;
#pragma unroll
          for (int c = 0; c < ER; ++c) o[c] = src[c * ET];
          ++os;
        }
        mbar_wait(vfull + vb, vp);
        const double* vr = vs + vb * C::V_DOUBLES + r0 * C::TX + lane;
        double v[ER];
#pragma unroll
        for (int c = 0; c < ER; ++c) v[c] = vr[c * C::TX];
        mbar_arrive(vempty + vb);
        if (++vb == C::NV) {
          vb = 0;
          vp ^= 1u;
        }
#pragma unroll
        for (int c = 0; c < ER; ++c) {
          v[c] = ok[c] ? v[c] : 0.0;
          if (OLD && ok[c]) v[c] = v[c] + coef * (o[c] * so);
        }
#pragma unroll
        for (int c = 0; c < ER; ++c)
          if (ok[c]) orow[(size_t)c * nx] = v[c];
        orow += nxy;
        if (SEG) {
          // tree32 of each row's 32 squares (v[l] += v[l + off], off = 16 .. 1) as a butterfly:
          // every level pairs tree32's elements and halves the live values per lane
          const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
          double q[ER];
#pragma unroll
          for (int c = 0; c < ER; ++c) q[c] = v[c] * v[c];
          // level 16: lanes < 16 keep the even rows, lanes >= 16 the odd ones
          double a[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            a[j] = (h16 ? q[2 * j + 1] : q[2 * j]) + __shfl_xor_sync(0xffffffffu, h16 ? q[2 * j] : q[2 * j + 1], 16);
          // level 8: bit 3 clear keeps a[0] / a[2], set keeps a[1] / a[3]
          double b2[2];
#pragma unroll
          for (int j = 0; j < 2; ++j)
            b2[j] = (h8 ? a[2 * j + 1] : a[2 * j]) + __shfl_xor_sync(0xffffffffu, h8 ? a[2 * j] : a[2 * j + 1], 8);
          // level 4: bit 2 clear keeps b2[0], set keeps b2[1]
          double w = (h4 ? b2[1] : b2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? b2[0] : b2[1], 4);
          w = w + __shfl_xor_sync(0xffffffffu, w, 2);
          w = w + __shfl_xor_sync(0xffffffffu, w, 1);
          if (segok) *segp = w;
          segp += segstep;
        }
      }
    }
  }
}

// MMA variant of launch_b3 (same persistent schedule); false when TMA cannot address the grid.
// Outputs zb .. ze-1 of the (local) nz-plane grid; inputs zb-R .. ze+R-1 (ghost planes past the slab)
template <int R>
static bool launch_b3m_range(Ctx* c, const double* in, double* out, int nx, int ny, int nz, int zb, int ze,
                             const Taps& t, const EpiArgs& a);
template <int R>
static bool launch_b3m(Ctx* c, const double* in, double* out, int nx, int ny, int nz, const Taps& t,
                       const EpiArgs& a) {
  return launch_b3m_range<R>(c, in, out, nx, ny, nz, 0, nz, t, a);
}
template <int R>
static bool launch_b3m_range(Ctx* c, const double* in, double* out, int nx, int ny, int nz, int zb, int ze,
                             const Taps& t, const EpiArgs& a) {
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
  const int nzr = ze - zb;
  int zck = nzr;
  long best = -1;
  for (int zc = 1; zc <= nzr; ++zc) {
    const long items = (long)tiles * ((nzr + zc - 1) / zc);
    const long g = items < c->sm_count ? items : c->sm_count;
    const long cost = (items + g - 1) / g * (zc + 2 * R);
    if (best < 0 || cost < best) {
      best = cost;
      zck = zc;
    }
  }
  const int items = tiles * ((nzr + zck - 1) / zck);
  const unsigned grid = (unsigned)(items < c->sm_count ? items : c->sm_count);
  const bool sh = c->sharded();
  const int zoff = sh ? (int)c->zoff : 0, nzg = sh ? (int)c->nzg : nz;
  const int zshift = sh ? R : 0;
  CUtensorMap mi{};
  if (!tensor_map3d(&mi, in - (size_t)zshift * nx * ny, nx, ny, nz + 2 * zshift, C::P, C::H)) return false;
  auto k = a.old ? (a.seg ? blur3d_mma<R, true, true> : blur3d_mma<R, true, false>)
                 : (a.seg ? blur3d_mma<R, false, true> : blur3d_mma<R, false, false>);
  k<<<grid, C::THREADS, C::SMEM, c->stream>>>(in, out, nx, ny, zb, ze, tiles_x, tiles, zck, items, zoff, nzg, zshift, t, a,
                                              mi);
  c->count();
  return true;
}
