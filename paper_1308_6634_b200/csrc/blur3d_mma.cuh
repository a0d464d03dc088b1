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
// outside [0, 2R]).  An m8n8 output tile takes ceil((8 + 2R) / 4) k-steps; one DMMA replaces
// 256 DFMAs of which (2R + 1) / (8 + 2R) carry a nonzero tap -- the blur is issue-bound, not
// FP64-throughput-bound, so trading 8x fewer math instructions for that padding pays.
//  z pass: unchanged running accumulators; each thread owns the two outputs of its y-pass
//  fragment, Y[r0 + lane/4][o0 + 2 (lane % 4) + {0, 1}], of warp w's tile (r0, o0) =
//  (8 (w / 4), 8 (w % 4)), so every value stays in the registers of the thread that sums it.
// Shared-memory pitches are chosen for conflict-free 8-byte fragment loads: a half-warp reads
// 4 rows x 4 (x pass) or 4 rows x 4 columns (y pass), so row pitches are = 4 (mod 16) doubles.

template <int R>
struct B3M {
  static constexpr int NT = 2 * R + 1;
  static constexpr int TX = 32, TY = 32;
  static constexpr int THREADS = 512;
  static constexpr int W = TX + 2 * R;
  static constexpr int H = TY + 2 * R;
  static constexpr int XOFF = R & 1;           // TMA boxes start at an even x (see B3P)
  static constexpr int P = ((W + XOFF + 11) / 16) * 16 + 4;  // smallest pitch >= W + XOFF, = 4 mod 16
  static constexpr int KS = (8 + 2 * R + 3) / 4;               // k-steps per 8x8 tile
  static constexpr int MT = (H + 7) / 8;                       // x-pass row tiles
  static constexpr int XPAIRS = MT * 4;
  static constexpr int XP = 36;                                // xs pitch (= 4 mod 16)
  static constexpr int SQP = 34;
  static constexpr int OP = 32;
  static constexpr int NSTAGE = 4;
  static constexpr int TREE_WARP = 15;
  // the x pass of the last row tile reads up to 8 * MT - H rows past the tile: keep them inside
  static constexpr int IN_SLOT = ((H + 8) * P + 15) / 16 * 16;
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
};

// (not volatile: a pure function of its operands, so independent chains may interleave)
__device__ __forceinline__ void dmma8844(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <int R>
__global__ void __launch_bounds__(512, 1) blur3d_mma(const double* __restrict__ in, double* __restrict__ out,
                                                     int nx, int ny, int nz, int tiles_x, int tiles, int zchunk,
                                                     int items, int zoff, int nzg, int zshift, Taps taps, EpiArgs e,
                                                     const __grid_constant__ CUtensorMap map_in,
                                                     const __grid_constant__ CUtensorMap map_old) {
  using C = B3M<R>;
  if (e.gate && *e.gate == 0) return;
  extern __shared__ __align__(128) double sm[];
  double* tin = sm;                                       // [NSTAGE][IN_SLOT]  rows of pitch P
  double* olds = tin + C::NSTAGE * C::IN_SLOT;            // [NSTAGE][TY][TX]
  double* xs = olds + C::NSTAGE * C::OLD_DOUBLES;         // [2][H][XP]
  double* sq = xs + 2 * C::XS_DOUBLES;                    // [2][TY][SQP]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sq + 2 * C::SQ_DOUBLES);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const size_t nxy = (size_t)nx * ny;
  const double sx = e.sx ? *e.sx : 1.0;
  const double so = e.so ? *e.so : 1.0;
  const double coef = e.old ? *e.coef : 0.0;
  const size_t chunks = (size_t)(nx + 31) / 32;
#define TAP(k) taps.t[(k) <= R ? (k) : 2 * R - (k)]
  // tap fragments: t[4q + lane%4 - lane/4], zero outside the band
  double tq[C::KS];
#pragma unroll
  for (int q = 0; q < C::KS; ++q) {
    const int i = 4 * q + (lane & 3) - (lane >> 2);
    tq[q] = (i >= 0 && i <= 2 * R) ? taps.t[i <= R ? i : 2 * R - i] : 0.0;
  }
  double tz[R + 1];  // symmetric z taps t[0..R] in registers (no per-phase constant-bank loads)
#pragma unroll
  for (int k = 0; k <= R; ++k) tz[k] = taps.t[k];
  // this thread's outputs: row yr, columns yc, yc + 1 of the tile (y-pass fragment of warp w)
  const int yr = 8 * (warp >> 2) + (lane >> 2), yc = 8 * (warp & 3) + 2 * (lane & 3);
  static_assert(C::XPAIRS > 16 && C::XPAIRS <= 32, "x-pass pairs: one or two per warp");
  // x-pass fragment offsets of pair `warp` (row tile warp/4, column tile warp%4); pair warp+16
  // is 4 row tiles (32 rows) further down
  const int xa_off = (8 * (warp >> 2) + (lane >> 2)) * C::P + C::XOFF + 8 * (warp & 3) + (lane & 3);
  const int xd_off = (8 * (warp >> 2) + (lane >> 2)) * C::XP + 8 * (warp & 3) + 2 * (lane & 3);
  const bool xrow1_ok = 32 + 8 * (warp >> 2) + (lane >> 2) < C::H;
  // y-pass B fragment offset: row r0 + lane%4, column o0 + lane/4
  const int yb_off = (8 * (warp >> 2) + (lane & 3)) * C::XP + 8 * (warp & 3) + (lane >> 2);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < C::NSTAGE; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double acc[2][C::NT];
  unsigned qbase = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int t = item % tiles;
    const int z0 = (item / tiles) * zchunk;
    const int z1 = min(nz, z0 + zchunk);
    const int bx = t % tiles_x;
    const int x0 = bx * C::TX, y0 = (t / tiles_x) * C::TY;
    const int zlo = z0 - R, zhi = z1 + R - 1;
    const int zin_lo = max(zlo, -zoff), zin_hi = min(zhi, nzg - 1 - zoff);  // in the segment and the grid
    auto inside = [&](int zz) { return zz >= zin_lo && zz <= zin_hi; };
    auto stage = [&](int zz) { return (qbase + (unsigned)(zz - zlo)) & (C::NSTAGE - 1); };
    auto parity = [&](int zz) { return ((qbase + (unsigned)(zz - zlo)) >> 2) & 1u; };
    auto issue = [&](int zz) {  // called by thread 0 only
      if (zz > zhi) return;
      {
        const int st = stage(zz);
        const int zo = zz - R;
        const bool lin = inside(zz);
        const bool lold = e.old && zo >= z0 && zo < z1;
        mbar_arrive_expect(bars + st, (lin ? C::IN_BYTES : 0u) + (lold ? C::OLD_BYTES : 0u));
        if (lin) tma_load3d(tin + st * C::IN_SLOT, &map_in, x0 - R - C::XOFF, y0 - R, zz + zshift, bars + st);
        if (lold) tma_load3d(olds + st * C::OLD_DOUBLES, &map_old, x0, y0, zo, bars + st);
      }
    };

    const int gx = x0 + yc, gy = y0 + yr;
    const bool ok0 = gx < nx && gy < ny, ok1 = gx + 1 < nx && gy < ny;
    double* const obase = out + (size_t)gy * nx + gx;
    __syncthreads();
    if (tid == 0) {
      issue(zlo);
      issue(zlo + 1);
    }
    for (int pb = zlo - 1; pb <= zhi + 1; pb += C::NT) {
#pragma unroll
      for (int u = 0; u < C::NT; ++u) {
        const int p = pb + u;
        if (p <= zhi + 1) {  // block-uniform
          // one warp polls the TMA barrier; the CTA barrier then publishes the landed plane
          if (warp == 0 && p + 1 <= zhi) mbar_wait(bars + stage(p + 1), parity(p + 1));
          __syncthreads();
          if (tid == 0) issue(p + 3);
          // ---- x pass of plane p+1 on the tensor cores: 4 * MT tiles over 16 warps
          const int xz = p + 1;
          if (inside(xz)) {
            const double* tile = tin + stage(xz) * C::IN_SLOT + xa_off;
            double* xw = xs + ((xz - zlo) & 1) * C::XS_DOUBLES + xd_off;
            // pairs warp and warp + 16 (row tile (warp >> 2) + 4, same column tile): two independent
            // DMMA chains, interleaved; x * 1.0 == x when there is no scale
            if (warp + 16 < C::XPAIRS) {  // warp-uniform
              const double* arow1 = tile + 32 * C::P;
              double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
              for (int q = 0; q < C::KS; ++q) {
                dmma8844(d0, d1, tile[4 * q] * sx, tq[q]);
                dmma8844(e0, e1, arow1[4 * q] * sx, tq[q]);
              }
              *reinterpret_cast<double2*>(xw) = make_double2(d0, d1);
              if (xrow1_ok) *reinterpret_cast<double2*>(xw + 32 * C::XP) = make_double2(e0, e1);
            } else {
              double d0 = 0.0, d1 = 0.0;
#pragma unroll
              for (int q = 0; q < C::KS; ++q) dmma8844(d0, d1, tile[4 * q] * sx, tq[q]);
              *reinterpret_cast<double2*>(xw) = make_double2(d0, d1);
            }
          }
          if (p >= zlo && p <= zhi) {
            // ---- y pass of plane p (tile (8 (w/4), 8 (w%4)) of warp w) on the tensor cores
            double yv0 = 0.0, yv1 = 0.0;
            if (inside(p)) {
              const double* xb = xs + ((p - zlo) & 1) * C::XS_DOUBLES + yb_off;
#pragma unroll
              for (int q = 0; q < C::KS; ++q) dmma8844(yv0, yv1, tq[q], xb[4 * q * C::XP]);
            }
            // ---- z pass: output zo' = p - R + j takes tap 2R - j (taps from registers)
#pragma unroll
            for (int j = 0; j < C::NT; ++j) {
              const int s = (u + j) % C::NT;
              const double t = tz[(2 * R - j) <= R ? 2 * R - j : j];
              acc[0][s] = fma(t, yv0, j == C::NT - 1 ? 0.0 : acc[0][s]);
              acc[1][s] = fma(t, yv1, j == C::NT - 1 ? 0.0 : acc[1][s]);
            }
            const int zo = p - R;
            if (zo >= z0 && zo < z1) {
              double v0 = ok0 ? acc[0][u] : 0.0, v1 = ok1 ? acc[1][u] : 0.0;
              if (e.old) {
                const double2 o = *reinterpret_cast<const double2*>(olds + stage(p) * C::OLD_DOUBLES + yr * C::OP + yc);
                double o0 = o.x, o1 = o.y;
                if (e.so) {
                  o0 = o0 * so;
                  o1 = o1 * so;
                }
                if (ok0) v0 = v0 + coef * o0;
                if (ok1) v1 = v1 + coef * o1;
              }
              double* orow = obase + (size_t)zo * nxy;
              if (ok1) {
                *reinterpret_cast<double2*>(orow) = make_double2(v0, v1);
              } else if (ok0) {
                orow[0] = v0;
              }
              if (e.seg)
                *reinterpret_cast<double2*>(sq + ((zo - z0) & 1) * C::SQ_DOUBLES + yr * C::SQP + yc) =
                    make_double2(v0 * v0, v1 * v1);
            }
          }
          // canonical segment partials of the plane completed in the previous phase
          const int zt = p - R - 1;
          if (e.seg && warp == C::TREE_WARP && zt >= z0 && zt < z1) {
            const int gyt = y0 + lane;
            if (gyt < ny) {
              const double* r = sq + ((zt - z0) & 1) * C::SQ_DOUBLES + lane * C::SQP;
              double v[32];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const double2 q = *reinterpret_cast<const double2*>(r + 2 * j);
                v[2 * j] = q.x;
                v[2 * j + 1] = q.y;
              }
              e.seg[((size_t)zt * ny + gyt) * chunks + bx] = tree32_serial(v);
            }
          }
        }
      }
    }
    qbase += (unsigned)(zhi - zlo + 1);
  }
#undef TAP
}

// MMA variant of launch_b3 (same persistent schedule); false when TMA cannot address the grid
template <int R>
static bool launch_b3m(Ctx* c, const double* in, double* out, int nx, int ny, int nz, const Taps& t,
                       const EpiArgs& a) {
  using C = B3M<R>;
  static std::once_flag attr;
  std::call_once(attr, [] {
    MLSQR_CUDA(cudaFuncSetAttribute(blur3d_mma<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
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
  blur3d_mma<R><<<grid, C::THREADS, C::SMEM, c->stream>>>(in, out, nx, ny, nz, tiles_x, tiles, zck, items, zoff, nzg,
                                                          zshift, t, a, mi, mo);
  c->count();
  return true;
}
