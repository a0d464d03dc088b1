// blur3d_pipe.cuh -- the default fused 3D blur (included by blur.cu).
//
// Per output: fma(t[0], x[i-R], 0), fma(t[1], x[i-R+1], .) ... along x, then y, then z
// (the oracle's DEVICE order), scheduled for the issue-bound regime of the FP64 stencil:
//  * TMA: one thread loads each input plane tile (a (32+2R) x P box; the
//    hardware zero-fills everything outside the grid, so no per-element
//    predicates) and the old-vector tile into a 4-stage ring completed by
//    mbarriers.  Falls back to 8-byte cp.async when a tensor map is impossible
//    (odd nx, misaligned vector);
//  * phase p runs the x pass of plane p+1 next to the y pass of plane p (x-pass
//    results double-buffered), so one __syncthreads per plane suffices;
//  * the z pass keeps 2R+1 running accumulators per column instead of a ring of
//    raw planes: plane p adds its tap-(p - zo + R) term to every output zo it
//    touches -- 2R+1 independent DFMAs rather than one 2R+1-long dependent chain.
//    Each output still receives fma(t[0], y[zo-R], 0), fma(t[1], y[zo-R+1], .),
//    ... in ascending order;
//  * |out|^2 goes to shared memory and warp 15 (no x-pass work) forms the
//    canonical row-segment trees one phase later (tree32_serial == tree32).
// (included inside namespace mlsqr_b200 after tma.cuh)

template <int R>
struct B3P {
  static constexpr int NT = 2 * R + 1;
  static constexpr int TX = 32, TY = 32;
  static constexpr int THREADS = 512;
  static constexpr int W = TX + 2 * R;
  static constexpr int H = TY + 2 * R;
  static constexpr int XK = 4;
  static constexpr int XG = TX / XK;
  // smem column c holds global x = x0 - R - XOFF + c: the TMA box must start at a
  // 16-byte aligned x (an odd start coordinate faults), so odd R loads one extra column
  static constexpr int XOFF = R & 1;
  static constexpr int WE = (W + XOFF + 1) / 2 * 2;   // even box width
  static constexpr int P = ((WE / 2) % 2) ? WE : WE + 2;  // row pitch = box width (P/2 odd)
  static constexpr int WL = (XK + 2 * R + XOFF + 1) / 2 * 2;  // x-window doubles per task
  static constexpr int XP = 34;
  static constexpr int SQP = 34;
  static constexpr int NSTAGE = 4;  // input + old ring (old plane read 3 phases after issue)
  static constexpr int TREE_WARP = 15;
  static constexpr int IN_SLOT = (H * P + 15) / 16 * 16;  // 128-byte aligned TMA destinations
  static constexpr int OLD_DOUBLES = TX * TY;
  static constexpr int XS_DOUBLES = H * XP;
  static constexpr int SQ_DOUBLES = TY * SQP;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)NSTAGE * IN_SLOT + (size_t)NSTAGE * OLD_DOUBLES +
                                                   2 * XS_DOUBLES + 2 * SQ_DOUBLES) +
                                 NSTAGE * sizeof(unsigned long long);
  static constexpr unsigned IN_BYTES = H * P * 8u;
  static constexpr unsigned OLD_BYTES = TX * TY * 8u;
  static_assert(H * XG <= TREE_WARP * 32, "x-pass tasks must leave the tree warp free");
};

// Persistent: gridDim.x CTAs (one per SM) take work items round-robin; item k is column
// tile k % T of z chunk k / T (zchunk planes).  CTAs running at the same time therefore
// work on neighbouring tiles at the same depth, so the x/y halo re-reads hit L2, and each
// item pays the 2R + 2 phase pipeline fill once (the host picks zchunk to minimise
// waves x phases).  The TMA ring position (stage, parity) counts every issued plane
// across items, and every issued plane is waited for exactly once.
template <int R, bool TMA>
__global__ void __launch_bounds__(512, 1) blur3d_pipe(const double* __restrict__ in, double* __restrict__ out,
                                                      int nx, int ny, int nz, int tiles_x, int tiles, int zchunk,
                                                      int items, int zoff, int nzg, int zshift, Taps taps, EpiArgs e,
                                                      const __grid_constant__ CUtensorMap map_in,
                                                      const __grid_constant__ CUtensorMap map_old) {
  using C = B3P<R>;
  if (e.gate && *e.gate == 0) return;
  extern __shared__ __align__(128) double sm[];
  double* tin = sm;                                       // [NSTAGE][IN_SLOT]  rows of pitch P
  double* olds = tin + C::NSTAGE * C::IN_SLOT;            // [NSTAGE][TY][TX]
  double* xs = olds + C::NSTAGE * C::OLD_DOUBLES;         // [2][H][XP]
  double* sq = xs + 2 * C::XS_DOUBLES;                    // [2][TY][SQP]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sq + 2 * C::SQ_DOUBLES);
  const int tid = threadIdx.x;
  const size_t nxy = (size_t)nx * ny;
  const double sx = e.sx ? *e.sx : 1.0;
  const double so = e.so ? *e.so : 1.0;
  const double coef = e.old ? *e.coef : 0.0;
  const size_t chunks = (size_t)(nx + 31) / 32;
  const int tx = tid & 31, ty = tid >> 5;
  const int xr = tid % C::H, xg = tid / C::H;
  const bool xtask = tid < C::H * C::XG;
#define TAP(k) taps.t[(k) <= R ? (k) : 2 * R - (k)]

  if (TMA && tid == 0) {
#pragma unroll
    for (int s = 0; s < C::NSTAGE; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double acc[2][C::NT];
  unsigned qbase = 0;  // planes issued by earlier segments (ring position)
  // (a contiguous tile-major split needs 8% fewer phases but loses the halo L2 reuse: +50%
  //  DRAM traffic, more power, lower clocks under the power cap -- 94.5 vs 96.2 it/s at C5)
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int t = item % tiles;
    const int z0 = (item / tiles) * zchunk;
    const int z1 = min(nz, z0 + zchunk);
    const int bx = t % tiles_x;
    const int x0 = bx * C::TX, y0 = (t / tiles_x) * C::TY;
    const int zlo = z0 - R, zhi = z1 + R - 1;
    auto inside = [&](int zz) { return zz >= zlo && zz <= zhi && zz + zoff >= 0 && zz + zoff < nzg; };
    auto stage = [&](int zz) { return (qbase + (unsigned)(zz - zlo)) & (C::NSTAGE - 1); };
    auto parity = [&](int zz) { return ((qbase + (unsigned)(zz - zlo)) >> 2) & 1u; };
    // stage of plane q: input plane q and old plane q - R
    auto issue = [&](int zz) {
      const int st = stage(zz);
      const int zo = zz - R;
      const bool lin = inside(zz);
      const bool lold = e.old && zo >= z0 && zo < z1;
      if (TMA) {
        if (zz > zhi) return;  // only planes of this segment take ring stages
        if (tid == 0) {  // always arrive, so each stage's phase advances once per plane
          mbar_arrive_expect(bars + st, (lin ? C::IN_BYTES : 0u) + (lold ? C::OLD_BYTES : 0u));
          if (lin) tma_load3d(tin + st * C::IN_SLOT, &map_in, x0 - R - C::XOFF, y0 - R, zz + zshift, bars + st);
          if (lold) tma_load3d(olds + st * C::OLD_DOUBLES, &map_old, x0, y0, zo, bars + st);
        }
      } else {
        if (lin) {
          double* dst = tin + st * C::IN_SLOT;
          const double* src = in + (size_t)zz * nxy;
          for (int k = tid; k < C::H * C::W; k += C::THREADS) {
            const int ly = k / C::W, lx = k - ly * C::W;
            const int gx = x0 + lx - R, gy = y0 + ly - R;
            const bool ok = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
            cp_async8(dst + ly * C::P + lx + C::XOFF, ok ? src + (size_t)gy * nx + gx : in, ok);
          }
        }
        if (lold) {
          double* dst = olds + st * C::OLD_DOUBLES;
          const double* src = e.old + (size_t)zo * nxy;
          for (int k = tid; k < C::TX * C::TY; k += C::THREADS) {
            const int ly = k >> 5, lx = k & 31;
            const int gx = x0 + lx, gy = y0 + ly;
            const bool ok = gx < nx && gy < ny;
            cp_async8(dst + k, ok ? src + (size_t)gy * nx + gx : in, ok);
          }
        }
        cp_async_commit();  // one group per plane, empty ones included (wait<1> counts them)
      }
    };

    const int gx = x0 + tx, gy0 = y0 + 2 * ty;
    const bool ok0 = gx < nx && gy0 < ny, ok1 = gx < nx && gy0 + 1 < ny;
    double* const obase = out + (size_t)gy0 * nx + gx;
    __syncthreads();  // the previous segment is done with every buffer
    issue(zlo);
    issue(zlo + 1);
    for (int pb = zlo - 1; pb <= zhi + 1; pb += C::NT) {
#pragma unroll
      for (int u = 0; u < C::NT; ++u) {
        const int p = pb + u;
        if (p <= zhi + 1) {  // block-uniform
          // plane p+1 (x-pass input of this phase, old plane of the next) has landed
          if (TMA) {  // one warp polls the TMA barrier; the CTA barrier publishes the plane
            if (tid < 32 && p + 1 <= zhi) mbar_wait(bars + stage(p + 1), parity(p + 1));
          } else {
            cp_async_wait<1>();
          }
          __syncthreads();  // ... for everyone; phase p-1 is done with every buffer
          issue(p + 3);
          const int xz = p + 1;
          if (xtask && inside(xz)) {
            const double* row = tin + stage(xz) * C::IN_SLOT + xr * C::P + C::XK * xg;
            double wv[C::WL];
#pragma unroll
            for (int j = 0; j < C::WL / 2; ++j) {
              const double2 q = *reinterpret_cast<const double2*>(row + 2 * j);
              wv[2 * j] = q.x;
              wv[2 * j + 1] = q.y;
            }
            if (e.sx) {
#pragma unroll
              for (int j = C::XOFF; j < C::XK + 2 * R + C::XOFF; ++j) wv[j] = wv[j] * sx;
            }
            double a[C::XK];
#pragma unroll
            for (int o = 0; o < C::XK; ++o) {
              a[o] = 0.0;
#pragma unroll
              for (int k = 0; k < C::NT; ++k) a[o] = fma(TAP(k), wv[o + k + C::XOFF], a[o]);
            }
            double* xw = xs + ((xz - zlo) & 1) * C::XS_DOUBLES + xr * C::XP + C::XK * xg;
            *reinterpret_cast<double2*>(xw) = make_double2(a[0], a[1]);
            *reinterpret_cast<double2*>(xw + 2) = make_double2(a[2], a[3]);
          }
          if (p >= zlo && p <= zhi) {
            double yv0 = 0.0, yv1 = 0.0;
            if (inside(p)) {
              const double* xb = xs + ((p - zlo) & 1) * C::XS_DOUBLES + 2 * ty * C::XP + tx;
              double c[2 + 2 * R];
#pragma unroll
              for (int j = 0; j < 2 + 2 * R; ++j) c[j] = xb[j * C::XP];
#pragma unroll
              for (int k = 0; k < C::NT; ++k) {
                yv0 = fma(TAP(k), c[k], yv0);
                yv1 = fma(TAP(k), c[k + 1], yv1);
              }
            }
            // output zo' = p - R + j takes tap 2R - j; j = 2R starts output p + R
#pragma unroll
            for (int j = 0; j < C::NT; ++j) {
              const int s = (u + j) % C::NT;
              acc[0][s] = fma(TAP(2 * R - j), yv0, j == C::NT - 1 ? 0.0 : acc[0][s]);
              acc[1][s] = fma(TAP(2 * R - j), yv1, j == C::NT - 1 ? 0.0 : acc[1][s]);
            }
            const int zo = p - R;  // complete now (slot u)
            if (zo >= z0 && zo < z1) {
              const double* po = olds + stage(p) * C::OLD_DOUBLES + 2 * ty * 32 + tx;
              double* sqb = sq + ((zo - z0) & 1) * C::SQ_DOUBLES + 2 * ty * C::SQP + tx;
              double* orow = obase + (size_t)zo * nxy;
              double v0 = ok0 ? acc[0][u] : 0.0, v1 = ok1 ? acc[1][u] : 0.0;
              if (e.old) {
                double o0 = po[0], o1 = po[32];
                if (e.so) {
                  o0 = o0 * so;
                  o1 = o1 * so;
                }
                if (ok0) v0 = v0 + coef * o0;
                if (ok1) v1 = v1 + coef * o1;
              }
              if (ok0) orow[0] = v0;
              if (ok1) orow[nx] = v1;
              if (e.seg) {
                sqb[0] = v0 * v0;
                sqb[C::SQP] = v1 * v1;
              }
            }
          }
          // canonical segment partials of the plane completed in the previous phase
          const int zt = p - R - 1;
          if (e.seg && ty == C::TREE_WARP && zt >= z0 && zt < z1) {
            const int gy = y0 + tx;
            if (gy < ny) {
              const double* r = sq + ((zt - z0) & 1) * C::SQ_DOUBLES + tx * C::SQP;
              double v[32];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const double2 q = *reinterpret_cast<const double2*>(r + 2 * j);
                v[2 * j] = q.x;
                v[2 * j + 1] = q.y;
              }
              e.seg[((size_t)zt * ny + gy) * chunks + bx] = tree32_serial(v);
            }
          }
        }
      }
    }
    qbase += (unsigned)(zhi - zlo + 1);
  }
#undef TAP
}

template <int R>
static void launch_b3(Ctx* c, const double* in, double* out, int nx, int ny, int nz, const Taps& t,
                      const EpiArgs& a) {
  using C = B3P<R>;
  static std::once_flag attr;  // operators may be built on several threads (loopback ranks)
  std::call_once(attr, [] {
    MLSQR_CUDA(cudaFuncSetAttribute(blur3d_pipe<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    MLSQR_CUDA(cudaFuncSetAttribute(blur3d_pipe<R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  });
  const int tiles_x = (nx + C::TX - 1) / C::TX, tiles_y = (ny + C::TY - 1) / C::TY;
  const int tiles = tiles_x * tiles_y;
  // z chunk minimising (items per CTA) x (phases per item) on one CTA per SM
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
  const unsigned grid = (unsigned)(items < c->sm_count ? items : c->sm_count);  // persistent: one CTA per SM
  const bool sh = c->sharded();
  const int zoff = sh ? (int)c->zoff : 0, nzg = sh ? (int)c->nzg : nz;
  // z-sharded inputs carry R ghost planes on either side (guard zones): map them too
  const int zshift = sh ? R : 0;
  CUtensorMap mi{}, mo{};
  bool tma = tensor_map3d(&mi, in - (size_t)zshift * nx * ny, nx, ny, nz + 2 * zshift, C::P, C::H);
  if (tma && a.old) tma = tensor_map3d(&mo, a.old, nx, ny, nz, C::TX, C::TY);
  if (tma)
    blur3d_pipe<R, true><<<grid, C::THREADS, C::SMEM, c->stream>>>(in, out, nx, ny, nz, tiles_x, tiles, zck,
                                                                   items, zoff, nzg, zshift, t, a, mi, mo);
  else
    blur3d_pipe<R, false><<<grid, C::THREADS, C::SMEM, c->stream>>>(in, out, nx, ny, nz, tiles_x, tiles, zck,
                                                                    items, zoff, nzg, zshift, t, a, mi, mo);
  c->count();
}

