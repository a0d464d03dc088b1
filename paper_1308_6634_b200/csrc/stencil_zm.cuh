// stencil_zm.cuh -- z-marching V-cycle stencil kernels (included by vcycle.cu).
//
// A (32 x 8) block owns a column tile and walks a chunk of z planes: the z
// neighbours of the iterate and cz[z-1] stay in registers and the streams of
// plane z+1 (x, b, cx, cy, cz) are loaded one plane ahead.
//
// Branch-free rows: every internal V-cycle array (iterates, coefficients,
// coarse corrections) is allocated with a zero guard zone of one plane (+64)
// on both sides, and every missing edge has an exactly-zero coefficient.  So
// all 7 terms of a row are added unconditionally, in the CSR ascending-column
// order of m_row / diag_at (sparse.cpp:65-74): a skipped term of the reference
// becomes acc + (+-0), which is acc exactly (the accumulators start at +0 and
// can never reach -0).  Results are bit-identical to the oracle.

#ifndef MLSQR_ZM_PREFETCH
#define MLSQR_ZM_PREFETCH 1
#endif
constexpr bool kZmPrefetch = MLSQR_ZM_PREFETCH;
#ifndef MLSQR_ZM_AHEAD
#define MLSQR_ZM_AHEAD 3
#endif
constexpr int kZmAhead = MLSQR_ZM_AHEAD;  // planes ahead of the z march
// resident blocks per SM the compiler plans for: 4 (64 registers) for the plain and first sweeps, which
// otherwise take 76 registers and 3 blocks (last sweep 1.32 -> 1.22 ms per 512^3 launch in the power-capped
// bench); the prolongation sweep already fits 64 and gets slower under the constraint (1.26 -> 1.36 ms)
#ifndef MLSQR_ZM_MINB
#define MLSQR_ZM_MINB 4
#endif
#ifndef MLSQR_RZ_MINB
#define MLSQR_RZ_MINB 0  // restriction: no block target
#endif
#ifndef MLSQR_ZM_UNROLL_P
#define MLSQR_ZM_UNROLL_P 1
#endif
constexpr int kZmUnrollP = MLSQR_ZM_UNROLL_P;  // z-loop unroll of the prolongation sweep
#ifndef MLSQR_ZM_UNROLL_N
#define MLSQR_ZM_UNROLL_N 1
#endif
constexpr int kZmUnrollN = MLSQR_ZM_UNROLL_N;  // ... of the plain / first sweeps
#ifndef MLSQR_ZM_UNROLL_R
#define MLSQR_ZM_UNROLL_R 2
#endif
constexpr int kZmUnrollR = MLSQR_ZM_UNROLL_R;  // ... of the restriction
#ifndef MLSQR_ZM_MINB_P
#define MLSQR_ZM_MINB_P 0  // 0: no block target (the compiler settles on 64 registers)
#endif

// iterate value at fine index j (plus the prolongated coarse correction)
// I: element index type -- int where the level (with guards) fits 2^31 elements: every
// access is then one IMAD.WIDE instead of a 64-bit add chain (same loads, same bits)
template <int D, bool PROLONG, typename I = long>
__device__ __forceinline__ double xv_zm(const double* __restrict__ x, const double* __restrict__ xc,
                                        int cnx, int cny, int xx, int yy, int zz, I j) {
  double v = x[j];
  if (PROLONG) {
    // floor division: the ghost plane z = -1 of a slab belongs to coarse ghost plane -1
    const int Z = D >= 3 ? (zz >> 1) : 0, Y = D >= 2 ? yy / 2 : 0;
    v = v + xc[((I)Z * cny + Y) * cnx + xx / 2];
  }
  return v;
}

template <int D, int MODE, typename I = long>
__global__ void __launch_bounds__(256, MODE == kProlong ? MLSQR_ZM_MINB_P : MLSQR_ZM_MINB) sweep_zm_kernel(Lvl L, const double* __restrict__ x,
                                                       const double* __restrict__ xc, int cnx, int cny,
                                                       const double* __restrict__ b,
                                                       double* __restrict__ out, double omega,
                                                       double* __restrict__ seg, const int* gate, int zc) {
  if (gate && *gate == 0) return;
  constexpr bool P = MODE == kProlong;
  const int xx = blockIdx.x * 32 + threadIdx.x;
  const int yy = blockIdx.y * 8 + threadIdx.y;
  if (yy >= L.ny) return;  // whole warp (one row)
  const int z0 = blockIdx.z * zc;
  const int z1 = min(L.nz, z0 + zc);
  const int nx = L.nx;
  const I nxy = (I)nx * L.ny;
  const bool ix = xx < nx;
  const double eps = *L.eps;
  const double* __restrict__ cx = L.cx;
  const double* __restrict__ cy = L.cy;
  const double* __restrict__ cz = L.cz;
  const long chunks = (nx + 31) / 32;
  I i = ((I)z0 * L.ny + yy) * nx + (ix ? xx : nx - 1);
  double xm = 0.0, xcur = 0.0, xn = 0.0, czm = 0.0;
  double bc = b[i], cxc = cx[i], cyc = 0.0, czc = 0.0;
  if (D >= 2) cyc = cy[i];
  if (D >= 3) {
    czc = cz[i];
    czm = cz[i - nxy];  // guard zone below plane 0
  }
  if (MODE != kFirst) {
    xcur = xv_zm<D, P, I>(x, xc, cnx, cny, xx, yy, z0, i);
    if (D >= 3) {
      xm = xv_zm<D, P, I>(x, xc, cnx, cny, xx, yy, z0 - 1, i - nxy);
      xn = xv_zm<D, P, I>(x, xc, cnx, cny, xx, yy, z0 + 1, i + nxy);
    }
  }
#pragma unroll(MODE == kProlong ? kZmUnrollP : kZmUnrollN)
  for (int z = z0; z < z1; ++z, i += nxy) {
    if (kZmPrefetch && D >= 3 && z + kZmAhead < z1) {  // L2 prefetch of plane z+kZmAhead (no registers)
      const I j = i + kZmAhead * nxy;
      prefetch_l2(b + j);
      prefetch_l2(cx + j);
      prefetch_l2(cy + j);
      prefetch_l2(cz + j);
      if (MODE != kFirst) prefetch_l2(x + j + nxy);
    }
    // prefetch the streams of plane z+1 (plane-uniform condition)
    double bn = 0.0, cxn = 0.0, cyn = 0.0, czn = 0.0, xnn = 0.0;
    if (z + 1 < z1) {
      bn = b[i + nxy];
      cxn = cx[i + nxy];
      if (D >= 2) cyn = cy[i + nxy];
      if (D >= 3) czn = cz[i + nxy];
      if (D >= 3 && MODE != kFirst)
        xnn = xv_zm<D, P, I>(x, xc, cnx, cny, xx, yy, z + 2, i + 2 * nxy);  // guard covers z+2 = nz
    }
    double v;
    {
      // diag_at order: x-, x+, y-, y+, z-, z+ ; then + eps
      const double cxm = cx[i - 1];
      double d = 0.0;
      d = d + cxm;
      d = d + cxc;
      double cym = 0.0;
      if (D >= 2) {
        cym = cy[i - nx];
        d = d + cym;
        d = d + cyc;
      }
      if (D >= 3) {
        d = d + czm;
        d = d + czc;
      }
      d = d + eps;
      if (MODE == kFirst) {
        const double mx = 0.0;
        v = 0.0 + (omega * (bc - mx)) / d;
      } else {
        // m_row order: z-, y-, x-, diag, x+, y+, z+
        double acc = 0.0;
        if (D >= 3) acc = acc + -czm * xm;
        if (D >= 2) acc = acc + -cym * xv_zm<D, P, I>(x, xc, cnx, cny, xx, yy - 1, z, i - nx);
        acc = acc + -cxm * xv_zm<D, P, I>(x, xc, cnx, cny, xx - 1, yy, z, i - 1);
        acc = acc + d * xcur;
        acc = acc + -cxc * xv_zm<D, P, I>(x, xc, cnx, cny, xx + 1, yy, z, i + 1);
        if (D >= 2) acc = acc + -cyc * xv_zm<D, P, I>(x, xc, cnx, cny, xx, yy + 1, z, i + nx);
        if (D >= 3) acc = acc + -czc * xn;
        v = xcur + (omega * (bc - acc)) / d;
      }
    }
    if (ix) out[i] = v;
    else v = 0.0;
    if (seg) {
      const double s = tree32(v * (ix ? bc : 0.0));
      if (threadIdx.x == 0) seg[((long)z * L.ny + yy) * chunks + blockIdx.x] = s;
    }
    // roll
    czm = czc;
    xm = xcur;
    xcur = xn;
    xn = xnn;
    bc = bn;
    cxc = cxn;
    cyc = cyn;
    czc = czn;
  }
}

// fused residual + restriction: b_c[I] = sum over children (ascending fine index, i.e.
// dz, dy, dx nested) of r = b - M x.  Fine threads compute r; the (even x, even y) thread
// of each 2 x 2 patch accumulates the children in the canonical order across the two
// fine planes of the coarse cell.
template <int D, typename I = long>
__global__ void __launch_bounds__(256, MLSQR_RZ_MINB) restrict_zm_kernel(Lvl L, const double* __restrict__ x,
                                                          const double* __restrict__ b, int cnx, int cny,
                                                          double* __restrict__ bcoarse, const int* gate,
                                                          int zc) {
  if (gate && *gate == 0) return;
  __shared__ double rs[8][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int xx = blockIdx.x * 32 + tx;
  const int yy = blockIdx.y * 8 + ty;
  const int z0 = blockIdx.z * zc;
  const int z1 = min(L.nz, z0 + zc);
  const int nx = L.nx;
  const I nxy = (I)nx * L.ny;
  const bool ok = xx < nx && yy < L.ny;
  const double eps = *L.eps;
  const double* __restrict__ cx = L.cx;
  const double* __restrict__ cy = L.cy;
  const double* __restrict__ cz = L.cz;
  I i = ((I)z0 * L.ny + (yy < L.ny ? yy : L.ny - 1)) * nx + (xx < nx ? xx : nx - 1);
  double xm = 0.0, xcur = x[i], xn = 0.0, czm = 0.0;
  double bc = b[i], cxc = cx[i], cyc = 0.0, czc = 0.0;
  if (D >= 2) cyc = cy[i];
  if (D >= 3) {
    xm = x[i - nxy];
    xn = x[i + nxy];
    czm = cz[i - nxy];
    czc = cz[i];
  }
  const bool owner = ok && (tx % 2 == 0) && (D < 2 || ty % 2 == 0);
  double s = 0.0;
#pragma unroll(kZmUnrollR)
  for (int z = z0; z < z1; ++z, i += nxy) {
    if (kZmPrefetch && D >= 3 && z + kZmAhead < z1) {  // L2 prefetch of plane z+kZmAhead (no registers)
      const I j = i + kZmAhead * nxy;
      prefetch_l2(b + j);
      prefetch_l2(cx + j);
      prefetch_l2(cy + j);
      prefetch_l2(cz + j);
      prefetch_l2(x + j + nxy);
    }
    double bn = 0.0, cxn = 0.0, cyn = 0.0, czn = 0.0, xnn = 0.0;
    if (z + 1 < z1) {
      bn = b[i + nxy];
      cxn = cx[i + nxy];
      if (D >= 2) cyn = cy[i + nxy];
      if (D >= 3) {
        czn = cz[i + nxy];
        xnn = x[i + 2 * nxy];
      }
    }
    const double cxm = cx[i - 1];
    double d = 0.0;
    d = d + cxm;
    d = d + cxc;
    double cym = 0.0;
    if (D >= 2) {
      cym = cy[i - nx];
      d = d + cym;
      d = d + cyc;
    }
    if (D >= 3) {
      d = d + czm;
      d = d + czc;
    }
    d = d + eps;
    double acc = 0.0;
    if (D >= 3) acc = acc + -czm * xm;
    if (D >= 2) acc = acc + -cym * x[i - nx];
    acc = acc + -cxm * x[i - 1];
    acc = acc + d * xcur;
    acc = acc + -cxc * x[i + 1];
    if (D >= 2) acc = acc + -cyc * x[i + nx];
    if (D >= 3) acc = acc + -czc * xn;
    const double r = ok ? bc - acc : 0.0;
    const double rx1 = __shfl_down_sync(kFull, r, 1);
    if (D >= 2) {
      rs[ty][tx] = r;
      __syncthreads();
    }
    if (owner) {
      if (D < 3 || (z % 2 == 0)) s = 0.0;
      s = s + r;
      s = s + rx1;
      if (D >= 2) {
        s = s + rs[ty + 1][tx];
        s = s + rs[ty + 1][tx + 1];
      }
      if (D < 3 || (z % 2 == 1)) {
        const int Z = D >= 3 ? z / 2 : 0, Y = D >= 2 ? yy / 2 : 0;
        bcoarse[((I)Z * cny + Y) * cnx + xx / 2] = s;
      }
    }
    if (D >= 2) __syncthreads();
    czm = czc;
    xm = xcur;
    xcur = xn;
    xn = xnn;
    bc = bn;
    cxc = cxn;
    cyc = cyn;
    czc = czn;
  }
}

// zero the boundary edges of explicitly supplied coefficients (an edge that leaves the
// grid does not exist; the branch-free rows rely on its coefficient being exactly 0)
__global__ void zero_boundary_edges_kernel(Lvl L, int zoff, int nzg, double* cx, double* cy, double* cz) {
  const int rows = L.ny * L.nz;
  const int xx = blockIdx.x * 32 + threadIdx.x;
  if (xx >= L.nx) return;
  for (int row = blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += gridDim.y * blockDim.y) {  // gridDim.y <= 65535
    const int yy = row % L.ny, zz = row / L.ny;
    const long i = (long)row * L.nx + xx;
    if (xx + 1 == L.nx) cx[i] = 0.0;
    if (cy && yy + 1 == L.ny) cy[i] = 0.0;
    if (cz && zz + zoff + 1 == nzg) cz[i] = 0.0;  // global top plane
  }
}

// z chunk: enough blocks to fill the GPU a few times; even (restriction pairs fine planes)
// (MLSQR_ZM_BPS: target blocks per SM, default 24)
static inline int zm_chunk(int nx, int ny, int nz, int sms) {
  static const long bps = getenv("MLSQR_ZM_BPS") ? atol(getenv("MLSQR_ZM_BPS")) : 24;
  const long bxy = (long)((nx + 31) / 32) * ((ny + 7) / 8);
  long chunks = (sms * bps + bxy - 1) / bxy;
  if (chunks < 1) chunks = 1;
  if (chunks > nz) chunks = nz;
  int zc = (int)((nz + chunks - 1) / chunks);
  if (zc > 32) zc = 32;
  if (nz > 1 && (zc % 2)) ++zc;
  return zc < 1 ? 1 : zc;
}
