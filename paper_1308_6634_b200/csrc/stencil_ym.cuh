// stencil_ym.cuh -- 2D V-cycle stencil kernels that march along y (included by vcycle.cu).
//
// The 2D levels of C1/C2 are L2-resident, so their sweeps are bound by latency, not bytes: with
// one point per thread a 1024^2 level is 4096 blocks in 3.5 waves, each block waiting out its
// own L2 round trips.  Here a warp owns 32 columns and marches YC rows, like the 3D z-march
// kernels march planes: x of rows y-1, y, y+1 and cy[y-1] stay in registers and the streams of
// row y+1 (x of row y+2) are loaded one row ahead, so about one wave of blocks keeps every
// warp's next loads in flight.  Per point the arithmetic is sweep_zm_kernel<2>'s and
// restrict_zm_kernel<2>'s (diag_at order, m_row order, children (y, x)-nested ascending), so the
// results are bit-identical to them.

// rows per warp: the smallest even chunk (the restriction pairs rows) that leaves at most ~one
// wave of 256-thread blocks at `per_sm` resident blocks per SM
static inline int ym_chunk(int nx, int ny, int sms, int per_sm) {
  const long bx = (nx + 31) / 32;
  int yc = 2;
  while (yc < 16 && bx * ((ny + 8 * yc - 1) / (8 * yc)) > (long)per_sm * sms) yc *= 2;
  return yc;
}

template <int MODE>
__global__ void __launch_bounds__(256) sweep_ym_kernel(Lvl L, const double* __restrict__ x,
                                                       const double* __restrict__ xc, int cnx, int cny,
                                                       const double* __restrict__ b, double* __restrict__ out,
                                                       double omega, double* __restrict__ seg, const int* gate,
                                                       int yc) {
  if (gate && *gate == 0) return;
  constexpr bool P = MODE == kProlong;
  const int xx = blockIdx.x * 32 + threadIdx.x;
  const int y0 = (blockIdx.y * 8 + threadIdx.y) * yc;
  if (y0 >= L.ny) return;  // whole warp
  const int y1 = min(L.ny, y0 + yc);
  const int nx = L.nx;
  const bool ix = xx < nx;
  const double eps = *L.eps;
  const double* __restrict__ cx = L.cx;
  const double* __restrict__ cy = L.cy;
  const long chunks = (nx + 31) / 32;
  long i = (long)y0 * nx + (ix ? xx : nx - 1);
  double xm = 0.0, xcur = 0.0, xn = 0.0;
  double bc = b[i], cxc = cx[i], cyc = cy[i], cym = cy[i - nx];  // row -1: guard zone (0)
  if (MODE != kFirst) {
    xcur = xv_zm<2, P>(x, xc, cnx, cny, xx, y0, 0, i);
    xm = xv_zm<2, P>(x, xc, cnx, cny, xx, y0 - 1, 0, i - nx);
    xn = xv_zm<2, P>(x, xc, cnx, cny, xx, y0 + 1, 0, i + nx);
  }
  for (int y = y0; y < y1; ++y, i += nx) {
    // the streams of row y+1 (x of row y+2), one row ahead
    double bn = 0.0, cxn = 0.0, cyn = 0.0, xnn = 0.0;
    if (y + 1 < y1) {
      bn = b[i + nx];
      cxn = cx[i + nx];
      cyn = cy[i + nx];
      if (MODE != kFirst) xnn = xv_zm<2, P>(x, xc, cnx, cny, xx, y + 2, 0, i + 2 * nx);  // guard covers ny + 1
    }
    const double cxm = cx[i - 1];
    // diag_at order: x-, x+, y-, y+ ; then + eps
    double d = 0.0;
    d = d + cxm;
    d = d + cxc;
    d = d + cym;
    d = d + cyc;
    d = d + eps;
    double v;
    if (MODE == kFirst) {
      const double mx = 0.0;
      v = 0.0 + (omega * (bc - mx)) / d;
    } else {
      // m_row order: y-, x-, diag, x+, y+
      double acc = 0.0;
      acc = acc + -cym * xm;
      acc = acc + -cxm * xv_zm<2, P>(x, xc, cnx, cny, xx - 1, y, 0, i - 1);
      acc = acc + d * xcur;
      acc = acc + -cxc * xv_zm<2, P>(x, xc, cnx, cny, xx + 1, y, 0, i + 1);
      acc = acc + -cyc * xn;
      v = xcur + (omega * (bc - acc)) / d;
    }
    if (ix) out[i] = v;
    else v = 0.0;
    if (seg) {
      const double s = tree32(v * (ix ? bc : 0.0));
      if (threadIdx.x == 0) seg[(long)y * chunks + blockIdx.x] = s;
    }
    cym = cyc;
    xm = xcur;
    xcur = xn;
    xn = xnn;
    bc = bn;
    cxc = cxn;
    cyc = cyn;
  }
}

// fused residual + restriction, 2D, marching rows in pairs: the (even x) lane of each column pair
// sums r(x, y), r(x+1, y), r(x, y+1), r(x+1, y+1) -- restrict_zm_kernel<2>'s order
__global__ void __launch_bounds__(256) restrict_ym_kernel(Lvl L, const double* __restrict__ x,
                                                         const double* __restrict__ b, int cnx,
                                                         double* __restrict__ bcoarse, const int* gate, int yc) {
  if (gate && *gate == 0) return;
  const int tx = threadIdx.x;
  const int xx = blockIdx.x * 32 + tx;
  const int y0 = (blockIdx.y * 8 + threadIdx.y) * yc;
  if (y0 >= L.ny) return;  // whole warp
  const int y1 = min(L.ny, y0 + yc);
  const int nx = L.nx;
  const bool ok = xx < nx;
  const double eps = *L.eps;
  const double* __restrict__ cx = L.cx;
  const double* __restrict__ cy = L.cy;
  long i = (long)y0 * nx + (ok ? xx : nx - 1);
  double xm = x[i - nx], xcur = x[i], xn = x[i + nx];
  double bc = b[i], cxc = cx[i], cyc = cy[i], cym = cy[i - nx];
  const bool owner = ok && (tx % 2 == 0);
  double s = 0.0;
  for (int y = y0; y < y1; ++y, i += nx) {
    double bn = 0.0, cxn = 0.0, cyn = 0.0, xnn = 0.0;
    if (y + 1 < y1) {
      bn = b[i + nx];
      cxn = cx[i + nx];
      cyn = cy[i + nx];
      xnn = x[i + 2 * nx];
    }
    const double cxm = cx[i - 1];
    double d = 0.0;
    d = d + cxm;
    d = d + cxc;
    d = d + cym;
    d = d + cyc;
    d = d + eps;
    double acc = 0.0;
    acc = acc + -cym * xm;
    acc = acc + -cxm * x[i - 1];
    acc = acc + d * xcur;
    acc = acc + -cxc * x[i + 1];
    acc = acc + -cyc * xn;
    const double r = ok ? bc - acc : 0.0;
    const double rx1 = __shfl_down_sync(kFull, r, 1);
    if (owner) {
      if (y % 2 == 0) s = 0.0;
      s = s + r;
      s = s + rx1;
      if (y % 2 == 1) bcoarse[(long)(y / 2) * cnx + xx / 2] = s;
    }
    cym = cyc;
    xm = xcur;
    xcur = xn;
    xn = xnn;
    bc = bn;
    cxc = cxn;
    cyc = cyn;
  }
}
