// stencil_zm.cuh -- z-marching versions of the V-cycle stencil kernels
// (included by vcycle.cu).  A (32 x 8) block owns a column tile and walks a
// chunk of z planes: the z neighbours of the iterate and cz[z-1] stay in
// registers, the streams of plane z+1 (x, b, cx, cy, cz) are loaded one plane
// ahead, and only the in-plane neighbours go through L1.  Arithmetic is
// operation-for-operation the one of m_row / diag_at (CSR ascending column
// order, sparse.cpp:65-74), so results are bit-identical to the per-voxel
// kernels and to the oracle.

// iterate value at fine index j (plus the prolongated coarse correction)
template <bool PROLONG>
__device__ __forceinline__ double xv_zm(const double* __restrict__ x, const double* __restrict__ xc,
                                        int cnx, int cny, bool has_y, bool has_z, int xx, int yy, int zz,
                                        size_t j) {
  double v = x[j];
  if (PROLONG) {
    const int Z = has_z ? zz / 2 : 0, Y = has_y ? yy / 2 : 0;
    v = v + xc[((size_t)Z * cny + Y) * cnx + xx / 2];
  }
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256) sweep_zm_kernel(Lvl L, const double* __restrict__ x,
                                                       const double* __restrict__ xc, int cnx, int cny,
                                                       const double* __restrict__ b,
                                                       double* __restrict__ out, double omega,
                                                       double* __restrict__ seg, const int* gate, int zc) {
  if (gate && *gate == 0) return;
  constexpr bool P = MODE == kProlong || MODE == kProlongOnly;
  const int xx = blockIdx.x * 32 + threadIdx.x;
  const int yy = blockIdx.y * 8 + threadIdx.y;
  if (yy >= L.ny) return;  // whole warp (one row)
  const int z0 = blockIdx.z * zc;
  const int z1 = min(L.nz, z0 + zc);
  const bool hy = L.cy != nullptr, hz = L.cz != nullptr;
  const size_t nxy = (size_t)L.nx * L.ny;
  const bool ix = xx < L.nx;
  const double eps = *L.eps;
  const size_t chunks = (size_t)(L.nx + 31) / 32;
  size_t i = ((size_t)z0 * L.ny + yy) * L.nx + xx;
  // rolling registers: iterate at z-1, z, z+1 and cz at z-1
  double xm = 0.0, xcur = 0.0, czm = 0.0;
  // streams of the current plane
  double bc = 0.0, cxc = 0.0, cyc = 0.0, czc = 0.0, xn = 0.0;
  if (ix) {
    if (MODE != kFirst) {
      xcur = xv_zm<P>(x, xc, cnx, cny, hy, hz, xx, yy, z0, i);
      if (hz && z0 > 0) xm = xv_zm<P>(x, xc, cnx, cny, hy, hz, xx, yy, z0 - 1, i - nxy);
      if (hz && z0 + 1 < L.nz) xn = xv_zm<P>(x, xc, cnx, cny, hy, hz, xx, yy, z0 + 1, i + nxy);
    }
    if (hz && z0 > 0) czm = L.cz[i - nxy];
    bc = b[i];
    cxc = L.cx[i];
    if (hy) cyc = L.cy[i];
    if (hz) czc = L.cz[i];
  }
  for (int z = z0; z < z1; ++z, i += nxy) {
    // prefetch the streams of plane z+1 (one plane of HBM loads in flight)
    double bn = 0.0, cxn = 0.0, cyn = 0.0, czn = 0.0, xnn = 0.0;
    if (ix && z + 1 < z1) {
      bn = b[i + nxy];
      cxn = L.cx[i + nxy];
      if (hy) cyn = L.cy[i + nxy];
      if (hz) czn = L.cz[i + nxy];
      if (MODE != kFirst && MODE != kProlongOnly && hz && z + 2 < L.nz)
        xnn = xv_zm<P>(x, xc, cnx, cny, hy, hz, xx, yy, z + 2, i + 2 * nxy);
    }
    double v = 0.0;
    if (ix) {
      if (MODE == kProlongOnly) {
        v = xcur;
      } else {
        // diag_at order: x-, x+, y-, y+, z-, z+ ; then + eps
        double d = 0.0;
        if (xx > 0) d = d + L.cx[i - 1];
        if (xx + 1 < L.nx) d = d + cxc;
        if (hy) {
          if (yy > 0) d = d + L.cy[i - L.nx];
          if (yy + 1 < L.ny) d = d + cyc;
        }
        if (hz) {
          if (z > 0) d = d + czm;
          if (z + 1 < L.nz) d = d + czc;
        }
        d = d + eps;
        if (MODE == kFirst) {
          const double mx = 0.0;
          v = 0.0 + (omega * (bc - mx)) / d;
        } else {
          // m_row order: z-, y-, x-, diag, x+, y+, z+
          double acc = 0.0;
          if (hz && z > 0) acc = acc + -czm * xm;
          if (hy && yy > 0) acc = acc + -L.cy[i - L.nx] * xv_zm<P>(x, xc, cnx, cny, hy, hz, xx, yy - 1, z, i - L.nx);
          if (xx > 0) acc = acc + -L.cx[i - 1] * xv_zm<P>(x, xc, cnx, cny, hy, hz, xx - 1, yy, z, i - 1);
          acc = acc + d * xcur;
          if (xx + 1 < L.nx) acc = acc + -cxc * xv_zm<P>(x, xc, cnx, cny, hy, hz, xx + 1, yy, z, i + 1);
          if (hy && yy + 1 < L.ny) acc = acc + -cyc * xv_zm<P>(x, xc, cnx, cny, hy, hz, xx, yy + 1, z, i + L.nx);
          if (hz && z + 1 < L.nz) acc = acc + -czc * xn;
          v = xcur + (omega * (bc - acc)) / d;
        }
      }
      out[i] = v;
    }
    if (seg) {
      const double s = tree32(v * bc);
      if (threadIdx.x == 0) seg[((size_t)z * L.ny + yy) * chunks + blockIdx.x] = s;
    }
    // roll
    czm = czc;
    xm = xcur;
    if (MODE == kProlongOnly) {
      if (ix && z + 1 < z1) xcur = xv_zm<P>(x, xc, cnx, cny, hy, hz, xx, yy, z + 1, i + nxy);
    } else {
      xcur = xn;
      xn = xnn;
    }
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
__global__ void __launch_bounds__(256) restrict_zm_kernel(Lvl L, const double* __restrict__ x,
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
  const bool hy = L.cy != nullptr, hz = L.cz != nullptr;
  const size_t nxy = (size_t)L.nx * L.ny;
  const bool ok = xx < L.nx && yy < L.ny;
  const double eps = *L.eps;
  size_t i = ((size_t)z0 * L.ny + (yy < L.ny ? yy : 0)) * L.nx + (xx < L.nx ? xx : 0);
  double xm = 0.0, xcur = 0.0, xn = 0.0, czm = 0.0;
  double bc = 0.0, cxc = 0.0, cyc = 0.0, czc = 0.0;
  if (ok) {
    xcur = x[i];
    if (hz && z0 > 0) {
      xm = x[i - nxy];
      czm = L.cz[i - nxy];
    }
    if (hz && z0 + 1 < L.nz) xn = x[i + nxy];
    bc = b[i];
    cxc = L.cx[i];
    if (hy) cyc = L.cy[i];
    if (hz) czc = L.cz[i];
  }
  const bool owner = ok && (tx % 2 == 0) && (!hy || ty % 2 == 0);
  double s = 0.0;
  for (int z = z0; z < z1; ++z, i += nxy) {
    double bn = 0.0, cxn = 0.0, cyn = 0.0, czn = 0.0, xnn = 0.0;
    if (ok && z + 1 < z1) {
      bn = b[i + nxy];
      cxn = L.cx[i + nxy];
      if (hy) cyn = L.cy[i + nxy];
      if (hz) czn = L.cz[i + nxy];
      if (hz && z + 2 < L.nz) xnn = x[i + 2 * nxy];
    }
    double r = 0.0;
    if (ok) {
      double d = 0.0;
      if (xx > 0) d = d + L.cx[i - 1];
      if (xx + 1 < L.nx) d = d + cxc;
      if (hy) {
        if (yy > 0) d = d + L.cy[i - L.nx];
        if (yy + 1 < L.ny) d = d + cyc;
      }
      if (hz) {
        if (z > 0) d = d + czm;
        if (z + 1 < L.nz) d = d + czc;
      }
      d = d + eps;
      double acc = 0.0;
      if (hz && z > 0) acc = acc + -czm * xm;
      if (hy && yy > 0) acc = acc + -L.cy[i - L.nx] * x[i - L.nx];
      if (xx > 0) acc = acc + -L.cx[i - 1] * x[i - 1];
      acc = acc + d * xcur;
      if (xx + 1 < L.nx) acc = acc + -cxc * x[i + 1];
      if (hy && yy + 1 < L.ny) acc = acc + -cyc * x[i + L.nx];
      if (hz && z + 1 < L.nz) acc = acc + -czc * xn;
      r = bc - acc;
    }
    const double rx1 = __shfl_down_sync(kFull, r, 1);
    rs[ty][tx] = r;
    __syncthreads();
    if (owner) {
      const bool first = !hz || (z % 2 == 0);
      if (first) s = 0.0;
      s = s + r;
      s = s + rx1;
      if (hy) {
        s = s + rs[ty + 1][tx];
        s = s + rs[ty + 1][tx + 1];
      }
      if (!hz || (z % 2 == 1)) {
        const int Z = hz ? z / 2 : 0, Y = hy ? yy / 2 : 0;
        bcoarse[((size_t)Z * cny + Y) * cnx + xx / 2] = s;
      }
    }
    __syncthreads();
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

// z chunk: enough blocks to fill the GPU a few times; even (restriction pairs fine planes)
static inline int zm_chunk(int nx, int ny, int nz, int sms) {
  const long bxy = (long)((nx + 31) / 32) * ((ny + 7) / 8);
  long chunks = (sms * 12L + bxy - 1) / bxy;
  if (chunks < 1) chunks = 1;
  if (chunks > nz) chunks = nz;
  int zc = (int)((nz + chunks - 1) / chunks);
  if (zc > 32) zc = 32;
  if (nz > 1 && (zc % 2)) ++zc;
  return zc < 1 ? 1 : zc;
}
