// sweep_pn.cuh -- the first two post-smoothing sweeps of a level fused in one
// z-marching kernel (3D, whole grids; included by vcycle.cu after sweep_fn.cuh).
//
//   x3  = xp + (omega * (b - M xp)) / D,   xp = x + P xc    (sweep 3: prolongate, correct, sweep)
//   out = x3 + (omega * (b - M x3)) / D                     (sweep 4, + optional <out, b> partials)
//
// The same plane-lagged scheme as sweep_fn: each thread computes x3 at its own point one plane
// ahead (loading xp's x/y neighbours like sweep_zm_kernel<kProlong> does) and publishes it in a
// 3-plane shared ring; after one __syncthreads per plane the output rows apply sweep 4 to plane z
// from the ring and their own column's x3 at z-1, z+1.  D is formed once per point and used by
// both sweeps.  x3 never touches HBM and b and the coefficients are read once: level-0 traffic
// drops from 5 1/8 + 1 plus 5 + 1 words per voxel (two sweep_zm launches) to 5 1/8 + 1.
//
// Measured slower than the two sweep_zm launches it replaces (512^3 V-cycle 5.95 vs 4.97 ms;
// a variant staging xp in a second shared ring, 6.83 ms): sweep 3's x/y neighbour loads sit
// in front of the per-plane barrier with 19 warps per SM.  Off by default (MLSQR_PN_SWEEPS=1
// turns it on); the parity tests run both paths.
//
// Bit-exactness: both sweeps use exactly sweep_zm_kernel's operation order (diag_at / m_row,
// sparse.cpp:65-74) and xv_zm's prolongation; x3 outside the domain is 0 here where the unfused
// kernel read some finite value -- either way it meets an exactly-zero coefficient.
namespace pn {
constexpr int TX = fn::TX, TY = fn::TY;
constexpr int ROWS = TY + 2, COLS = TX + 2;
constexpr int WARPS = ROWS + 1;
constexpr int THREADS = 32 * WARPS;
}  // namespace pn

#ifndef MLSQR_PN_AHEAD
#define MLSQR_PN_AHEAD 2
#endif
constexpr int kPnL2Ahead = MLSQR_PN_AHEAD;  // L2 prefetch distance beyond the plane being loaded

struct PnPlane {
  double b, cx, cxm, cy, cym, cz, xq;  // xq = x + P xc at the thread's own point
};

template <typename I>
__device__ __forceinline__ PnPlane pn_load(const Lvl& L, const double* __restrict__ x,
                                           const double* __restrict__ xc, int cnx, int cny,
                                           const double* __restrict__ b, bool on, I i, int nx, int px,
                                           int py, int z) {
  PnPlane s{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (on) {
    s.b = b[i];
    s.cx = L.cx[i];
    s.cxm = L.cx[i - 1];
    s.cy = L.cy[i];
    s.cym = L.cy[i - nx];
    s.cz = L.cz[i];
    s.xq = xv_zm<3, true, I>(x, xc, cnx, cny, px, py, z, i);
  }
  return s;
}

template <typename I>
__global__ void __launch_bounds__(pn::THREADS, 1) sweep_pn_kernel(Lvl L, const double* __restrict__ x,
                                                                  const double* __restrict__ xc, int cnx,
                                                                  int cny, const double* __restrict__ b,
                                                                  double* __restrict__ out, double omega,
                                                                  double* __restrict__ seg, const int* gate,
                                                                  int zc) {
  using namespace pn;
  if (gate && *gate == 0) return;
  __shared__ double ring[3][ROWS][COLS];  // x3, planes z-1..z+1
  const int lane = threadIdx.x, w = threadIdx.y;
  const int nx = L.nx, ny = L.ny, nz = L.nz;
  const I nxy = (I)nx * ny;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(nz, z0 + zc);
  int px, py, sr, sc;
  bool act;
  if (w < ROWS) {
    px = x0 + lane;
    py = y0 - 1 + w;
    sr = w;
    sc = lane + 1;
    act = true;
  } else {
    const int side = lane / TY, k = lane % TY;
    px = side ? x0 + TX : x0 - 1;
    py = y0 + k;
    sr = k + 1;
    sc = side ? COLS - 1 : 0;
    act = lane < 2 * TY;
  }
  const bool inxy = act && px >= 0 && px < nx && py >= 0 && py < ny;
  const bool outw = w >= 1 && w <= TY && py < ny;  // output rows (whole warps)
  const bool ix = inxy && outw;
  const double eps = *L.eps;
  const long chunks = (nx + 31) / 32;
  const I col = inxy ? (I)py * nx + px : 0;
  auto idx = [&](int z) { return (I)z * nxy + col; };
  auto on = [&](int z) { return inxy && z >= 0 && z < nz; };
  auto ld = [&](int z) { return pn_load<I>(L, x, xc, cnx, cny, b, on(z), idx(z), nx, px, py, z); };
  auto xp = [&](int xx, int yy, int z, I j) { return xv_zm<3, true, I>(x, xc, cnx, cny, xx, yy, z, j); };
  // sweep 3 at the thread's own point of plane p: s = plane p, czm/xm = cz/xp of plane p-1,
  // xn = xp of plane p+1; d <- D at the point
  auto s3 = [&](const PnPlane& s, double czm, double xm, double xn, int p, double& d) {
    d = 0.0;
    d = d + s.cxm;
    d = d + s.cx;
    d = d + s.cym;
    d = d + s.cy;
    d = d + czm;
    d = d + s.cz;
    d = d + eps;
    if (!on(p)) return 0.0;
    const I i = idx(p);
    // m_row order: z-, y-, x-, diag, x+, y+, z+
    double acc = 0.0;
    acc = acc + -czm * xm;
    acc = acc + -s.cym * xp(px, py - 1, p, i - nx);
    acc = acc + -s.cxm * xp(px - 1, py, p, i - 1);
    acc = acc + d * s.xq;
    acc = acc + -s.cx * xp(px + 1, py, p, i + 1);
    acc = acc + -s.cy * xp(px, py + 1, p, i + nx);
    acc = acc + -s.cz * xn;
    return s.xq + (omega * (s.b - acc)) / d;
  };

  // prologue: x3 of plane z0-1 (own column), x3 of plane z0 (published)
  double dd;
  const PnPlane pm2 = ld(z0 - 2);
  const PnPlane pm = ld(z0 - 1);
  PnPlane o = ld(z0);
  PnPlane c = ld(z0 + 1);
  double x3m = s3(pm, pm2.cz, pm2.xq, o.xq, z0 - 1, dd);
  double d_o;
  double x3c = s3(o, pm.cz, pm.xq, c.xq, z0, d_o);
  double czm_o = pm.cz;  // cz of plane z-1
  if (act) ring[0][sr][sc] = x3c;
  int slot = 0;
#pragma unroll 1
  for (int z = z0; z < z1; ++z) {
    // plane z+2: only its xq is needed now (last term of sweep 3); the L2 prefetch runs ahead
    const PnPlane n = ld(z + 2);
    if (on(z + 2 + kPnL2Ahead)) {
      const I i = idx(z + 2 + kPnL2Ahead);
      prefetch_l2(b + i);
      prefetch_l2(x + i);
      prefetch_l2(L.cx + i);
      prefetch_l2(L.cy + i);
      prefetch_l2(L.cz + i);
    }
    double d_c;
    const double x3n = s3(c, o.cz, o.xq, n.xq, z + 1, d_c);
    const int ns = slot == 2 ? 0 : slot + 1;
    if (act) ring[ns][sr][sc] = x3n;
    __syncthreads();
    if (outw) {
      double v = 0.0;
      if (ix) {
        double acc = 0.0;
        acc = acc + -czm_o * x3m;
        acc = acc + -o.cym * ring[slot][sr - 1][sc];
        acc = acc + -o.cxm * ring[slot][sr][sc - 1];
        acc = acc + d_o * x3c;
        acc = acc + -o.cx * ring[slot][sr][sc + 1];
        acc = acc + -o.cy * ring[slot][sr + 1][sc];
        acc = acc + -o.cz * x3n;
        v = x3c + (omega * (o.b - acc)) / d_o;
        out[idx(z)] = v;
      }
      if (seg) {
        const double s = tree32(v * (ix ? o.b : 0.0));
        if (lane == 0) seg[((long)z * ny + py) * chunks + blockIdx.x] = s;
      }
    }
    x3m = x3c;
    x3c = x3n;
    czm_o = o.cz;
    d_o = d_c;
    o = c;
    c = n;
    slot = ns;
  }
}
