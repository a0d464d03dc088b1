// sweep_fn.cuh -- the first two pre-smoothing sweeps of a level fused in one
// z-marching kernel (3D; included by vcycle.cu).
//
//   x1  = 0 + (omega * (b - 0)) / D                     (sweep 1 from zero: pointwise)
//   out = x1 + (omega * (b - M x1)) / D                 (sweep 2, + optional <out, b> partials)
//
// Sweep 1 needs no neighbours, so the intermediate iterate never touches HBM:
// each thread computes x1 at its own point one plane ahead and publishes it in
// a 3-plane shared ring (one __syncthreads per plane); two extra warps compute
// x1 on the y-halo rows and a third on the x-halo columns.  b and the edge
// coefficients are read once (the neighbour coefficients cx[i-1], cy[i-nx] are
// L1/L2 hits, cz[i-nxy] stays in a register), so level-0 traffic drops from
// 5 + 6 words per voxel (two sweeps) to 4 + 1.
//
// z slabs: planes -1 and nz are ghost planes (b, cx, cy, cz exchanged; cz two planes below), so
// x1 on them is computed here too; `on` admits a plane iff it lies in the global grid.
//
// Bit-exactness: D and both row sums are formed in exactly the order of
// sweep_zm_kernel (diag_at / m_row, sparse.cpp:65-74).  x1 outside the domain is
// 0 here where the unfused kernel read some finite in-domain value -- either way
// it meets an exactly-zero boundary coefficient and acc + (+-0) == acc.
namespace fn {
constexpr int TX = 32, TY = 16;
constexpr int ROWS = TY + 2, COLS = TX + 2;
constexpr int WARPS = ROWS + 1;  // rows y0-1 .. y0+TY, then the x-halo warp
constexpr int THREADS = 32 * WARPS;
#ifndef MLSQR_FN_MINB
#define MLSQR_FN_MINB 1
#endif
constexpr int MINB = MLSQR_FN_MINB;  // resident blocks per SM (19 warps, 85-92 registers at 1)
}  // namespace fn

constexpr int kFnL2Ahead = 1;  // L2 prefetch distance beyond the register prefetch (planes)

struct FnPlane {
  double b, cx, cxm, cy, cym, cz;
};

__device__ __forceinline__ FnPlane fn_load(const Lvl& L, const double* __restrict__ b, bool on, long i,
                                           long nx) {
  FnPlane s{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (on) {
    s.b = b[i];
    s.cx = L.cx[i];
    s.cxm = L.cx[i - 1];
    s.cy = L.cy[i];
    s.cym = L.cy[i - nx];
    s.cz = L.cz[i];
  }
  return s;
}

// diag_at order: x-, x+, y-, y+, z-, z+ ; then + eps
__device__ __forceinline__ double fn_diag(const FnPlane& s, double czm, double eps) {
  double d = 0.0;
  d = d + s.cxm;
  d = d + s.cx;
  d = d + s.cym;
  d = d + s.cy;
  d = d + czm;
  d = d + s.cz;
  return d + eps;
}

__global__ void __launch_bounds__(fn::THREADS, fn::MINB) sweep_fn_kernel(Lvl L, const double* __restrict__ b,
                                                                  double* __restrict__ out, double omega,
                                                                  double* __restrict__ seg, const int* gate,
                                                                  int zc, int zoff, int nzg) {
  using namespace fn;
  if (gate && *gate == 0) return;
  __shared__ double ring[3][ROWS][COLS];
  const int lane = threadIdx.x, w = threadIdx.y;
  const int nx = L.nx, ny = L.ny, nz = L.nz;
  const long nxy = (long)nx * ny;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(nz, z0 + zc);
  // the point this thread computes x1 for, and where it publishes it
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
  const long col = inxy ? (long)py * nx + px : 0;
  auto idx = [&](int z) { return (long)z * nxy + col; };
  // a plane exists if it is in the global grid and local or one of the two ghost planes
  const int zon_lo = max(-1, -zoff), zon_hi = min(nz, nzg - 1 - zoff);
  auto on = [&](int z) { return inxy && z >= zon_lo && z <= zon_hi; };
  auto first = [&](const FnPlane& s, double d, bool in) { return in ? 0.0 + (omega * (s.b - 0.0)) / d : 0.0; };

  // prologue: plane z0-1 (own column only), plane z0 (published), plane z0+1 (loaded)
  double czm = on(z0 - 1) ? L.cz[idx(z0 - 2)] : 0.0;
  FnPlane m = fn_load(L, b, on(z0 - 1), idx(z0 - 1), nx);
  double x1m = first(m, fn_diag(m, czm, eps), on(z0 - 1));
  FnPlane c = fn_load(L, b, on(z0), idx(z0), nx);
  double czm_c = m.cz;  // cz of plane z0-1
  double dc = fn_diag(c, czm_c, eps);
  double x1c = first(c, dc, on(z0));
  if (act) ring[0][sr][sc] = x1c;
  FnPlane n = fn_load(L, b, on(z0 + 1), idx(z0 + 1), nx);
  int slot = 0;  // ring slot of plane z
  long o = idx(z0);  // offset of plane z, advanced by one plane per step
#pragma unroll 3
  for (int z = z0; z < z1; ++z, o += nxy) {
    FnPlane f = fn_load(L, b, on(z + 2), o + 2 * nxy, nx);  // prefetch
    if (on(z + 2 + kFnL2Ahead)) {
      const long i = o + (2 + kFnL2Ahead) * nxy;
      prefetch_l2(b + i);
      prefetch_l2(L.cx + i);
      prefetch_l2(L.cy + i);
      prefetch_l2(L.cz + i);
    }
    const double dn = fn_diag(n, c.cz, eps);
    const double x1n = first(n, dn, on(z + 1));
    const int ns = slot == 2 ? 0 : slot + 1;
    if (act) ring[ns][sr][sc] = x1n;
    __syncthreads();
    if (outw) {
      double v = 0.0;
      if (ix) {
        // m_row order: z-, y-, x-, diag, x+, y+, z+
        double acc = 0.0;
        acc = acc + -czm_c * x1m;
        acc = acc + -c.cym * ring[slot][sr - 1][sc];
        acc = acc + -c.cxm * ring[slot][sr][sc - 1];
        acc = acc + dc * x1c;
        acc = acc + -c.cx * ring[slot][sr][sc + 1];
        acc = acc + -c.cy * ring[slot][sr + 1][sc];
        acc = acc + -c.cz * x1n;
        v = x1c + (omega * (c.b - acc)) / dc;
        out[o] = v;
      }
      if (seg) {
        const double s = tree32(v * (ix ? c.b : 0.0));
        if (lane == 0) seg[((long)z * ny + py) * chunks + blockIdx.x] = s;
      }
    }
    x1m = x1c;
    x1c = x1n;
    czm_c = c.cz;
    c = n;
    dc = dn;
    n = f;
    slot = ns;
  }
}

// TMA-fed variant (the default where the four streams can be tensor-mapped): one thread issues,
// per plane, four TMA boxes -- b, cx, cy, cz over columns x0-2 .. x0+33 and rows y0-2 .. y0+16, the
// tile's x1 region plus the x- / y- neighbour of its first column / row -- into an NS-stage ring
// completed by mbarriers, NS - 1 planes ahead of the plane whose x1 is formed.  Every thread then
// reads its point's six values from shared memory instead of issuing six 64-bit-addressed loads
// and L2 prefetches.  A box (or a plane outside the grid) is zero-filled by the hardware, which
// gives x1 = 0 there, as the plain kernel's predicates do; the arithmetic is the plain kernel's,
// operand for operand, so the two are bit-identical.
namespace fnt {
constexpr int BX = 36, BY = fn::TY + 3;  // box: columns x0-2 .., rows y0-2 ..
constexpr int BOX = (BX * BY + 15) / 16 * 16;  // TMA destinations are 128-byte aligned
#ifndef MLSQR_FN_NS
#define MLSQR_FN_NS 8
#endif
constexpr int NS = MLSQR_FN_NS;         // ring stages (planes)
constexpr int STAGE = 4 * BOX;           // b, cx, cy, cz
constexpr size_t SMEM = sizeof(double) * ((size_t)NS * STAGE + 3 * fn::ROWS * fn::COLS) + NS * 8;
constexpr unsigned STAGE_BYTES = 4u * BX * BY * 8u;  // the bytes the four boxes deliver
}  // namespace fnt

__global__ void __launch_bounds__(fn::THREADS, fn::MINB)
    sweep_fn_tma_kernel(Lvl L, double* __restrict__ out, double omega, double* __restrict__ seg, const int* gate,
                        int zc, int zoff, int nzg, int gb, int gcz, const __grid_constant__ CUtensorMap mb,
                        const __grid_constant__ CUtensorMap mcx, const __grid_constant__ CUtensorMap mcy,
                        const __grid_constant__ CUtensorMap mcz) {
  using namespace fn;
  if (gate && *gate == 0) return;
  extern __shared__ __align__(128) double smf[];
  double* stg = smf;                                             // [NS][4][BY][BX]
  double (*ring)[ROWS][COLS] = reinterpret_cast<double (*)[ROWS][COLS]>(stg + fnt::NS * fnt::STAGE);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(stg + fnt::NS * fnt::STAGE + 3 * ROWS * COLS);
  const int lane = threadIdx.x, w = threadIdx.y;
  const int tid = w * 32 + lane;
  const int nx = L.nx, ny = L.ny, nz = L.nz;
  const long nxy = (long)nx * ny;
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
  const bool outw = w >= 1 && w <= TY && py < ny;
  const bool ix = inxy && outw;
  const double eps = *L.eps;
  const long chunks = (nx + 31) / 32;
  const int bo = act ? (py - y0 + 2) * fnt::BX + (px - x0 + 2) : fnt::BX + 1;  // the point in a box
  const int zon_lo = max(-1, -zoff), zon_hi = min(nz, nzg - 1 - zoff);
  auto on = [&](int z) { return inxy && z >= zon_lo && z <= zon_hi; };
  // plane q (>= z0 - 2) -> ring stage; a plane is read from the maps when they cover it
  // (b: gb guard planes, the coefficients: gcz) and zero-filled from far outside otherwise
  auto slot = [&](int q) { return (unsigned)(q - z0 + 2) % fnt::NS; };
  auto parity = [&](int q) { return ((unsigned)(q - z0 + 2) / fnt::NS) & 1u; };
  auto issue = [&](int q) {
    if (tid != 0 || q > z1) return;  // x1 is formed up to plane z1
    const unsigned st = slot(q);
    double* d = stg + st * fnt::STAGE;
    const int far = -(1 << 20);
    const int zb = q + gb >= 0 && q < nz + gb ? q + gb : far;
    const int zq = q + gcz >= 0 && q < nz + gcz ? q + gcz : far;
    mbar_arrive_expect(bars + st, fnt::STAGE_BYTES);
    tma_load3d(d, &mb, x0 - 2, y0 - 2, zb, bars + st);
    tma_load3d(d + fnt::BOX, &mcx, x0 - 2, y0 - 2, zq, bars + st);
    tma_load3d(d + 2 * fnt::BOX, &mcy, x0 - 2, y0 - 2, zq, bars + st);
    tma_load3d(d + 3 * fnt::BOX, &mcz, x0 - 2, y0 - 2, zq, bars + st);
  };
  auto load = [&](int q) {  // this point's values of plane q (waits for the stage)
    const unsigned st = slot(q);
    mbar_wait(bars + st, parity(q));
    const double* d = stg + st * fnt::STAGE + bo;
    FnPlane s;
    s.b = d[0];
    s.cx = d[fnt::BOX];
    s.cxm = d[fnt::BOX - 1];
    s.cy = d[2 * fnt::BOX];
    s.cym = d[2 * fnt::BOX - fnt::BX];
    s.cz = d[3 * fnt::BOX];
    return s;
  };
  auto first = [&](const FnPlane& s, double d, bool in) { return in ? 0.0 + (omega * (s.b - 0.0)) / d : 0.0; };

  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < fnt::NS; ++k) mbar_init(bars + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < fnt::NS; ++k) issue(z0 - 2 + k);
  // prologue: cz of plane z0-2, plane z0-1 (own column), plane z0 (published)
  // every thread waits for every stage it lets be re-armed (an arrive on a barrier whose phase is
  // still pending would corrupt it), so plane z0-2 is waited for even where it is not used
  const FnPlane mm = load(z0 - 2);
  const double czm = on(z0 - 1) ? mm.cz : 0.0;
  __syncthreads();  // plane z0-2's stage is read by everyone
  issue(z0 - 2 + fnt::NS);
  FnPlane m = load(z0 - 1);
  const double x1m0 = first(m, fn_diag(m, czm, eps), on(z0 - 1));
  const double czm_c0 = on(z0 - 1) ? m.cz : 0.0;
  FnPlane c = load(z0);
  if (!on(z0)) c = FnPlane{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  double czm_c = czm_c0;
  double dc = fn_diag(c, czm_c, eps);
  double x1c = first(c, dc, on(z0));
  double x1m = x1m0;
  if (act) ring[0][sr][sc] = x1c;
  __syncthreads();  // planes z0-1, z0 are read by everyone
  issue(z0 - 1 + fnt::NS);
  issue(z0 + fnt::NS);
  int rs = 0;  // ring slot of plane z
  long o = (long)z0 * nxy + (inxy ? (long)py * nx + px : 0);
#pragma unroll 1
  for (int z = z0; z < z1; ++z, o += nxy) {
    FnPlane n = load(z + 1);
    if (!on(z + 1)) n = FnPlane{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const double dn = fn_diag(n, c.cz, eps);
    const double x1n = first(n, dn, on(z + 1));
    const int ns = rs == 2 ? 0 : rs + 1;
    if (act) ring[ns][sr][sc] = x1n;
    __syncthreads();  // x1 of plane z+1 published; plane z+1's stage read by everyone
    issue(z + 1 + fnt::NS);
    if (outw) {
      double v = 0.0;
      if (ix) {
        // m_row order: z-, y-, x-, diag, x+, y+, z+
        double acc = 0.0;
        acc = acc + -czm_c * x1m;
        acc = acc + -c.cym * ring[rs][sr - 1][sc];
        acc = acc + -c.cxm * ring[rs][sr][sc - 1];
        acc = acc + dc * x1c;
        acc = acc + -c.cx * ring[rs][sr][sc + 1];
        acc = acc + -c.cy * ring[rs][sr + 1][sc];
        acc = acc + -c.cz * x1n;
        v = x1c + (omega * (c.b - acc)) / dc;
        out[o] = v;
      }
      if (seg) {
        const double s = tree32(v * (ix ? c.b : 0.0));
        if (lane == 0) seg[((long)z * ny + py) * chunks + blockIdx.x] = s;
      }
    }
    x1m = x1c;
    x1c = x1n;
    czm_c = c.cz;
    c = n;
    dc = dn;
    rs = ns;
  }
}

// 2D: the same pair on a 32 x 8 tile -- x1 on the tile plus its one-point halo ring goes to shared
// memory (x1 is 0 outside the grid, where it meets exactly-zero boundary coefficients), then the
// second sweep; D and the row sums in sweep_zm_kernel<2>'s order.  Level-0 traffic 4 + 1 words
// per point instead of 3 + 5 for the two kernels, and one launch fewer per level.
// TY = tile rows (8: one row per warp; 32: four rows per warp and a 34 x 34 x1 ring instead of
// 10 x 34 per 32 x 8 outputs -- 1.13 instead of 1.33 first-sweep points per output, a quarter of
// the blocks)
template <int TY>
__global__ void __launch_bounds__(256) sweep_fn2d_kernel(Lvl L, const double* __restrict__ b,
                                                         double* __restrict__ out, double omega,
                                                         double* __restrict__ seg, const int* gate) {
  if (gate && *gate == 0) return;
  __shared__ double xs[TY + 2][35];
  const int nx = L.nx, ny = L.ny;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * TY;
  const double eps = *L.eps;
  auto diag = [&](long i) {  // diag_at order: x-, x+, y-, y+ ; then + eps
    double d = 0.0;
    d = d + L.cx[i - 1];
    d = d + L.cx[i];
    d = d + L.cy[i - nx];
    d = d + L.cy[i];
    return d + eps;
  };
  for (int k = threadIdx.y * 32 + threadIdx.x; k < (TY + 2) * 34; k += 256) {
    const int r = k / 34, cc = k - r * 34;
    const int gx = x0 - 1 + cc, gy = y0 - 1 + r;
    double x1 = 0.0;
    if (gx >= 0 && gx < nx && gy >= 0 && gy < ny) {
      const long i = (long)gy * nx + gx;
      x1 = 0.0 + (omega * (b[i] - 0.0)) / diag(i);
    }
    xs[r][cc] = x1;
  }
  __syncthreads();
  const int tx = threadIdx.x;
  const int gx = x0 + tx;
#pragma unroll
  for (int rr = 0; rr < TY / 8; ++rr) {
    const int ty = threadIdx.y * (TY / 8) + rr;
    const int gy = y0 + ty;
    if (gy >= ny) break;  // whole warp (one row segment)
    double v = 0.0, bi = 0.0;
    if (gx < nx) {
      const long i = (long)gy * nx + gx;
      const double d = diag(i);
      bi = b[i];
      const double xc = xs[ty + 1][tx + 1];
      // m_row order: y-, x-, diag, x+, y+
      double acc = 0.0;
      acc = acc + -L.cy[i - nx] * xs[ty][tx + 1];
      acc = acc + -L.cx[i - 1] * xs[ty + 1][tx];
      acc = acc + d * xc;
      acc = acc + -L.cx[i] * xs[ty + 1][tx + 2];
      acc = acc + -L.cy[i] * xs[ty + 2][tx + 1];
      v = xc + (omega * (bi - acc)) / d;
      out[i] = v;
    }
    if (seg) {
      const double s2 = tree32(v * bi);
      if (tx == 0) seg[(long)gy * ((nx + 31) / 32) + blockIdx.x] = s2;
    }
  }
}

// z chunk minimising (waves x planes per block), chunks of >= 8 planes
static inline int fn_chunk(int nx, int ny, int nz, int sms) {
  const long bxy = (long)((nx + fn::TX - 1) / fn::TX) * ((ny + fn::TY - 1) / fn::TY);
  const long slots = (long)fn::MINB * sms;
  int best = nz;
  double best_cost = 1e30;
  for (int ch = 1; ch <= nz; ++ch) {
    const int zc = (nz + ch - 1) / ch;
    if (zc < 8 && ch > 1) break;
    const long blocks = bxy * ((nz + zc - 1) / zc);
    const long waves = (blocks + slots - 1) / slots;
    // time ~ waves of (zc + 2) planes
    const double cost = (double)waves * (zc + 2);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = zc;
    }
  }
  return best;
}
