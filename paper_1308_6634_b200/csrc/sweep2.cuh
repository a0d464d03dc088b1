// sweep2.cuh -- two consecutive omega-Jacobi sweeps fused in one z-marching
// kernel (included by vcycle.cu).
//
//   ZERO    : x' = 0 + (omega * (b - 0)) / D             (first pre-sweep from zero)
//   PROLONG : x' = x + P xc, then one sweep              (first post-sweep)
//   then    : out = x' + (omega * (b - M x')) / D        (second sweep, + <out, b> partials)
//
// A 512-thread CTA owns a 32 x 16 output tile and a z chunk.  Plane tiles of
// (x), b, cx, cy, cz with a 2-point halo stream through a 5-slot cp.async ring
// in shared memory (16-byte copies); x' lives in a 3-plane shared ring on the
// 1-halo region, so the intermediate iterate never touches HBM.  HBM traffic:
// read b, cx, cy, cz (+ x, xc) once, write out once -- instead of two full
// sweep passes.  Arithmetic per point is exactly diag_at / m_row (CSR
// ascending column order), so results equal the unfused kernels bit for bit.
namespace s2 {
constexpr int TX = 32, TY = 16, THREADS = 512;
constexpr int W2 = TX + 4, H2 = TY + 4;  // 2-halo input region
constexpr int W1 = TX + 2, H1 = TY + 2;  // 1-halo intermediate region
constexpr int N2 = W2 * H2, N1 = W1 * H1;
constexpr int NSLOT = 5;
constexpr int PAIRS = N2 / 2;  // 16-byte copies per array per plane
}  // namespace s2

template <bool PROLONG>
__global__ void __launch_bounds__(512, 1) sweep2_kernel(Lvl L, const double* __restrict__ x,
                                                        const double* __restrict__ xc, int cnx, int cny,
                                                        const double* __restrict__ b,
                                                        double* __restrict__ out, double omega,
                                                        double* __restrict__ seg, const int* gate, int zc) {
  using namespace s2;
  if (gate && *gate == 0) return;
  constexpr int NA = PROLONG ? 5 : 4;  // arrays per plane: [x,] b, cx, cy, cz
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;                              // [NSLOT][NA][N2]
  double* xr = sm + (size_t)NSLOT * NA * N2;      // [3][N1] intermediate x'
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(L.nz, z0 + zc);
  const bool hy = L.cy != nullptr, hz = L.cz != nullptr;
  const int nx = L.nx, ny = L.ny, nz = L.nz;
  const size_t nxy = (size_t)nx * ny;
  const double eps = *L.eps;
  const int base = z0 - 2;
  // array ids inside a slot
  constexpr int AX = 0, AB = PROLONG ? 1 : 0, ACX = AB + 1, ACY = AB + 2, ACZ = AB + 3;
  auto arr = [&](int plane, int a) -> double* {
    return ring + ((size_t)((plane - base) % NSLOT) * NA + a) * N2;
  };
  // one 16-byte pair per thread per array (PAIRS = 360 <= 512)
  const bool cp_on = tid < PAIRS;
  const int cly = tid / (W2 / 2), clx = 2 * (tid - cly * (W2 / 2));
  const int cgx = x0 - 2 + clx, cgy = y0 - 2 + cly;
  const bool cok = cp_on && cgx >= 0 && cgx < nx && cgy >= 0 && cgy < ny;
  const long coff = cok ? (long)cgy * nx + cgx : 0;
  auto issue = [&](int plane) {
    if (cp_on && plane >= 0 && plane < nz && plane <= z1 + 1) {
      const size_t po = (size_t)plane * nxy;
      const int so = cly * W2 + clx;
      const double* src[5];
      int na = 0;
      if (PROLONG) src[na++] = x;
      src[na++] = b;
      src[na++] = L.cx;
      src[na++] = hy ? L.cy : L.cx;
      src[na++] = hz ? L.cz : L.cx;
#pragma unroll
      for (int a = 0; a < NA; ++a) cp_async16(arr(plane, a) + so, cok ? src[a] + po + coff : b, cok);
    }
    cp_async_commit();
  };
  // add the coarse correction to a freshly landed x plane (PROLONG), in place
  auto prolong_plane = [&](int plane) {
    if (!PROLONG || plane < 0 || plane >= nz) return;
    double* xs = arr(plane, AX);
    const int Z = hz ? plane / 2 : 0;
    for (int k = tid; k < N2; k += THREADS) {
      const int ly = k / W2, lx = k - ly * W2;
      const int gx = x0 - 2 + lx, gy = y0 - 2 + ly;
      if (gx >= 0 && gx < nx && gy >= 0 && gy < ny) {
        const int Y = hy ? gy / 2 : 0;
        xs[k] = xs[k] + xc[((size_t)Z * cny + Y) * cnx + gx / 2];
      }
    }
  };

  issue(base);
  issue(base + 1);
  issue(base + 2);
  cp_async_wait<0>();
  __syncthreads();
  prolong_plane(base);
  prolong_plane(base + 1);
  prolong_plane(base + 2);
  const size_t chunks = (size_t)(nx + 31) / 32;

  for (int p = z0 - 1; p <= z1; ++p) {
    issue(p + 2);
    cp_async_wait<1>();
    __syncthreads();
    if (p > z0 - 1) prolong_plane(p + 1);
    if (PROLONG) __syncthreads();
    // ---- stage 1: x' at plane p on the 1-halo region
    if (p >= 0 && p < nz) {
      const double* cxp = arr(p, ACX);
      const double* cyp = arr(p, ACY);
      const double* czp = arr(p, ACZ);
      const double* czm = (hz && p > 0) ? arr(p - 1, ACZ) : czp;
      const double* bp = arr(p, AB);
      const double* xp = PROLONG ? arr(p, AX) : nullptr;
      const double* xm = (PROLONG && hz && p > 0) ? arr(p - 1, AX) : xp;
      const double* xn = (PROLONG && hz && p + 1 < nz) ? arr(p + 1, AX) : xp;
      double* xo = xr + (size_t)(p % 3) * N1;
      for (int k = tid; k < N1; k += THREADS) {
        const int ly = k / W1, lx = k - ly * W1;
        const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
        if (gx < 0 || gx >= nx || gy < 0 || gy >= ny) continue;
        const int j = (ly + 1) * W2 + (lx + 1);
        double d = 0.0;
        if (gx > 0) d = d + cxp[j - 1];
        if (gx + 1 < nx) d = d + cxp[j];
        if (hy) {
          if (gy > 0) d = d + cyp[j - W2];
          if (gy + 1 < ny) d = d + cyp[j];
        }
        if (hz) {
          if (p > 0) d = d + czm[j];
          if (p + 1 < nz) d = d + czp[j];
        }
        d = d + eps;
        double v;
        if (!PROLONG) {
          const double mx = 0.0;
          v = 0.0 + (omega * (bp[j] - mx)) / d;
        } else {
          double acc = 0.0;
          if (hz && p > 0) acc = acc + -czm[j] * xm[j];
          if (hy && gy > 0) acc = acc + -cyp[j - W2] * xp[j - W2];
          if (gx > 0) acc = acc + -cxp[j - 1] * xp[j - 1];
          acc = acc + d * xp[j];
          if (gx + 1 < nx) acc = acc + -cxp[j] * xp[j + 1];
          if (hy && gy + 1 < ny) acc = acc + -cyp[j] * xp[j + W2];
          if (hz && p + 1 < nz) acc = acc + -czp[j] * xn[j];
          v = xp[j] + (omega * (bp[j] - acc)) / d;
        }
        xo[k] = v;
      }
    }
    __syncthreads();
    // ---- stage 2: out at plane q = p - 1 (or q = p without a z dimension)
    const int q = hz ? p - 1 : p;
    if (q >= z0 && q < z1 && (hz || p < nz)) {
      const double* cxq = arr(q, ACX);
      const double* cyq = arr(q, ACY);
      const double* czq = arr(q, ACZ);
      const double* czm = (hz && q > 0) ? arr(q - 1, ACZ) : czq;
      const double* bq = arr(q, AB);
      const double* xq = xr + (size_t)(q % 3) * N1;
      const double* xm = (hz && q > 0) ? xr + (size_t)((q + 2) % 3) * N1 : xq;
      const double* xn = (hz && q + 1 < nz) ? xr + (size_t)((q + 1) % 3) * N1 : xq;
      const int lx = tid & 31, ly = tid >> 5;  // 32 x 16 outputs, one per thread
      const int gx = x0 + lx, gy = y0 + ly;
      double v = 0.0, bi = 0.0;
      if (gx < nx && gy < ny) {
        const int j = (ly + 2) * W2 + (lx + 2);
        const int k = (ly + 1) * W1 + (lx + 1);
        bi = bq[j];
        double d = 0.0;
        if (gx > 0) d = d + cxq[j - 1];
        if (gx + 1 < nx) d = d + cxq[j];
        if (hy) {
          if (gy > 0) d = d + cyq[j - W2];
          if (gy + 1 < ny) d = d + cyq[j];
        }
        if (hz) {
          if (q > 0) d = d + czm[j];
          if (q + 1 < nz) d = d + czq[j];
        }
        d = d + eps;
        double acc = 0.0;
        if (hz && q > 0) acc = acc + -czm[j] * xm[k];
        if (hy && gy > 0) acc = acc + -cyq[j - W2] * xq[k - W1];
        if (gx > 0) acc = acc + -cxq[j - 1] * xq[k - 1];
        acc = acc + d * xq[k];
        if (gx + 1 < nx) acc = acc + -cxq[j] * xq[k + 1];
        if (hy && gy + 1 < ny) acc = acc + -cyq[j] * xq[k + W1];
        if (hz && q + 1 < nz) acc = acc + -czq[j] * xn[k];
        v = xq[k] + (omega * (bi - acc)) / d;
        out[(size_t)q * nxy + (size_t)gy * nx + gx] = v;
      }
      if (seg && gy < ny) {
        const double s = tree32(v * bi);
        if (lx == 0) seg[((size_t)q * ny + gy) * chunks + blockIdx.x] = s;
      }
    }
    __syncthreads();
  }
}

static inline int sweep2_chunk(int nx, int ny, int nz, int sms) {
  const long bxy = (long)((nx + s2::TX - 1) / s2::TX) * ((ny + s2::TY - 1) / s2::TY);
  long chunks = (sms * 8L + bxy - 1) / bxy;
  if (chunks < 1) chunks = 1;
  int zc = (int)((nz + chunks - 1) / chunks);
  if (zc < 4) zc = 4;
  return zc > nz ? nz : zc;
}

static inline size_t sweep2_smem(bool prolong) {
  return sizeof(double) * ((size_t)s2::NSLOT * (prolong ? 5 : 4) * s2::N2 + 3 * (size_t)s2::N1);
}
