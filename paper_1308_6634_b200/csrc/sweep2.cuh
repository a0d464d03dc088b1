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
// 1-halo region, so the intermediate iterate never touches HBM.
//
// Bit-exactness with diag_at / m_row (CSR ascending column order): the halo
// is zero-filled and a missing edge has an exactly-zero coefficient, so the
// in-plane terms are added unconditionally -- acc + (+-0) == acc because the
// accumulators start at +0 and can never become -0 -- and out-of-range planes
// read a zero plane.  Only the order of the additions matters, and it is the
// reference's.  x' outside the domain is forced to 0 (never NaN).
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
  constexpr int AX = 0, AB = PROLONG ? 1 : 0, ACX = AB + 1, ACY = AB + 2, ACZ = AB + 3;
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;                                // [NSLOT][NA][N2]
  double* xr = ring + (size_t)NSLOT * NA * N2;      // [3][N1] intermediate x'
  double* zero = xr + 3 * N1;                       // [N2] zeros (planes outside the domain)
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(L.nz, z0 + zc);
  const bool hy = L.cy != nullptr, hz = L.cz != nullptr;
  const int nx = L.nx, ny = L.ny, nz = L.nz;
  const size_t nxy = (size_t)nx * ny;
  const double eps = *L.eps;
  const int base = z0 - 2;
  for (int k = tid; k < N2; k += THREADS) zero[k] = 0.0;

  // ---- per-thread constant descriptors
  // cp.async: one 16-byte pair per array per plane (PAIRS = 360 <= 512 threads)
  const bool cp_on = tid < PAIRS;
  const int cly = tid / (W2 / 2), clx = 2 * (tid - cly * (W2 / 2));
  const int cgx = x0 - 2 + clx, cgy = y0 - 2 + cly;
  const bool cok = cp_on && cgx >= 0 && cgx < nx && cgy >= 0 && cgy < ny;
  const long coff = cok ? (long)cgy * nx + cgx : 0;
  const int cso = cly * W2 + clx;
  // stage-1 points (1-halo region, N1 = 612): k = tid and tid + 512
  int s1k[2], s1j[2];
  bool s1in[2], s1on[2];
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int k = tid + m * THREADS;
    s1on[m] = k < N1;
    const int ly = k / W1, lx = k - ly * W1;
    const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
    s1in[m] = s1on[m] && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
    s1k[m] = k;
    s1j[m] = (ly + 1) * W2 + (lx + 1);
  }
  // prolongation targets of this thread in the 2-halo region (N2 = 720): k = tid, tid + 512
  int prk[2];
  long prc[2];
  bool pron[2];
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int k = tid + m * THREADS;
    const int ly = k / W2, lx = k - ly * W2;
    const int gx = x0 - 2 + lx, gy = y0 - 2 + ly;
    pron[m] = k < N2 && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
    prk[m] = k;
    prc[m] = pron[m] ? (long)(hy ? gy / 2 : 0) * cnx + gx / 2 : 0;
  }
  // stage-2 output of this thread
  const int olx = tid & 31, oly = tid >> 5;
  const int ogx = x0 + olx, ogy = y0 + oly;
  const bool oin = ogx < nx && ogy < ny;
  const int oj = (oly + 2) * W2 + (olx + 2), ok1 = (oly + 1) * W1 + (olx + 1);
  const size_t ooff = (size_t)ogy * nx + ogx;
  const size_t chunks = (size_t)(nx + 31) / 32;

  auto slot = [&](int plane) -> double* { return ring + (size_t)((plane - base) % NSLOT) * NA * N2; };
  auto issue = [&](int plane) {
    if (cp_on && plane >= 0 && plane < nz && plane <= z1 + 1) {
      double* d = slot(plane) + cso;
      const size_t po = (size_t)plane * nxy + coff;
      if (PROLONG) cp_async16(d + AX * N2, cok ? x + po : b, cok);
      cp_async16(d + AB * N2, cok ? b + po : b, cok);
      cp_async16(d + ACX * N2, cok ? L.cx + po : b, cok);
      if (hy) cp_async16(d + ACY * N2, cok ? L.cy + po : b, cok);
      if (hz) cp_async16(d + ACZ * N2, cok ? L.cz + po : b, cok);
    }
    cp_async_commit();
  };
  auto prolong_plane = [&](int plane) {
    if (!PROLONG || plane < 0 || plane >= nz) return;
    double* xs = slot(plane) + AX * N2;
    const size_t zo = (size_t)(hz ? plane / 2 : 0) * cny * cnx;
#pragma unroll
    for (int m = 0; m < 2; ++m)
      if (pron[m]) xs[prk[m]] = xs[prk[m]] + xc[zo + prc[m]];
  };
  // array of a plane, or the zero plane outside [0, nz)
  auto A = [&](int plane, int a) -> const double* {
    return (plane >= 0 && plane < nz) ? slot(plane) + a * N2 : zero;
  };
  if (!hy || !hz) {
    // missing axes read the zero plane through ACY / ACZ: clear those slots once
    for (int s = 0; s < NSLOT; ++s) {
      double* d = ring + (size_t)s * NA * N2;
      for (int k = tid; k < N2; k += THREADS) {
        if (!hy) d[ACY * N2 + k] = 0.0;
        if (!hz) d[ACZ * N2 + k] = 0.0;
      }
    }
    __syncthreads();
  }

  issue(base);
  issue(base + 1);
  issue(base + 2);
  cp_async_wait<0>();
  __syncthreads();
  prolong_plane(base);
  prolong_plane(base + 1);
  prolong_plane(base + 2);

  for (int p = z0 - 1; p <= z1; ++p) {
    issue(p + 2);
    cp_async_wait<1>();
    __syncthreads();
    if (PROLONG) {
      if (p > z0 - 1) prolong_plane(p + 1);
      __syncthreads();
    }
    // ---- stage 1: x' at plane p on the 1-halo region
    if (p >= 0 && p < nz) {
      const double* cxp = A(p, ACX);
      const double* cyp = A(p, ACY);
      const double* czp = (p + 1 < nz) ? A(p, ACZ) : zero;  // no +z edge on the last plane
      const double* czm = A(p - 1, ACZ);
      const double* bp = A(p, AB);
      const double* xp = PROLONG ? A(p, AX) : zero;
      const double* xm = PROLONG ? A(p - 1, AX) : zero;
      const double* xn = PROLONG ? A(p + 1, AX) : zero;
      double* xo = xr + (size_t)(p % 3) * N1;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        if (!s1on[m]) continue;
        const int j = s1j[m];
        double v = 0.0;
        if (s1in[m]) {
          double d = 0.0;
          d = d + cxp[j - 1];
          d = d + cxp[j];
          d = d + cyp[j - W2];
          d = d + cyp[j];
          d = d + czm[j];
          d = d + czp[j];
          d = d + eps;
          const double bj = bp[j];
          if (!PROLONG) {
            const double mx = 0.0;
            v = 0.0 + (omega * (bj - mx)) / d;
          } else {
            double acc = 0.0;
            acc = acc + -czm[j] * xm[j];
            acc = acc + -cyp[j - W2] * xp[j - W2];
            acc = acc + -cxp[j - 1] * xp[j - 1];
            acc = acc + d * xp[j];
            acc = acc + -cxp[j] * xp[j + 1];
            acc = acc + -cyp[j] * xp[j + W2];
            acc = acc + -czp[j] * xn[j];
            v = xp[j] + (omega * (bj - acc)) / d;
          }
        }
        xo[s1k[m]] = v;
      }
    }
    __syncthreads();
    // ---- stage 2: out at plane q = p - 1 (q = p without a z dimension)
    const int q = hz ? p - 1 : p;
    if (q >= z0 && q < z1 && q < nz) {
      const double* cxq = A(q, ACX);
      const double* cyq = A(q, ACY);
      const double* czq = (q + 1 < nz) ? A(q, ACZ) : zero;
      const double* czm = A(q - 1, ACZ);
      const double* bq = A(q, AB);
      const double* xq = xr + (size_t)(q % 3) * N1;
      const double* xm = (hz && q > 0) ? xr + (size_t)((q + 2) % 3) * N1 : zero;
      const double* xn = (hz && q + 1 < nz) ? xr + (size_t)((q + 1) % 3) * N1 : zero;
      double v = 0.0, bi = 0.0;
      if (oin) {
        const int j = oj, k = ok1;
        bi = bq[j];
        double d = 0.0;
        d = d + cxq[j - 1];
        d = d + cxq[j];
        d = d + cyq[j - W2];
        d = d + cyq[j];
        d = d + czm[j];
        d = d + czq[j];
        d = d + eps;
        double acc = 0.0;
        acc = acc + -czm[j] * xm[k];
        acc = acc + -cyq[j - W2] * xq[k - W1];
        acc = acc + -cxq[j - 1] * xq[k - 1];
        acc = acc + d * xq[k];
        acc = acc + -cxq[j] * xq[k + 1];
        acc = acc + -cyq[j] * xq[k + W1];
        acc = acc + -czq[j] * xn[k];
        v = xq[k] + (omega * (bi - acc)) / d;
        out[(size_t)q * nxy + ooff] = v;
      }
      if (seg && ogy < ny) {
        const double s = tree32(v * bi);
        if (olx == 0) seg[((size_t)q * ny + ogy) * chunks + blockIdx.x] = s;
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
  return sizeof(double) * ((size_t)s2::NSLOT * (prolong ? 5 : 4) * s2::N2 + 3 * (size_t)s2::N1 + s2::N2);
}
