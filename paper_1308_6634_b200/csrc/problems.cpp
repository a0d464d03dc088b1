// problems.cpp -- seeded synthetic inputs on the host (input generation is
// out of the GPU scope).  Conventions of the reference's
// problems.cpp: std::mt19937_64, u = ((x >> 11) + 1) 2^-53 (problems.cpp:17-18),
// Box-Muller pairs cos-first (problems.cpp:12-28), cell-centred coordinates,
// shapes painted in order over a zero background (problems.cpp:111-130).
// Compiled without FMA contraction, so every generated value is bit-identical
// to the oracle's independent restatement (tests/test_gpu_parity.py checks).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "../../include/mlsqr_b200.h"

namespace {

struct Uniform {
  std::mt19937_64 eng;
  explicit Uniform(uint64_t seed) : eng(seed) {}
  double operator()() { return static_cast<double>((eng() >> 11) + 1) * 0x1p-53; }
};

}  // namespace

extern "C" {

// GaussianConvolution1D taps (linop.cpp:93-102) with an explicit radius
int mlsqr_taps(size_t n, double sigma_f, double domain_length, int radius, double* taps,
               int* radius_out) {
  if (n < 1 || !(sigma_f > 0.0) || !(domain_length > 0.0)) return MLSQR_EINVAL;
  const double h = domain_length / static_cast<double>(n);
  if (radius < 0) radius = static_cast<int>(std::ceil(6.0 * sigma_f / h));
  const double norm = std::sqrt(2.0 / (M_PI * sigma_f * sigma_f));
  if (taps) {
    for (int k = 0; k < 2 * radius + 1; ++k) {
      const double d = (static_cast<double>(k) - static_cast<double>(radius)) * h;
      taps[k] = h * norm * std::exp(-d * d / (2.0 * sigma_f * sigma_f));
    }
  }
  if (radius_out) *radius_out = radius;
  return MLSQR_OK;
}

int mlsqr_gauss_fill(uint64_t seed, size_t n, double stddev, double* out) {
  Uniform u(seed);
  bool have = false;
  double spare = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double z;
    if (have) {
      have = false;
      z = spare;
    } else {
      const double u1 = u(), u2 = u();
      const double radius = std::sqrt(-2.0 * std::log(u1));
      const double angle = 2.0 * M_PI * u2;
      spare = radius * std::sin(angle);
      have = true;
      z = radius * std::cos(angle);
    }
    out[i] = stddev * z;
  }
  return MLSQR_OK;
}

int mlsqr_phantom_rects2d(size_t nx, size_t ny, int count, uint64_t seed, double* out) {
  Uniform u(seed);
  struct R { double x0, x1, y0, y1, v; };
  std::vector<R> rs;
  for (int k = 0; k < count; ++k) {
    const double xa = u(), xb = u(), ya = u(), yb = u();
    rs.push_back({std::min(xa, xb), std::max(xa, xb), std::min(ya, yb), std::max(ya, yb), u()});
  }
  const double hx = 1.0 / static_cast<double>(nx), hy = 1.0 / static_cast<double>(ny);
  for (size_t iy = 0; iy < ny; ++iy) {
    const double y = (static_cast<double>(iy) + 0.5) * hy;
    for (size_t ix = 0; ix < nx; ++ix) {
      const double x = (static_cast<double>(ix) + 0.5) * hx;
      double v = 0.0;
      for (const R& r : rs)
        if (x >= r.x0 && x <= r.x1 && y >= r.y0 && y <= r.y1) v = r.v;
      out[iy * nx + ix] = v;
    }
  }
  return MLSQR_OK;
}

int mlsqr_phantom_shapes2d(size_t nx, size_t ny, int count, uint64_t seed, double* out) {
  Uniform u(seed);
  std::vector<double> sh(6 * static_cast<size_t>(count > 0 ? count : 0));
  for (double& v : sh) v = u();
  const double hx = 1.0 / static_cast<double>(nx), hy = 1.0 / static_cast<double>(ny);
  for (size_t iy = 0; iy < ny; ++iy) {
    const double y = (static_cast<double>(iy) + 0.5) * hy;
    for (size_t ix = 0; ix < nx; ++ix) {
      const double x = (static_cast<double>(ix) + 0.5) * hx;
      double v = 0.0;
      for (int k = 0; k < count; ++k) {
        const double* r = sh.data() + 6 * k;
        const double cx = r[1], cy = r[2];
        const double a = 0.02 + 0.08 * r[3], b = 0.02 + 0.08 * r[4];
        const bool inside = r[0] < 0.5 ? (x - cx) * (x - cx) + (y - cy) * (y - cy) <= a * a
                                       : (x >= cx - a && x <= cx + a && y >= cy - b && y <= cy + b);
        if (inside) v = r[5];
      }
      out[iy * nx + ix] = v;
    }
  }
  return MLSQR_OK;
}

int mlsqr_phantom_ellipsoids3d(size_t nx, size_t ny, size_t nz, int count, double semi_lo,
                               double semi_hi, double vlo, double vhi, uint64_t seed,
                               double* out) {
  Uniform u(seed);
  std::memset(out, 0, sizeof(double) * nx * ny * nz);
  for (int k = 0; k < count; ++k) {
    const double cx = u() * static_cast<double>(nx);
    const double cy = u() * static_cast<double>(ny);
    const double cz = u() * static_cast<double>(nz);
    const double a = semi_lo + (semi_hi - semi_lo) * u();
    const double b = semi_lo + (semi_hi - semi_lo) * u();
    const double c = semi_lo + (semi_hi - semi_lo) * u();
    const double val = vlo + (vhi - vlo) * u();
    const long x0 = std::max(0L, static_cast<long>(std::floor(cx - a)) - 1);
    const long x1 = std::min(static_cast<long>(nx) - 1, static_cast<long>(std::ceil(cx + a)) + 1);
    const long y0 = std::max(0L, static_cast<long>(std::floor(cy - b)) - 1);
    const long y1 = std::min(static_cast<long>(ny) - 1, static_cast<long>(std::ceil(cy + b)) + 1);
    const long z0 = std::max(0L, static_cast<long>(std::floor(cz - c)) - 1);
    const long z1 = std::min(static_cast<long>(nz) - 1, static_cast<long>(std::ceil(cz + c)) + 1);
    for (long z = z0; z <= z1; ++z) {
      const double dz = (static_cast<double>(z) + 0.5 - cz) / c;
      for (long y = y0; y <= y1; ++y) {
        const double dy = (static_cast<double>(y) + 0.5 - cy) / b;
        for (long x = x0; x <= x1; ++x) {
          const double dx = (static_cast<double>(x) + 0.5 - cx) / a;
          if (dx * dx + dy * dy + dz * dz <= 1.0)
            out[(static_cast<size_t>(z) * ny + static_cast<size_t>(y)) * nx + static_cast<size_t>(x)] = val;
        }
      }
    }
  }
  return MLSQR_OK;
}

int mlsqr_fdot_tables(size_t n, int n_src, int n_det, double mu, uint64_t seed, double* gs,
                      double* gd) {
  Uniform u(seed);
  const size_t N = n * n * n;
  std::vector<double> src(3 * static_cast<size_t>(n_src)), det(3 * static_cast<size_t>(n_det));
  for (int k = 0; k < n_src; ++k) {
    src[3 * k] = u() * static_cast<double>(n);
    src[3 * k + 1] = u() * static_cast<double>(n);
    src[3 * k + 2] = 0.0;
  }
  for (int k = 0; k < n_det; ++k) {
    det[3 * k] = u() * static_cast<double>(n);
    det[3 * k + 1] = u() * static_cast<double>(n);
    det[3 * k + 2] = static_cast<double>(n);
  }
  const double four_pi = 4.0 * M_PI;
  for (int pass = 0; pass < 2; ++pass) {
    const int cnt = pass == 0 ? n_src : n_det;
    const double* pts = pass == 0 ? src.data() : det.data();
    double* o = pass == 0 ? gs : gd;
    for (int k = 0; k < cnt; ++k) {
      size_t i = 0;
      for (size_t z = 0; z < n; ++z)
        for (size_t y = 0; y < n; ++y)
          for (size_t x = 0; x < n; ++x, ++i) {
            const double dx = static_cast<double>(x) + 0.5 - pts[3 * k];
            const double dy = static_cast<double>(y) + 0.5 - pts[3 * k + 1];
            const double dz = static_cast<double>(z) + 0.5 - pts[3 * k + 2];
            const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
            o[static_cast<size_t>(k) * N + i] = std::exp(-mu * r) / (four_pi * r);
          }
    }
  }
  return MLSQR_OK;
}

}  // extern "C"
