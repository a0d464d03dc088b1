/*
 * oracle/mlsqr_oracle.c -- TEST INFRASTRUCTURE ONLY (see mlsqr_oracle.h).
 *
 * Plain C99 restatement of the reference path.  Every reduction is a plain
 * ascending scalar loop, i.e. the semantics of the reference's scalar BLAS-1
 * backend (kernels_scalar.cpp:7-23, selected by MLSQR_KERNELS=scalar).
 * Never linked into the product library.
 */
#include "mlsqr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ======================================================================== */
/* arithmetic order                                                          */
/* ======================================================================== */

/* REFERENCE order (default): ascending scalar sums, libm hypot -- bit-exact
 * with the reference's scalar backend.  DEVICE order: the canonical order the
 * CUDA product implements:
 *   - dot / nrm2 / penalty sums: 32-element row segments reduced by a
 *     shuffle-down tree (lane l += lane l+off, off = 16,8,4,2,1), then
 *     repeated tree-32 levels over consecutive partials (zero padded);
 *   - dense adjoint: rows split in 8 fixed chunks, sequential within a chunk,
 *     chunk partials summed in order;
 *   - hypot(a,b) = max * sqrt(1 + (min/max)^2);
 * every other operation is identical in both orders. */
static int g_device = 0;
void orc_set_device_order(int on) { g_device = on; }
int orc_get_device_order(void) { return g_device; }

static double tree32(double* v) {
  for (int off = 16; off >= 1; off >>= 1)
    for (int l = 0; l < off; ++l) v[l] = v[l] + v[l + off];
  return v[0];
}

/* repeated tree-32 levels until one value remains (at least one level) */
static double canon_reduce(double* work, size_t J) {
  if (J == 0) return 0.0;
  do {
    const size_t G = (J + 31) / 32;
    for (size_t g = 0; g < G; ++g) {
      double v[32];
      for (int l = 0; l < 32; ++l) {
        const size_t k = 32 * g + (size_t)l;
        v[l] = k < J ? work[k] : 0.0;
      }
      work[g] = tree32(v);
    }
    J = G;
  } while (J > 1);
  return work[0];
}

/* canonical sum of per-element values produced by fn(i) over rows of length L */
typedef double (*elem_fn)(const void* ctx, size_t i);
static double canon_sum(elem_fn fn, const void* ctx, size_t n, size_t L) {
  if (n == 0) return 0.0;
  if (L == 0 || n % L) L = n;
  const size_t rows = n / L, chunks = (L + 31) / 32;
  double* S = (double*)malloc(sizeof(double) * rows * chunks);
  size_t j = 0;
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < chunks; ++c, ++j) {
      double v[32];
      for (int l = 0; l < 32; ++l) {
        const size_t x = 32 * c + (size_t)l;
        v[l] = x < L ? fn(ctx, r * L + x) : 0.0;
      }
      S[j] = tree32(v);
    }
  const double out = canon_reduce(S, j);
  free(S);
  return out;
}

typedef struct { const double *x, *y; } dot_ctx;
static double dot_elem(const void* c, size_t i) {
  const dot_ctx* d = (const dot_ctx*)c;
  return d->x[i] * d->y[i];
}

double orc_canon_dot(const double* x, const double* y, size_t n, size_t L) {
  dot_ctx c = {x, y};
  return canon_sum(dot_elem, &c, n, L);
}

/* deterministic hypot built from IEEE basic operations only */
double orc_dhypot(double a, double b) {
  a = fabs(a);
  b = fabs(b);
  if (a < b) {
    const double t = a;
    a = b;
    b = t;
  }
  if (a == 0.0) return 0.0;
  if (isinf(a)) return a;
  const double r = b / a;
  return a * sqrt(1.0 + r * r);
}

static double hyp(double a, double b) { return g_device ? orc_dhypot(a, b) : hypot(a, b); }

/* ======================================================================== */
/* RNG                                                                       */
/* ======================================================================== */

/* std::mt19937_64 (published parameters; bit-specified by the C++ standard). */
void orc_mt64_seed(orc_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  s->mti = 312;
}

uint64_t orc_mt64_next(orc_mt64* s) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* problems.cpp:17-18 */
double orc_uniform(orc_mt64* s) { return (double)((orc_mt64_next(s) >> 11) + 1) * 0x1p-53; }

/* GaussianSampler::next / fill (problems.cpp:12-32): Box-Muller pairs, cos first. */
void orc_gauss_fill(uint64_t seed, size_t n, double stddev, double* out) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  int have_spare = 0;
  double spare = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double z;
    if (have_spare) {
      have_spare = 0;
      z = spare;
    } else {
      const double u1 = orc_uniform(&s);
      const double u2 = orc_uniform(&s);
      const double radius = sqrt(-2.0 * log(u1));
      const double angle = 2.0 * M_PI * u2;
      spare = radius * sin(angle);
      have_spare = 1;
      z = radius * cos(angle);
    }
    out[i] = stddev * z;
  }
}

/* ======================================================================== */
/* penalty (penalty.cpp:35-84)                                               */
/* ======================================================================== */

double orc_r_value(int kind, double T, double t) {
  switch (kind) {
    case ORC_PEN_TIKHONOV: return 0.5 * t * t;
    case ORC_PEN_TV: return hyp(T, t);
    case ORC_PEN_PM_LOG: {
      const double u = t / T;
      return 0.5 * T * T * log1p(u * u);
    }
    case ORC_PEN_PM_EXP: {
      const double u = t / T;
      return 0.5 * T * T * (1.0 - exp(-u * u));
    }
  }
  return 0.0;
}

double orc_diffusivity(int kind, double T, double t) {
  double c = 1.0;
  switch (kind) {
    case ORC_PEN_TIKHONOV: return 1.0;
    case ORC_PEN_TV: c = 1.0 / hyp(T, t); break;
    case ORC_PEN_PM_LOG: {
      const double u = t / T;
      c = u > 1e8 ? (T / t) * (T / t) : 1.0 / (1.0 + u * u);
      break;
    }
    case ORC_PEN_PM_EXP: {
      const double u = t / T;
      c = exp(-u * u);
      break;
    }
  }
  const double dmin = 2.2250738585072014e-308; /* DBL_MIN, penalty.cpp:83 */
  return c > dmin ? c : dmin;
}

/* ======================================================================== */
/* taps + operators (linop.cpp:64-170)                                       */
/* ======================================================================== */

int orc_taps(size_t n, double sigma_f, double domain_length, int radius, double* taps_out) {
  const double h = domain_length / (double)n;
  if (radius < 0) radius = (int)ceil(6.0 * sigma_f / h);
  const double norm = sqrt(2.0 / (M_PI * sigma_f * sigma_f));
  if (taps_out) {
    for (int k = 0; k < 2 * radius + 1; ++k) {
      const double d = ((double)k - (double)radius) * h;
      taps_out[k] = h * norm * exp(-d * d / (2.0 * sigma_f * sigma_f));
    }
  }
  return radius;
}

enum { OP_IDENTITY = 0, OP_DENSE = 1, OP_BLUR = 2 };

struct orc_linop {
  int kind;
  size_t rows, cols;
  const double* a;   /* dense, borrowed */
  int dims;
  size_t nx, ny, nz;
  int radius;
  double* taps;
  size_t data_len, sol_len; /* row lengths for the canonical reductions */
};

orc_linop* orc_identity_new(size_t n) {
  orc_linop* op = (orc_linop*)calloc(1, sizeof(orc_linop));
  op->kind = OP_IDENTITY;
  op->rows = op->cols = n;
  op->data_len = op->sol_len = n;
  return op;
}

orc_linop* orc_dense_new(size_t rows, size_t cols, const double* row_major) {
  orc_linop* op = (orc_linop*)calloc(1, sizeof(orc_linop));
  op->kind = OP_DENSE;
  op->rows = rows;
  op->cols = cols;
  op->a = row_major;
  op->data_len = rows;
  op->sol_len = cols;
  return op;
}

orc_linop* orc_blur_new(int dims, size_t nx, size_t ny, size_t nz, int radius,
                        const double* taps) {
  orc_linop* op = (orc_linop*)calloc(1, sizeof(orc_linop));
  op->kind = OP_BLUR;
  op->dims = dims;
  op->nx = nx;
  op->ny = dims >= 2 ? ny : 1;
  op->nz = dims >= 3 ? nz : 1;
  op->rows = op->cols = op->nx * op->ny * op->nz;
  op->radius = radius;
  op->data_len = op->sol_len = op->nx;
  op->taps = (double*)malloc(sizeof(double) * (size_t)(2 * radius + 1));
  memcpy(op->taps, taps, sizeof(double) * (size_t)(2 * radius + 1));
  return op;
}

void orc_linop_free(orc_linop* op) {
  if (!op) return;
  free(op->taps);
  free(op);
}

void orc_linop_set_row_lengths(orc_linop* op, size_t data_len, size_t sol_len) {
  op->data_len = data_len;
  op->sol_len = sol_len;
}

size_t orc_linop_rows(const orc_linop* op) { return op->rows; }
size_t orc_linop_cols(const orc_linop* op) { return op->cols; }

/* GaussianConvolution1D::convolve (linop.cpp:115-121): zero extension, ascending dot. */
static void conv_line_f(const double* taps, int R, size_t n, const double* x, size_t xs, double* y,
                        size_t ys, int use_fma) {
  for (size_t i = 0; i < n; ++i) {
    const size_t lo = i >= (size_t)R ? i - (size_t)R : 0;
    const size_t hi = (i + (size_t)R < n - 1) ? i + (size_t)R : n - 1;
    const double* t = taps + ((size_t)R + lo - i);
    double acc = 0.0;
    if (use_fma) {
      for (size_t j = lo; j <= hi; ++j) acc = fma(t[j - lo], x[j * xs], acc);
    } else {
      for (size_t j = lo; j <= hi; ++j) acc += t[j - lo] * x[j * xs];
    }
    y[i * ys] = acc;
  }
}

/* DEVICE order for 3D blurs (no reference implementation exists): every tap sum is an
 * fma chain in ascending source index; 1D/2D keep the reference's mul+add order. */
static int g_conv_fma = 0;
static void conv_line(const double* taps, int R, size_t n, const double* x, size_t xs, double* y,
                      size_t ys) {
  conv_line_f(taps, R, n, x, xs, y, ys, g_conv_fma);
}

/* SeparableGaussianBlur2D::blur (linop.cpp:151-162): x rows, then y columns, then (3D) z. */
static void blur_apply(const orc_linop* op, const double* in, double* out) {
  g_conv_fma = g_device && op->dims == 3;
  const size_t nx = op->nx, ny = op->ny, nz = op->nz;
  const size_t nxy = nx * ny;
  for (size_t z = 0; z < nz; ++z)
    for (size_t y = 0; y < ny; ++y)
      conv_line(op->taps, op->radius, nx, in + z * nxy + y * nx, 1, out + z * nxy + y * nx, 1);
  size_t maxn = ny > nz ? ny : nz;
  double* col = (double*)malloc(sizeof(double) * maxn);
  double* conv = (double*)malloc(sizeof(double) * maxn);
  if (op->dims >= 2) {
    for (size_t z = 0; z < nz; ++z)
      for (size_t x = 0; x < nx; ++x) {
        double* base = out + z * nxy + x;
        for (size_t j = 0; j < ny; ++j) col[j] = base[j * nx];
        conv_line(op->taps, op->radius, ny, col, 1, conv, 1);
        for (size_t j = 0; j < ny; ++j) base[j * nx] = conv[j];
      }
  }
  if (op->dims >= 3) {
    for (size_t y = 0; y < ny; ++y)
      for (size_t x = 0; x < nx; ++x) {
        double* base = out + y * nx + x;
        for (size_t j = 0; j < nz; ++j) col[j] = base[j * nxy];
        conv_line(op->taps, op->radius, nz, col, 1, conv, 1);
        for (size_t j = 0; j < nz; ++j) base[j * nxy] = conv[j];
      }
  }
  free(col);
  free(conv);
}

void orc_linop_apply(const orc_linop* op, const double* x, double* y) {
  switch (op->kind) {
    case OP_IDENTITY: memcpy(y, x, sizeof(double) * op->rows); break;
    case OP_DENSE:  /* DenseOperator::do_apply (linop.cpp:71-76) */
      for (size_t i = 0; i < op->rows; ++i) {
        const double* row = op->a + i * op->cols;
        if (g_device) {
          y[i] = orc_canon_dot(row, x, op->cols, op->cols);
          continue;
        }
        double acc = 0.0;
        for (size_t j = 0; j < op->cols; ++j) acc += row[j] * x[j];
        y[i] = acc;
      }
      break;
    case OP_BLUR: blur_apply(op, x, y); break;
  }
}

void orc_linop_adjoint(const orc_linop* op, const double* y, double* x) {
  switch (op->kind) {
    case OP_IDENTITY: memcpy(x, y, sizeof(double) * op->rows); break;
    case OP_DENSE:  /* DenseOperator::do_apply_adjoint (linop.cpp:78-84) */
      if (g_device && op->rows % 8 == 0) {
        /* 8 fixed row chunks, sequential inside, chunk partials summed in order:
         * x[j] = ((0 + acc_0[j]) + acc_1[j]) + ...,  acc_c[j] = (0 + y[i0] a[i0][j]) + y[i0+1] a[i0+1][j] + ...
         * The loops run row-major (the per-column operation sequence is unchanged), so the
         * matrix streams once per chunk instead of being walked column by column. */
        const size_t ch = op->rows / 8;
        double* acc = (double*)malloc(sizeof(double) * op->cols);
        for (size_t j = 0; j < op->cols; ++j) x[j] = 0.0;
        for (size_t c = 0; c < 8; ++c) {
          for (size_t j = 0; j < op->cols; ++j) acc[j] = 0.0;
          for (size_t i = c * ch; i < (c + 1) * ch; ++i) {
            const double yi = y[i];
            const double* row = op->a + i * op->cols;
            for (size_t j = 0; j < op->cols; ++j) acc[j] += yi * row[j];
          }
          for (size_t j = 0; j < op->cols; ++j) x[j] += acc[j];
        }
        free(acc);
        break;
      }
      for (size_t j = 0; j < op->cols; ++j) x[j] = 0.0;
      for (size_t i = 0; i < op->rows; ++i) {
        const double* row = op->a + i * op->cols;
        const double yi = y[i];
        for (size_t j = 0; j < op->cols; ++j) x[j] += yi * row[j];
      }
      break;
    case OP_BLUR: blur_apply(op, y, x); break; /* self-adjoint (linop.cpp:168-170) */
  }
}

/* ======================================================================== */
/* edge-based M (diffusion.cpp:27-106, sparse.cpp:65-74)                     */
/* ======================================================================== */

static int grid_ok(const orc_grid* g) {
  if (g->dims < 1 || g->dims > 3) return ORC_EINVAL;
  if (g->nx < 2 || (g->dims >= 2 && g->ny < 2) || (g->dims >= 3 && g->nz < 2)) return ORC_EDIM;
  if (!(g->h > 0.0)) return ORC_EINVAL;
  return ORC_OK;
}

static void grid_ext(const orc_grid* g, size_t* nx, size_t* ny, size_t* nz) {
  *nx = g->nx;
  *ny = g->dims >= 2 ? g->ny : 1;
  *nz = g->dims >= 3 ? g->nz : 1;
}

/* w_e / h^2 with w_e = h^dims (grid.hpp:23-25 extended to 3D) */
static double edge_scale(const orc_grid* g) {
  const double h = g->h;
  double w = h;
  if (g->dims >= 2) w = h * h;
  if (g->dims >= 3) w = h * h * h;
  return w / (h * h);
}

int orc_edge_coeffs(const orc_grid* g, const double* f, int kind, double T, double* cx,
                    double* cy, double* cz) {
  int st = grid_ok(g);
  if (st) return st;
  size_t nx, ny, nz;
  grid_ext(g, &nx, &ny, &nz);
  const double h = g->h, scale = edge_scale(g);
  const size_t nxy = nx * ny;
  for (size_t z = 0; z < nz; ++z)
    for (size_t y = 0; y < ny; ++y)
      for (size_t x = 0; x < nx; ++x) {
        const size_t i = z * nxy + y * nx + x;
        if (cx) cx[i] = x + 1 < nx ? orc_diffusivity(kind, T, fabs((f[i + 1] - f[i]) / h)) * scale : 0.0;
        if (cy) cy[i] = y + 1 < ny ? orc_diffusivity(kind, T, fabs((f[i + nx] - f[i]) / h)) * scale : 0.0;
        if (cz) cz[i] = z + 1 < nz ? orc_diffusivity(kind, T, fabs((f[i + nxy] - f[i]) / h)) * scale : 0.0;
      }
  return ORC_OK;
}

/* Diagonal in the triplet accumulation order of from_triplets: x-edges are
 * enumerated before y-edges (before z-edges), each in row-major order, so
 * node i receives c(i-1,i), c(i,i+1), c(i-nx,i), c(i,i+nx), c(i-nxy,i), c(i,i+nxy). */
static double diag_at(size_t nx, size_t ny, size_t nz, size_t x, size_t y, size_t z, size_t i,
                      const double* cx, const double* cy, const double* cz) {
  const size_t nxy = nx * ny;
  double d = 0.0;
  if (x > 0) d += cx[i - 1];
  if (x + 1 < nx) d += cx[i];
  if (cy) {
    if (y > 0) d += cy[i - nx];
    if (y + 1 < ny) d += cy[i];
  }
  if (cz) {
    if (z > 0) d += cz[i - nxy];
    if (z + 1 < nz) d += cz[i];
  }
  return d;
}

double orc_max_diag(const orc_grid* g, const double* cx, const double* cy, const double* cz) {
  size_t nx, ny, nz;
  grid_ext(g, &nx, &ny, &nz);
  if (g->dims < 2) cy = NULL;
  if (g->dims < 3) cz = NULL;
  double m = 0.0;
  size_t i = 0;
  for (size_t z = 0; z < nz; ++z)
    for (size_t y = 0; y < ny; ++y)
      for (size_t x = 0; x < nx; ++x, ++i) {
        const double d = diag_at(nx, ny, nz, x, y, z, i, cx, cy, cz);
        if (d > m) m = d;
      }
  return m;
}

/* one stencil row in ascending column order (sparse.cpp:65-74) */
static inline double m_row(size_t nx, size_t ny, size_t nz, size_t x, size_t y, size_t z,
                           size_t i, const double* cx, const double* cy, const double* cz,
                           double eps, const double* v) {
  const size_t nxy = nx * ny;
  const double diag = diag_at(nx, ny, nz, x, y, z, i, cx, cy, cz) + eps;
  double acc = 0.0;
  if (cz && z > 0) acc += -cz[i - nxy] * v[i - nxy];
  if (cy && y > 0) acc += -cy[i - nx] * v[i - nx];
  if (x > 0) acc += -cx[i - 1] * v[i - 1];
  acc += diag * v[i];
  if (x + 1 < nx) acc += -cx[i] * v[i + 1];
  if (cy && y + 1 < ny) acc += -cy[i] * v[i + nx];
  if (cz && z + 1 < nz) acc += -cz[i] * v[i + nxy];
  return acc;
}

static void m_apply_ext(size_t nx, size_t ny, size_t nz, const double* cx, const double* cy,
                        const double* cz, double eps, const double* v, double* out) {
  size_t i = 0;
  for (size_t z = 0; z < nz; ++z)
    for (size_t y = 0; y < ny; ++y)
      for (size_t x = 0; x < nx; ++x, ++i)
        out[i] = m_row(nx, ny, nz, x, y, z, i, cx, cy, cz, eps, v);
}

void orc_m_apply(const orc_grid* g, const double* cx, const double* cy, const double* cz,
                 double eps, const double* x, double* y) {
  size_t nx, ny, nz;
  grid_ext(g, &nx, &ny, &nz);
  m_apply_ext(nx, ny, nz, cx, g->dims >= 2 ? cy : NULL, g->dims >= 3 ? cz : NULL, eps, x, y);
}

/* penalty_functional (diffusion.cpp:89-101): x-edges, then y, then z, row-major */
typedef struct {
  const orc_grid* g;
  const double* f;
  int kind;
  double T, w;
  size_t nx, ny, nz;
} pen_ctx;
static double pen_elem(const void* c, size_t i) {
  const pen_ctx* p = (const pen_ctx*)c;
  const size_t nxy = p->nx * p->ny;
  const size_t x = i % p->nx, y = (i / p->nx) % p->ny, z = i / nxy;
  const double h = p->g->h;
  double v = 0.0;
  if (x + 1 < p->nx) v += p->w * orc_r_value(p->kind, p->T, fabs((p->f[i + 1] - p->f[i]) / h));
  if (p->g->dims >= 2 && y + 1 < p->ny)
    v += p->w * orc_r_value(p->kind, p->T, fabs((p->f[i + p->nx] - p->f[i]) / h));
  if (p->g->dims >= 3 && z + 1 < p->nz)
    v += p->w * orc_r_value(p->kind, p->T, fabs((p->f[i + nxy] - p->f[i]) / h));
  return v;
}

double orc_penalty_functional(const orc_grid* g, const double* f, int kind, double T) {
  if (g_device) {
    pen_ctx c;
    c.g = g;
    c.f = f;
    c.kind = kind;
    c.T = T;
    grid_ext(g, &c.nx, &c.ny, &c.nz);
    const double h = g->h;
    c.w = h;
    if (g->dims >= 2) c.w = h * h;
    if (g->dims >= 3) c.w = h * h * h;
    return canon_sum(pen_elem, &c, c.nx * c.ny * c.nz, c.nx);
  }
  size_t nx, ny, nz;
  grid_ext(g, &nx, &ny, &nz);
  const double h = g->h;
  double w = h;
  if (g->dims >= 2) w = h * h;
  if (g->dims >= 3) w = h * h * h;
  const size_t nxy = nx * ny;
  double acc = 0.0;
  for (size_t z = 0; z < nz; ++z)
    for (size_t y = 0; y < ny; ++y)
      for (size_t x = 0; x + 1 < nx; ++x) {
        const size_t i = z * nxy + y * nx + x;
        acc += w * orc_r_value(kind, T, fabs((f[i + 1] - f[i]) / h));
      }
  if (g->dims >= 2)
    for (size_t z = 0; z < nz; ++z)
      for (size_t y = 0; y + 1 < ny; ++y)
        for (size_t x = 0; x < nx; ++x) {
          const size_t i = z * nxy + y * nx + x;
          acc += w * orc_r_value(kind, T, fabs((f[i + nx] - f[i]) / h));
        }
  if (g->dims >= 3)
    for (size_t z = 0; z + 1 < nz; ++z)
      for (size_t y = 0; y < ny; ++y)
        for (size_t x = 0; x < nx; ++x) {
          const size_t i = z * nxy + y * nx + x;
          acc += w * orc_r_value(kind, T, fabs((f[i + nxy] - f[i]) / h));
        }
  return acc;
}

/* ======================================================================== */
/* SPD maps                                                                  */
/* ======================================================================== */

enum { MAP_IDENTITY = 0, MAP_CHOL = 1, MAP_VCYCLE = 2, MAP_CALLBACK = 3, MAP_ENVCHOL = 4, MAP_INNERCG = 5 };

typedef struct {
  size_t nx, ny, nz, n;
  double *cx, *cy, *cz; /* cy/cz NULL when the axis is inactive */
  double eps;
  double *x, *b, *r, *t; /* work vectors */
} vc_level;

struct orc_map {
  int kind;
  size_t n;
  /* cholesky */
  double* l;
  /* vcycle */
  int dims, levels, nu_pre, nu_post, coarse_sweeps;
  double omega;
  vc_level* lv;
  int ready;
  /* callback */
  orc_map_fn fn;
  void* ctx;
  /* envelope Cholesky / inner CG over a stencil M (grid extents, bandwidth, M snapshot) */
  size_t gnx, gny, gnz, band;
  double *mcx, *mcy, *mcz, meps;
  int k_inner;
};

orc_map* orc_identity_map_new(size_t n) {
  orc_map* m = (orc_map*)calloc(1, sizeof(orc_map));
  m->kind = MAP_IDENTITY;
  m->n = n;
  return m;
}

orc_map* orc_dense_chol_map_new(size_t n, const double* a) {
  orc_map* m = (orc_map*)calloc(1, sizeof(orc_map));
  m->kind = MAP_CHOL;
  m->n = n;
  m->l = (double*)calloc(n * n, sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    for (size_t j = 0; j <= i; ++j) {
      double sum = a[i * n + j];
      for (size_t k = 0; k < j; ++k) sum -= m->l[i * n + k] * m->l[j * n + k];
      if (i == j) {
        if (!(sum > 0.0)) {
          free(m->l);
          free(m);
          return NULL;
        }
        m->l[i * n + i] = sqrt(sum);
      } else {
        m->l[i * n + j] = sum / m->l[j * n + j];
      }
    }
  }
  return m;
}

orc_map* orc_callback_map_new(size_t n, orc_map_fn fn, void* ctx) {
  orc_map* m = (orc_map*)calloc(1, sizeof(orc_map));
  m->kind = MAP_CALLBACK;
  m->n = n;
  m->fn = fn;
  m->ctx = ctx;
  return m;
}

/* SpdSolver::factorize (spdsolve.cpp:22-75): envelope storage, row i = columns
 * [first_col(i), i], first_col = the smallest column of row i of the assembled M
 * (sparse.cpp row order: z-, y-, x- neighbour).  E(i, j) lives at l[i*(band+1) + band + j - i]. */
static size_t env_first(const orc_map* m, size_t i) {
  const size_t nxy = m->gnx * m->gny;
  const size_t z = i / nxy, y = (i / m->gnx) % m->gny, x = i % m->gnx;
  if (z > 0) return i - nxy;
  if (y > 0) return i - m->gnx;
  if (x > 0) return i - 1;
  return i;
}
#define ENV(m, i, j) ((m)->l[(i) * ((m)->band + 1) + (m)->band + (j) - (i)])

static orc_map* stencil_map_new(const orc_grid* g, const double* cx, const double* cy,
                                const double* cz, double eps) {
  if (grid_ok(g) || !(eps >= 0.0)) return NULL;
  orc_map* m = (orc_map*)calloc(1, sizeof(orc_map));
  grid_ext(g, &m->gnx, &m->gny, &m->gnz);
  m->n = m->gnx * m->gny * m->gnz;
  m->dims = g->dims;
  m->band = g->dims >= 3 ? m->gnx * m->gny : g->dims >= 2 ? m->gnx : 1;
  m->mcx = (double*)malloc(sizeof(double) * m->n);
  memcpy(m->mcx, cx, sizeof(double) * m->n);
  if (g->dims >= 2) {
    m->mcy = (double*)malloc(sizeof(double) * m->n);
    memcpy(m->mcy, cy, sizeof(double) * m->n);
  }
  if (g->dims >= 3) {
    m->mcz = (double*)malloc(sizeof(double) * m->n);
    memcpy(m->mcz, cz, sizeof(double) * m->n);
  }
  m->meps = eps;
  return m;
}

orc_map* orc_env_chol_map_new(const orc_grid* g, const double* cx, const double* cy,
                              const double* cz, double eps, long long* pivot_row) {
  if (pivot_row) *pivot_row = -1;
  orc_map* m = stencil_map_new(g, cx, cy, cz, eps);
  if (!m) return NULL;
  m->kind = MAP_ENVCHOL;
  const size_t n = m->n, W = m->band + 1, nxy = m->gnx * m->gny;
  m->l = (double*)calloc(n * W, sizeof(double));
  /* lower triangle of M + eps I (spdsolve.cpp:40-48; values as assemble_m / with_shift) */
  size_t i = 0;
  for (size_t z = 0; z < m->gnz; ++z)
    for (size_t y = 0; y < m->gny; ++y)
      for (size_t x = 0; x < m->gnx; ++x, ++i) {
        if (m->mcz && z > 0) ENV(m, i, i - nxy) = -m->mcz[i - nxy];
        if (m->mcy && y > 0) ENV(m, i, i - m->gnx) = -m->mcy[i - m->gnx];
        if (x > 0) ENV(m, i, i - 1) = -m->mcx[i - 1];
        ENV(m, i, i) = diag_at(m->gnx, m->gny, m->gnz, x, y, z, i, m->mcx, m->mcy, m->mcz) + eps;
      }
  /* in-place skyline Cholesky (spdsolve.cpp:51-73): sum = E(i,j) - dot(...), sequential dot */
  for (i = 0; i < n; ++i) {
    const size_t fi = env_first(m, i);
    for (size_t j = fi; j <= i; ++j) {
      const size_t fj = env_first(m, j);
      const size_t lo = fi > fj ? fi : fj;
      double sum = ENV(m, i, j);
      if (j > lo) {
        double acc = 0.0;
        for (size_t k = lo; k < j; ++k) acc += ENV(m, i, k) * ENV(m, j, k);
        sum -= acc;
      }
      if (j < i) {
        ENV(m, i, j) = sum / ENV(m, j, j);
      } else {
        if (!(sum > 0.0)) {
          if (pivot_row) *pivot_row = (long long)i;
          orc_map_free(m);
          return NULL;
        }
        ENV(m, i, i) = sqrt(sum);
      }
    }
  }
  return m;
}

/* SpdSolver::inner_cg (spdsolve.cpp:77-85): the solver keeps its own copy of M */
orc_map* orc_inner_cg_map_new(const orc_grid* g, const double* cx, const double* cy,
                              const double* cz, double eps, int k_inner) {
  if (k_inner < 1) return NULL;
  orc_map* m = stencil_map_new(g, cx, cy, cz, eps);
  if (!m) return NULL;
  m->kind = MAP_INNERCG;
  m->k_inner = k_inner;
  return m;
}

orc_map* orc_vcycle_new(const orc_grid* g, int levels, int nu_pre, int nu_post, double omega,
                        int coarse_sweeps) {
  if (grid_ok(g) || levels < 1 || nu_pre < 1 || nu_post < 0 || coarse_sweeps < 1) return NULL;
  size_t nx, ny, nz;
  grid_ext(g, &nx, &ny, &nz);
  /* every active axis must halve evenly down to the coarsest level, keeping >= 2 cells */
  const size_t f = (size_t)1 << (levels - 1);
  if (nx % f || nx / f < 2) return NULL;
  if (g->dims >= 2 && (ny % f || ny / f < 2)) return NULL;
  if (g->dims >= 3 && (nz % f || nz / f < 2)) return NULL;
  orc_map* m = (orc_map*)calloc(1, sizeof(orc_map));
  m->kind = MAP_VCYCLE;
  m->n = nx * ny * nz;
  m->dims = g->dims;
  m->levels = levels;
  m->nu_pre = nu_pre;
  m->nu_post = nu_post;
  m->omega = omega;
  m->coarse_sweeps = coarse_sweeps;
  m->lv = (vc_level*)calloc((size_t)levels, sizeof(vc_level));
  for (int l = 0; l < levels; ++l) {
    vc_level* L = &m->lv[l];
    L->nx = nx >> l;
    L->ny = g->dims >= 2 ? ny >> l : 1;
    L->nz = g->dims >= 3 ? nz >> l : 1;
    L->n = L->nx * L->ny * L->nz;
    L->cx = (double*)calloc(L->n, sizeof(double));
    L->cy = g->dims >= 2 ? (double*)calloc(L->n, sizeof(double)) : NULL;
    L->cz = g->dims >= 3 ? (double*)calloc(L->n, sizeof(double)) : NULL;
    L->x = (double*)calloc(L->n, sizeof(double));
    L->b = (double*)calloc(L->n, sizeof(double));
    L->r = (double*)calloc(L->n, sizeof(double));
    L->t = (double*)calloc(L->n, sizeof(double));
  }
  return m;
}

/* Galerkin coarse edge: sum of the 2^(d-1) fine edges crossing the coarse
 * face, in ascending fine linear index order (z outer, y inner). */
static void coarsen(const vc_level* F, vc_level* C, int dims) {
  const size_t fnx = F->nx, fnxy = F->nx * F->ny;
  const size_t cnx = C->nx, cny = C->ny, cnz = C->nz;
  const size_t zc = dims >= 3 ? 2 : 1, yc = dims >= 2 ? 2 : 1;
  size_t I = 0;
  for (size_t Z = 0; Z < cnz; ++Z)
    for (size_t Y = 0; Y < cny; ++Y)
      for (size_t X = 0; X < cnx; ++X, ++I) {
        double sx = 0.0, sy = 0.0, sz = 0.0;
        for (size_t dz = 0; dz < zc; ++dz)
          for (size_t dy = 0; dy < yc; ++dy) {
            /* x-face between aggregates X and X+1: fine edge (2X+1 -> 2X+2) */
            if (X + 1 < cnx) sx += F->cx[(zc * Z + dz) * fnxy + (yc * Y + dy) * fnx + 2 * X + 1];
          }
        if (dims >= 2)
          for (size_t dz = 0; dz < zc; ++dz)
            for (size_t dx = 0; dx < 2; ++dx)
              if (Y + 1 < cny) sy += F->cy[(zc * Z + dz) * fnxy + (2 * Y + 1) * fnx + 2 * X + dx];
        if (dims >= 3)
          for (size_t dy = 0; dy < 2; ++dy)
            for (size_t dx = 0; dx < 2; ++dx)
              if (Z + 1 < cnz) sz += F->cz[(2 * Z + 1) * fnxy + (2 * Y + dy) * fnx + 2 * X + dx];
        C->cx[I] = sx;
        if (C->cy) C->cy[I] = sy;
        if (C->cz) C->cz[I] = sz;
      }
  double mult = 2.0;
  if (dims >= 2) mult *= 2.0;
  if (dims >= 3) mult *= 2.0;
  C->eps = F->eps * mult; /* P^T (eps I) P = 2^d eps I */
}

int orc_vcycle_set(orc_map* m, const double* cx, const double* cy, const double* cz,
                   double eps) {
  if (!m || m->kind != MAP_VCYCLE) return ORC_EINVAL;
  vc_level* L0 = &m->lv[0];
  memcpy(L0->cx, cx, sizeof(double) * L0->n);
  if (L0->cy) memcpy(L0->cy, cy, sizeof(double) * L0->n);
  if (L0->cz) memcpy(L0->cz, cz, sizeof(double) * L0->n);
  L0->eps = eps;
  for (int l = 1; l < m->levels; ++l) coarsen(&m->lv[l - 1], &m->lv[l], m->dims);
  m->ready = 1;
  return ORC_OK;
}

/* x <- x + (omega * (b - M x)) / D, Jacobi (all rows from the old x) */
static void jacobi(const vc_level* L, double omega, double* x, const double* b, double* tmp) {
  const size_t nx = L->nx, ny = L->ny, nz = L->nz;
  m_apply_ext(nx, ny, nz, L->cx, L->cy, L->cz, L->eps, x, tmp);
  size_t i = 0;
  for (size_t z = 0; z < nz; ++z)
    for (size_t y = 0; y < ny; ++y)
      for (size_t xx = 0; xx < nx; ++xx, ++i) {
        const double d = diag_at(nx, ny, nz, xx, y, z, i, L->cx, L->cy, L->cz) + L->eps;
        x[i] = x[i] + (omega * (b[i] - tmp[i])) / d;
      }
}

static void vcycle_level(const orc_map* m, int l, const double* b, double* x) {
  const vc_level* L = &m->lv[l];
  const int coarsest = l == m->levels - 1;
  const int sweeps = coarsest ? m->coarse_sweeps : m->nu_pre;
  for (size_t i = 0; i < L->n; ++i) x[i] = 0.0;
  for (int s = 0; s < sweeps; ++s) jacobi(L, m->omega, x, b, L->t);
  if (coarsest) return;
  /* residual r = b - M x, restricted by summing the 2^d children */
  m_apply_ext(L->nx, L->ny, L->nz, L->cx, L->cy, L->cz, L->eps, x, L->t);
  for (size_t i = 0; i < L->n; ++i) L->r[i] = b[i] - L->t[i];
  const vc_level* C = &m->lv[l + 1];
  const size_t zc = m->dims >= 3 ? 2 : 1, yc = m->dims >= 2 ? 2 : 1;
  const size_t fnx = L->nx, fnxy = L->nx * L->ny;
  size_t I = 0;
  for (size_t Z = 0; Z < C->nz; ++Z)
    for (size_t Y = 0; Y < C->ny; ++Y)
      for (size_t X = 0; X < C->nx; ++X, ++I) {
        double s = 0.0;
        for (size_t dz = 0; dz < zc; ++dz)
          for (size_t dy = 0; dy < yc; ++dy)
            for (size_t dx = 0; dx < 2; ++dx)
              s += L->r[(zc * Z + dz) * fnxy + (yc * Y + dy) * fnx + 2 * X + dx];
        C->b[I] = s;
      }
  vcycle_level(m, l + 1, C->b, C->x);
  /* prolongation by injection: x += P x_c */
  size_t i = 0;
  for (size_t z = 0; z < L->nz; ++z)
    for (size_t y = 0; y < L->ny; ++y)
      for (size_t xx = 0; xx < L->nx; ++xx, ++i) {
        const size_t Z = m->dims >= 3 ? z / 2 : 0, Y = m->dims >= 2 ? y / 2 : 0;
        x[i] += C->x[(Z * C->ny + Y) * C->nx + xx / 2];
      }
  for (int s = 0; s < m->nu_post; ++s) jacobi(L, m->omega, x, b, L->t);
}

int orc_vcycle_level(const orc_map* m, int l, size_t* dims3, double* cx, double* cy, double* cz,
                     double* eps) {
  if (!m || m->kind != MAP_VCYCLE || l < 0 || l >= m->levels) return ORC_EINVAL;
  const vc_level* L = &m->lv[l];
  if (dims3) {
    dims3[0] = L->nx;
    dims3[1] = L->ny;
    dims3[2] = L->nz;
  }
  if (cx) memcpy(cx, L->cx, sizeof(double) * L->n);
  if (cy && L->cy) memcpy(cy, L->cy, sizeof(double) * L->n);
  if (cz && L->cz) memcpy(cz, L->cz, sizeof(double) * L->n);
  if (eps) *eps = L->eps;
  return ORC_OK;
}

/* solve_cg (spdsolve.cpp:119-137): exactly k_inner iterations from v = 0; dots in the
 * active order (reference: sequential; device: canonical segments over rows of gnx) */
static double dotL(const double* x, const double* y, size_t n, size_t L);
static void inner_cg_solve(const orc_map* m, const double* p, double* v) {
  const size_t n = m->n, L = m->gnx;
  double* r = (double*)malloc(sizeof(double) * n);
  double* d = (double*)malloc(sizeof(double) * n);
  double* q = (double*)malloc(sizeof(double) * n);
  memset(v, 0, sizeof(double) * n);
  memcpy(r, p, sizeof(double) * n);
  memcpy(d, r, sizeof(double) * n);
  double rho = dotL(r, r, n, L);
  for (int it = 0; it < m->k_inner; ++it) {
    if (rho == 0.0) break;
    m_apply_ext(m->gnx, m->gny, m->gnz, m->mcx, m->mcy, m->mcz, m->meps, d, q);
    const double curv = dotL(d, q, n, L);
    if (curv == 0.0) break;
    const double gamma = rho / curv;
    for (size_t i = 0; i < n; ++i) v[i] += gamma * d[i];
    const double ng = -gamma;
    for (size_t i = 0; i < n; ++i) r[i] += ng * q[i];
    const double rho_next = dotL(r, r, n, L);
    const double beta = rho_next / rho;
    for (size_t i = 0; i < n; ++i) d[i] = r[i] + beta * d[i];
    rho = rho_next;
  }
  free(r);
  free(d);
  free(q);
}

void orc_map_solve(const orc_map* m, const double* p, double* v) {
  switch (m->kind) {
    case MAP_IDENTITY: memcpy(v, p, sizeof(double) * m->n); break;
    case MAP_CHOL: {
      const size_t n = m->n;
      for (size_t i = 0; i < n; ++i) {
        double s = p[i];
        for (size_t k = 0; k < i; ++k) s -= m->l[i * n + k] * v[k];
        v[i] = s / m->l[i * n + i];
      }
      for (size_t ii = n; ii-- > 0;) {
        double s = v[ii];
        for (size_t k = ii + 1; k < n; ++k) s -= m->l[k * n + ii] * v[k];
        v[ii] = s / m->l[ii * n + ii];
      }
      break;
    }
    case MAP_VCYCLE: vcycle_level(m, 0, p, v); break;
    case MAP_ENVCHOL: { /* solve_cholesky (spdsolve.cpp:101-117) */
      const size_t n = m->n;
      for (size_t i = 0; i < n; ++i) {
        const size_t fi = env_first(m, i);
        double sum = p[i];
        if (i > fi) {
          double acc = 0.0;
          for (size_t k = fi; k < i; ++k) acc += ENV(m, i, k) * v[k];
          sum -= acc;
        }
        v[i] = sum / ENV(m, i, i);
      }
      for (size_t ii = n; ii-- > 0;) {
        const size_t fi = env_first(m, ii);
        v[ii] /= ENV(m, ii, ii);
        const double a = -v[ii];
        for (size_t k = fi; k < ii; ++k) v[k] += a * ENV(m, ii, k);
      }
      break;
    }
    case MAP_INNERCG: inner_cg_solve(m, p, v); break;
    case MAP_CALLBACK: m->fn(m->ctx, p, v); break;
  }
}

void orc_map_free(orc_map* m) {
  if (!m) return;
  free(m->l);
  free(m->mcx);
  free(m->mcy);
  free(m->mcz);
  if (m->lv) {
    for (int l = 0; l < m->levels; ++l) {
      vc_level* L = &m->lv[l];
      free(L->cx); free(L->cy); free(L->cz);
      free(L->x); free(L->b); free(L->r); free(L->t);
    }
    free(m->lv);
  }
  free(m);
}

/* ======================================================================== */
/* Krylov (krylov.cpp:24-440)                                                */
/* ======================================================================== */

static double dot_ref(const double* x, const double* y, size_t n) {
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += x[i] * y[i];
  return acc;
}
/* L: row length of the vector's space (canonical segments never straddle rows) */
static double dotL(const double* x, const double* y, size_t n, size_t L) {
  return g_device ? orc_canon_dot(x, y, n, L) : dot_ref(x, y, n);
}
static double nrm2L(const double* x, size_t n, size_t L) { return sqrt(dotL(x, x, n, L)); }
static void axpy(double a, const double* x, double* y, size_t n) {
  for (size_t i = 0; i < n; ++i) y[i] += a * x[i];
}
static void xpby(const double* x, double b, double* y, size_t n) {
  for (size_t i = 0; i < n; ++i) y[i] = x[i] + b * y[i];
}
static void scal(double a, double* x, size_t n) {
  for (size_t i = 0; i < n; ++i) x[i] *= a;
}

/* LsqrRecurrence (krylov.cpp:24-108) */
typedef struct {
  double tau, damp, alpha_cur, phibar, rhobar, bnorm, rnorm, arnorm, anorm2, ddnorm, res2, cs2,
      sn2, z, xxnorm, xnorm;
} rec_t;

static void rec_init(rec_t* r, double alpha1, double beta1, double tau) {
  memset(r, 0, sizeof(*r));
  r->tau = tau;
  r->damp = sqrt(tau);
  r->alpha_cur = alpha1;
  r->phibar = beta1;
  r->rhobar = alpha1;
  r->bnorm = beta1;
  r->rnorm = beta1;
  r->cs2 = -1.0;
}

static void rec_advance(rec_t* r, double beta_next, double alpha_next, double wnorm2,
                        double* sol_coeff, double* dir_coeff) {
  r->anorm2 += r->alpha_cur * r->alpha_cur + beta_next * beta_next + r->tau;
  double rhobar1 = r->rhobar, psi = 0.0;
  if (r->damp > 0.0) {
    rhobar1 = hyp(r->rhobar, r->damp);
    const double cs1 = r->rhobar / rhobar1;
    psi = (r->damp / rhobar1) * r->phibar;
    r->phibar = cs1 * r->phibar;
  }
  const double rho = hyp(rhobar1, beta_next);
  const double cs = rhobar1 / rho;
  const double sn = beta_next / rho;
  const double theta = sn * alpha_next;
  r->rhobar = -cs * alpha_next;
  const double phi = cs * r->phibar;
  r->phibar = sn * r->phibar;
  r->ddnorm += wnorm2 / (rho * rho);
  const double delta = r->sn2 * rho;
  const double gambar = -r->cs2 * rho;
  const double rhs = phi - delta * r->z;
  const double zbar = rhs / gambar;
  r->xnorm = sqrt(r->xxnorm + zbar * zbar);
  const double gamma = hyp(gambar, theta);
  r->cs2 = gambar / gamma;
  r->sn2 = theta / gamma;
  r->z = rhs / gamma;
  r->xxnorm += r->z * r->z;
  r->res2 += psi * psi;
  r->rnorm = sqrt(r->phibar * r->phibar + r->res2);
  r->arnorm = alpha_next * fabs(sn * phi);
  r->alpha_cur = alpha_next;
  *sol_coeff = phi / rho;
  *dir_coeff = theta / rho;
}

static double rec_anorm(const rec_t* r) { return sqrt(r->anorm2); }
static double rec_acond(const rec_t* r) { return rec_anorm(r) * sqrt(r->ddnorm); }

/* evaluate_stopping (krylov.cpp:240-254); returns -1 for "continue" */
static int evaluate_stopping(double rbar, double atrbar, double anorm, double acond,
                             double xnorm, double bnorm, double data_res, int iteration,
                             const orc_stop* s) {
  if (s->use_s4 && data_res <= s->eta * s->delta) return ORC_STOP_S4;
  if (s->use_s1 && rbar <= s->btol * bnorm + s->atol * anorm * xnorm) return ORC_STOP_S1;
  if (s->use_s2) {
    const double den = anorm * rbar;
    if (atrbar <= s->atol * den || den == 0.0) return ORC_STOP_S2;
  }
  if (s->use_s3 && s->conlim > 0.0 && acond >= s->conlim) return ORC_STOP_S3;
  if (iteration >= s->max_iters) return ORC_STOP_MAX_ITERS;
  return -1;
}

static int stop_validate(const orc_stop* s) {
  if (s->max_iters < 1) return ORC_EINVAL;
  if (s->use_s4 && !(s->eta > 1.0)) return ORC_EINVAL;
  if (s->use_s4 && !(s->delta >= 0.0)) return ORC_EINVAL;
  if (!(s->atol >= 0.0) || !(s->btol >= 0.0)) return ORC_EINVAL;
  return ORC_OK;
}

/* finish_iteration (krylov.cpp:131-180); returns stop reason or -1 */
static int finish_iteration(int iter, const rec_t* rec, double beta, double alpha_next,
                            int breakdown, const orc_stop* stop, const orc_linop* a,
                            const double* f, const double* g, double* scratch_rows,
                            orc_iter_rec* trace, double* snapshots, size_t n) {
  orc_iter_rec row;
  memset(&row, 0, sizeof(row));
  row.iteration = iter;
  row.res_damped = rec->rnorm;
  if (rec->tau == 0.0) {
    row.res_data = rec->rnorm;
    row.res_data_exact = 1;
  } else if (stop->use_s4) {
    orc_linop_apply(a, f, scratch_rows);
    if (g_device) {
      for (size_t i = 0; i < a->rows; ++i) scratch_rows[i] = g[i] - scratch_rows[i];
      row.res_data = sqrt(orc_canon_dot(scratch_rows, scratch_rows, a->rows, a->data_len));
    } else {
      double acc = 0.0;
      for (size_t i = 0; i < a->rows; ++i) {
        const double d = g[i] - scratch_rows[i];
        acc += d * d;
      }
      row.res_data = sqrt(acc);
    }
    row.res_data_exact = 1;
  } else {
    const double est = rec->rnorm * rec->rnorm - rec->tau * rec->xnorm * rec->xnorm;
    row.res_data = sqrt(est > 0.0 ? est : 0.0);
    row.res_data_exact = 0;
  }
  const double den = rec_anorm(rec) * rec->rnorm;
  row.s2_value = den > 0.0 ? rec->arnorm / den : 0.0;
  row.anorm_est = rec_anorm(rec);
  row.cond_est = rec_acond(rec);
  row.xnorm_est = rec->xnorm;
  row.alpha = alpha_next;
  row.beta = beta;
  if (trace) trace[iter - 1] = row;
  if (snapshots) memcpy(snapshots + (size_t)(iter - 1) * n, f, sizeof(double) * n);
  const int fired = evaluate_stopping(rec->rnorm, rec->arnorm, rec_anorm(rec), rec_acond(rec),
                                      rec->xnorm, rec->bnorm, row.res_data, iter, stop);
  if (fired >= 0) return fired;
  if (breakdown) return ORC_STOP_BREAKDOWN;
  return -1;
}

int orc_mlsqr(const orc_linop* a, const orc_map* msolver, const double* g, double tau,
              const orc_stop* stop, double* f_out, orc_iter_rec* trace, double* alphas,
              double* betas, double* snapshots, orc_solve_info* info) {
  orc_solve_info dummy;
  if (!info) info = &dummy;
  memset(info, 0, sizeof(*info));
  if (stop_validate(stop)) return ORC_EINVAL;
  if (!(tau >= 0.0)) return ORC_EINVAL;
  if (msolver->n != a->cols) return ORC_EDIM;
  const size_t n = a->cols, m = a->rows;
  double* f = (double*)calloc(n, sizeof(double));
  int na = 0, nb = 0, status = ORC_OK;
  info->stop_reason = ORC_STOP_MAX_ITERS;

  const double beta1 = nrm2L(g, m, a->data_len);
  if (betas) betas[nb] = beta1;
  nb++;
  double *u = NULL, *p = NULL, *v = NULL, *w = NULL, *q = NULL, *tr = NULL, *tc = NULL;
  if (beta1 == 0.0) {
    info->stop_reason = ORC_STOP_BREAKDOWN;
    goto done;
  }
  u = (double*)malloc(sizeof(double) * m);
  memcpy(u, g, sizeof(double) * m);
  scal(1.0 / beta1, u, m);
  p = (double*)malloc(sizeof(double) * n);
  orc_linop_adjoint(a, u, p);
  v = (double*)calloc(n, sizeof(double));
  if (nrm2L(p, n, a->sol_len) == 0.0) {
    info->stop_reason = ORC_STOP_BREAKDOWN;
    goto done;
  }
  orc_map_solve(msolver, p, v);
  {
    const double s0 = dotL(v, p, n, a->sol_len);
    if (!(s0 > 0.0)) {
      status = ORC_EBREAKDOWN;
      info->breakdown_iteration = 0;
      goto done;
    }
    const double alpha1 = sqrt(s0);
    scal(1.0 / alpha1, v, n);
    scal(1.0 / alpha1, p, n);
    if (alphas) alphas[na] = alpha1;
    na++;
    w = (double*)malloc(sizeof(double) * n);
    q = (double*)malloc(sizeof(double) * n);
    memcpy(w, v, sizeof(double) * n);
    memcpy(q, p, sizeof(double) * n);
    tr = (double*)malloc(sizeof(double) * m);
    tc = (double*)malloc(sizeof(double) * n);
    rec_t rec;
    rec_init(&rec, alpha1, beta1, tau);
    double alpha = alpha1;
    for (int iter = 1; iter <= stop->max_iters; ++iter) {
      orc_linop_apply(a, v, tr);
      xpby(tr, -alpha, u, m);
      const double beta = nrm2L(u, m, a->data_len);
      double alpha_next = 0.0;
      int breakdown = 1;
      if (beta > 0.0) {
        scal(1.0 / beta, u, m);
        orc_linop_adjoint(a, u, tc);
        xpby(tc, -beta, p, n);
        if (nrm2L(p, n, a->sol_len) > 0.0) {
          orc_map_solve(msolver, p, v);
          const double s = dotL(v, p, n, a->sol_len);
          if (!(s > 0.0)) {
            status = ORC_EBREAKDOWN;
            info->breakdown_iteration = iter;
            goto done;
          }
          alpha_next = sqrt(s);
          scal(1.0 / alpha_next, v, n);
          scal(1.0 / alpha_next, p, n);
          breakdown = 0;
        }
      }
      const double wnorm2 = dotL(w, q, n, a->sol_len);
      double sc, dc;
      rec_advance(&rec, beta, alpha_next, wnorm2, &sc, &dc);
      axpy(sc, w, f, n);
      if (!breakdown) {
        xpby(v, -dc, w, n);
        xpby(p, -dc, q, n);
        if (alphas) alphas[na] = alpha_next;
        na++;
      }
      if (betas) betas[nb] = beta;
      nb++;
      alpha = alpha_next;
      info->iterations = iter;
      const int fired = finish_iteration(iter, &rec, beta, alpha_next, breakdown, stop, a, f, g,
                                         tr, trace, snapshots, n);
      if (fired >= 0) {
        info->stop_reason = fired;
        break;
      }
    }
    if (na > info->iterations) na = info->iterations; /* trim_bidiag (krylov.cpp:182-186) */
  }
done:
  info->n_alphas = na;
  info->n_betas = nb;
  if (f_out) memcpy(f_out, f, sizeof(double) * n);
  free(f); free(u); free(p); free(v); free(w); free(q); free(tr); free(tc);
  return status;
}

int orc_lsqr(const orc_linop* a, const double* g, double tau, const orc_stop* stop,
             double* f_out, orc_iter_rec* trace, double* alphas, double* betas,
             double* snapshots, orc_solve_info* info) {
  orc_solve_info dummy;
  if (!info) info = &dummy;
  memset(info, 0, sizeof(*info));
  if (stop_validate(stop)) return ORC_EINVAL;
  if (!(tau >= 0.0)) return ORC_EINVAL;
  const size_t n = a->cols, m = a->rows;
  double* f = (double*)calloc(n, sizeof(double));
  int na = 0, nb = 0;
  info->stop_reason = ORC_STOP_MAX_ITERS;
  double *u = NULL, *v = NULL, *w = NULL, *tr = NULL, *tc = NULL;
  const double beta1 = nrm2L(g, m, a->data_len);
  if (betas) betas[nb] = beta1;
  nb++;
  if (beta1 == 0.0) {
    info->stop_reason = ORC_STOP_BREAKDOWN;
    goto done;
  }
  u = (double*)malloc(sizeof(double) * m);
  memcpy(u, g, sizeof(double) * m);
  scal(1.0 / beta1, u, m);
  v = (double*)malloc(sizeof(double) * n);
  orc_linop_adjoint(a, u, v);
  {
    const double alpha1 = nrm2L(v, n, a->sol_len);
    if (alpha1 == 0.0) {
      info->stop_reason = ORC_STOP_BREAKDOWN;
      goto done;
    }
    scal(1.0 / alpha1, v, n);
    if (alphas) alphas[na] = alpha1;
    na++;
    w = (double*)malloc(sizeof(double) * n);
    memcpy(w, v, sizeof(double) * n);
    tr = (double*)malloc(sizeof(double) * m);
    tc = (double*)malloc(sizeof(double) * n);
    rec_t rec;
    rec_init(&rec, alpha1, beta1, tau);
    double alpha = alpha1;
    for (int iter = 1; iter <= stop->max_iters; ++iter) {
      orc_linop_apply(a, v, tr);
      xpby(tr, -alpha, u, m);
      const double beta = nrm2L(u, m, a->data_len);
      double alpha_next = 0.0;
      if (beta > 0.0) {
        scal(1.0 / beta, u, m);
        orc_linop_adjoint(a, u, tc);
        xpby(tc, -beta, v, n);
        alpha_next = nrm2L(v, n, a->sol_len);
        if (alpha_next > 0.0) scal(1.0 / alpha_next, v, n);
      }
      const int breakdown = beta == 0.0 || alpha_next == 0.0;
      const double wnorm2 = dotL(w, w, n, a->sol_len);
      double sc, dc;
      rec_advance(&rec, beta, alpha_next, wnorm2, &sc, &dc);
      axpy(sc, w, f, n);
      xpby(v, -dc, w, n);
      alpha = alpha_next;
      if (betas) betas[nb] = beta;
      nb++;
      if (!breakdown) {
        if (alphas) alphas[na] = alpha_next;
        na++;
      }
      info->iterations = iter;
      const int fired = finish_iteration(iter, &rec, beta, alpha_next, breakdown, stop, a, f, g,
                                         tr, trace, snapshots, n);
      if (fired >= 0) {
        info->stop_reason = fired;
        break;
      }
    }
    (void)alpha;
    if (na > info->iterations) na = info->iterations;
  }
done:
  info->n_alphas = na;
  info->n_betas = nb;
  if (f_out) memcpy(f_out, f, sizeof(double) * n);
  free(f); free(u); free(v); free(w); free(tr); free(tc);
  return ORC_OK;
}

/* ======================================================================== */
/* outer loop (outer.cpp:31-100)                                             */
/* ======================================================================== */

int orc_outer_stop_check(const double* history, int k, double threshold) {
  if (k < 2) return 0;
  const double prev = history[k - 2];
  if (prev == 0.0) return 1;
  return (history[k - 1] - prev) / prev > -threshold;
}

int orc_nonlinear(const orc_linop* a, const double* g, const orc_grid* grid,
                  const orc_outer_cfg* cfg, double* f_out, orc_outer_step* steps,
                  int* n_steps, int* stop_reason, int* triggered_at, double* alphas,
                  double* betas, double* iterates) {
  int st = grid_ok(grid);
  if (st) return st;
  size_t nx, ny, nz;
  grid_ext(grid, &nx, &ny, &nz);
  const size_t n = nx * ny * nz;
  if (n != a->cols) return ORC_EDIM;
  if (cfg->inner_cap < 1 || cfg->max_outer < 1 || !(cfg->tau >= 0.0)) return ORC_EINVAL;
  if (cfg->rel_decrease_threshold >= 1.0) return ORC_EINVAL;
  orc_stop inner = cfg->inner_stop;
  if (cfg->inner_cap < inner.max_iters) inner.max_iters = cfg->inner_cap;
  if (stop_validate(&inner)) return ORC_EINVAL;

  /* mg_levels == 0: exact dense Cholesky of the assembled M per outer step, i.e. the
   * reference's SpdSolverMode::direct_cholesky (outer.cpp:64-67); small grids only. */
  const int stencil_mode = cfg->spd_mode == 1 || cfg->spd_mode == 2;
  if (cfg->spd_mode < 0 || cfg->spd_mode > 2 || (cfg->spd_mode == 2 && cfg->k_inner < 1)) return ORC_EINVAL;
  const int dense_mode = !stencil_mode && cfg->mg_levels == 0;
  orc_map* mg = NULL;
  double* mdense = NULL;
  if (dense_mode) {
    mdense = (double*)malloc(sizeof(double) * n * n);
  } else if (!stencil_mode) {
    mg = orc_vcycle_new(grid, cfg->mg_levels, cfg->nu_pre, cfg->nu_post, cfg->omega,
                        cfg->coarse_sweeps);
    if (!mg) return ORC_EINVAL;
  }
  double* prev = (double*)calloc(n, sizeof(double));
  double* cur = (double*)calloc(n, sizeof(double));
  double* cx = (double*)calloc(n, sizeof(double));
  double* cy = (double*)calloc(n, sizeof(double));
  double* cz = (double*)calloc(n, sizeof(double));
  double* history = (double*)calloc((size_t)cfg->max_outer, sizeof(double));
  orc_iter_rec* trace = (orc_iter_rec*)calloc((size_t)inner.max_iters, sizeof(orc_iter_rec));
  *stop_reason = 1; /* max_outer */
  *triggered_at = 0;
  *n_steps = 0;
  const int ab = cfg->inner_cap + 1, bb = cfg->inner_cap + 2;
  for (int k = 1; k <= cfg->max_outer; ++k) {
    orc_edge_coeffs(grid, prev, cfg->pen_kind, cfg->T, cx, cy, cz);
    const double eps = cfg->epsilon >= 0.0 ? cfg->epsilon
                                           : 1e-8 * orc_max_diag(grid, cx, cy, cz);
    if (stencil_mode) { /* outer.cpp:64-70: this step's SpdSolver */
      orc_map_free(mg);
      mg = cfg->spd_mode == 1 ? orc_env_chol_map_new(grid, cx, cy, cz, eps, NULL)
                              : orc_inner_cg_map_new(grid, cx, cy, cz, eps, cfg->k_inner);
      if (!mg) { st = ORC_EINVAL; break; }
    } else if (dense_mode) {
      double* e = (double*)calloc(n, sizeof(double));
      double* col = (double*)malloc(sizeof(double) * n);
      for (size_t j = 0; j < n; ++j) {
        e[j] = 1.0;
        orc_m_apply(grid, cx, cy, cz, eps, e, col);
        for (size_t i = 0; i < n; ++i) mdense[i * n + j] = col[i];
        e[j] = 0.0;
      }
      free(e);
      free(col);
      orc_map_free(mg);
      mg = orc_dense_chol_map_new(n, mdense);
      if (!mg) { st = ORC_EINVAL; break; }
    } else {
      orc_vcycle_set(mg, cx, cy, cz, eps);
    }
    orc_solve_info info;
    st = orc_mlsqr(a, mg, g, cfg->tau, &inner, cur, trace,
                   alphas ? alphas + (size_t)(k - 1) * ab : NULL,
                   betas ? betas + (size_t)(k - 1) * bb : NULL, NULL, &info);
    if (st) break;
    const double pv = orc_penalty_functional(grid, cur, cfg->pen_kind, cfg->T);
    history[k - 1] = pv;
    orc_outer_step* s = &steps[k - 1];
    s->k = k;
    s->penalty_value = pv;
    s->inner_iterations = info.iterations;
    s->inner_stop = info.stop_reason;
    s->final_residual = info.iterations == 0 ? nrm2L(g, a->rows, a->data_len) : trace[info.iterations - 1].res_data;
    s->eps_used = eps;
    *n_steps = k;
    if (iterates) memcpy(iterates + (size_t)(k - 1) * n, cur, sizeof(double) * n);
    if (cfg->rel_decrease_threshold > 0.0 &&
        orc_outer_stop_check(history, k, cfg->rel_decrease_threshold)) {
      *stop_reason = 0; /* stagnation: return f^{k-1} */
      *triggered_at = k;
      break;
    }
    double* t = prev;
    prev = cur;
    cur = t;
  }
  if (f_out && st == ORC_OK) memcpy(f_out, prev, sizeof(double) * n);
  orc_map_free(mg);
  free(mdense);
  free(prev); free(cur); free(cx); free(cy); free(cz); free(history); free(trace);
  return st;
}

/* ======================================================================== */
/* seeded synthetic problems                                                 */
/* ======================================================================== */

void orc_phantom_rects2d(size_t nx, size_t ny, int count, uint64_t seed, double* out) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  double* sh = (double*)malloc(sizeof(double) * 5 * (size_t)(count > 0 ? count : 1));
  for (int k = 0; k < count; ++k) {
    const double xa = orc_uniform(&s), xb = orc_uniform(&s);
    const double ya = orc_uniform(&s), yb = orc_uniform(&s);
    sh[5 * k + 0] = xa < xb ? xa : xb;
    sh[5 * k + 1] = xa < xb ? xb : xa;
    sh[5 * k + 2] = ya < yb ? ya : yb;
    sh[5 * k + 3] = ya < yb ? yb : ya;
    sh[5 * k + 4] = orc_uniform(&s);
  }
  const double hx = 1.0 / (double)nx, hy = 1.0 / (double)ny;
  for (size_t iy = 0; iy < ny; ++iy) {
    const double y = ((double)iy + 0.5) * hy;
    for (size_t ix = 0; ix < nx; ++ix) {
      const double x = ((double)ix + 0.5) * hx;
      double v = 0.0;
      for (int k = 0; k < count; ++k) {
        const double* r = sh + 5 * k;
        if (x >= r[0] && x <= r[1] && y >= r[2] && y <= r[3]) v = r[4];
      }
      out[iy * nx + ix] = v;
    }
  }
  free(sh);
}

void orc_phantom_shapes2d(size_t nx, size_t ny, int count, uint64_t seed, double* out) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  double* sh = (double*)malloc(sizeof(double) * 6 * (size_t)(count > 0 ? count : 1));
  for (int k = 0; k < count; ++k)
    for (int j = 0; j < 6; ++j) sh[6 * k + j] = orc_uniform(&s);
  const double hx = 1.0 / (double)nx, hy = 1.0 / (double)ny;
  for (size_t iy = 0; iy < ny; ++iy) {
    const double y = ((double)iy + 0.5) * hy;
    for (size_t ix = 0; ix < nx; ++ix) {
      const double x = ((double)ix + 0.5) * hx;
      double v = 0.0;
      for (int k = 0; k < count; ++k) {
        const double* r = sh + 6 * k;
        const double cx = r[1], cy = r[2];
        const double a = 0.02 + 0.08 * r[3], b = 0.02 + 0.08 * r[4];
        int inside;
        if (r[0] < 0.5) {
          inside = (x - cx) * (x - cx) + (y - cy) * (y - cy) <= a * a;
        } else {
          inside = x >= cx - a && x <= cx + a && y >= cy - b && y <= cy + b;
        }
        if (inside) v = r[5];
      }
      out[iy * nx + ix] = v;
    }
  }
  free(sh);
}

void orc_phantom_ellipsoids3d(size_t nx, size_t ny, size_t nz, int count, double semi_lo,
                              double semi_hi, double vlo, double vhi, uint64_t seed,
                              double* out) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  memset(out, 0, sizeof(double) * nx * ny * nz);
  for (int k = 0; k < count; ++k) {
    /* centres and semi-axes in voxel units; voxel centres at i + 0.5 */
    const double cx = orc_uniform(&s) * (double)nx;
    const double cy = orc_uniform(&s) * (double)ny;
    const double cz = orc_uniform(&s) * (double)nz;
    const double a = semi_lo + (semi_hi - semi_lo) * orc_uniform(&s);
    const double b = semi_lo + (semi_hi - semi_lo) * orc_uniform(&s);
    const double c = semi_lo + (semi_hi - semi_lo) * orc_uniform(&s);
    const double val = vlo + (vhi - vlo) * orc_uniform(&s);
    long x0 = (long)floor(cx - a) - 1, x1 = (long)ceil(cx + a) + 1;
    long y0 = (long)floor(cy - b) - 1, y1 = (long)ceil(cy + b) + 1;
    long z0 = (long)floor(cz - c) - 1, z1 = (long)ceil(cz + c) + 1;
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (z0 < 0) z0 = 0;
    if (x1 > (long)nx - 1) x1 = (long)nx - 1;
    if (y1 > (long)ny - 1) y1 = (long)ny - 1;
    if (z1 > (long)nz - 1) z1 = (long)nz - 1;
    for (long z = z0; z <= z1; ++z) {
      const double dz = ((double)z + 0.5 - cz) / c;
      for (long y = y0; y <= y1; ++y) {
        const double dy = ((double)y + 0.5 - cy) / b;
        for (long x = x0; x <= x1; ++x) {
          const double dx = ((double)x + 0.5 - cx) / a;
          if (dx * dx + dy * dy + dz * dz <= 1.0) out[((size_t)z * ny + (size_t)y) * nx + (size_t)x] = val;
        }
      }
    }
  }
}

void orc_fdot_tables(size_t n, int n_src, int n_det, double mu, uint64_t seed, double* gs,
                     double* gd) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  const size_t N = n * n * n;
  double* src = (double*)malloc(sizeof(double) * 3 * (size_t)n_src);
  double* det = (double*)malloc(sizeof(double) * 3 * (size_t)n_det);
  for (int k = 0; k < n_src; ++k) {
    src[3 * k] = orc_uniform(&s) * (double)n;
    src[3 * k + 1] = orc_uniform(&s) * (double)n;
    src[3 * k + 2] = 0.0;
  }
  for (int k = 0; k < n_det; ++k) {
    det[3 * k] = orc_uniform(&s) * (double)n;
    det[3 * k + 1] = orc_uniform(&s) * (double)n;
    det[3 * k + 2] = (double)n;
  }
  const double four_pi = 4.0 * M_PI;
  for (int pass = 0; pass < 2; ++pass) {
    const int cnt = pass == 0 ? n_src : n_det;
    const double* pts = pass == 0 ? src : det;
    double* out = pass == 0 ? gs : gd;
    for (int k = 0; k < cnt; ++k) {
      size_t i = 0;
      for (size_t z = 0; z < n; ++z)
        for (size_t y = 0; y < n; ++y)
          for (size_t x = 0; x < n; ++x, ++i) {
            const double dx = (double)x + 0.5 - pts[3 * k];
            const double dy = (double)y + 0.5 - pts[3 * k + 1];
            const double dz = (double)z + 0.5 - pts[3 * k + 2];
            const double r = sqrt(dx * dx + dy * dy + dz * dz);
            out[(size_t)k * N + i] = exp(-mu * r) / (four_pi * r);
          }
    }
  }
  free(src);
  free(det);
}

void orc_fdot_matrix(size_t N, int n_src, int n_det, const double* gs, const double* gd,
                     double* a) {
  for (int s = 0; s < n_src; ++s)
    for (int d = 0; d < n_det; ++d) {
      double* row = a + ((size_t)s * (size_t)n_det + (size_t)d) * N;
      const double* ps = gs + (size_t)s * N;
      const double* pd = gd + (size_t)d * N;
      for (size_t x = 0; x < N; ++x) row[x] = ps[x] * pd[x];
    }
}

int orc_linop_apply_cb(void* op, const double* x, double* y) {
  orc_linop_apply((const orc_linop*)op, x, y);
  return 0;
}
int orc_linop_adjoint_cb(void* op, const double* y, double* x) {
  orc_linop_adjoint((const orc_linop*)op, y, x);
  return 0;
}
int orc_map_solve_cb(void* m, const double* p, double* v) {
  orc_map_solve((const orc_map*)m, p, v);
  return 0;
}

/* ======================================================================== */
/* cg_normal (krylov.cpp:551-628)                                            */
/* ======================================================================== */
int orc_cg_normal(const orc_linop* a, const orc_grid* gr, const double* cx, const double* cy,
                  const double* cz, double eps, double tau, const double* g, const orc_stop* stop,
                  double* f_out, orc_iter_rec* trace, orc_solve_info* info) {
  orc_solve_info dummy;
  if (!info) info = &dummy;
  memset(info, 0, sizeof(*info));
  if (stop_validate(stop)) return ORC_EINVAL;
  if (!(tau >= 0.0)) return ORC_EINVAL;
  const size_t n = a->cols, m = a->rows;
  if (gr->nx * gr->ny * gr->nz != n) return ORC_EDIM;
  const size_t Ls = a->sol_len, Ld = a->data_len;
  const double nan = NAN;
  int status = ORC_OK;
  double* x = (double*)calloc(n, sizeof(double));
  double* b = (double*)malloc(sizeof(double) * n);
  double* r = (double*)malloc(sizeof(double) * n);
  double* d = (double*)malloc(sizeof(double) * n);
  double* q = (double*)malloc(sizeof(double) * n);
  double* mx = (double*)malloc(sizeof(double) * n);
  double* tr = (double*)malloc(sizeof(double) * m);
  orc_linop_adjoint(a, g, b); /* b = A^T g */
  memcpy(r, b, sizeof(double) * n);
  memcpy(d, r, sizeof(double) * n);
  double rho = dotL(r, r, n, Ls);
  const double nres0 = sqrt(rho);
  info->stop_reason = ORC_STOP_MAX_ITERS;
  if (nres0 == 0.0) {
    info->stop_reason = ORC_STOP_BREAKDOWN;
    goto done;
  }
  for (int iter = 1; iter <= stop->max_iters; ++iter) {
    /* q = (A^T A + tau M) d */
    orc_linop_apply(a, d, tr);
    orc_linop_adjoint(a, tr, q);
    if (tau > 0.0) {
      orc_m_apply(gr, cx, cy, cz, eps, d, mx);
      axpy(tau, mx, q, n);
    }
    const double curv = dotL(d, q, n, Ls);
    if (!(curv > 0.0)) {
      status = ORC_EBREAKDOWN;
      info->breakdown_iteration = iter;
      goto done;
    }
    const double gamma = rho / curv;
    axpy(gamma, d, x, n);
    axpy(-gamma, q, r, n);
    const double rho_next = dotL(r, r, n, Ls);

    orc_iter_rec row;
    memset(&row, 0, sizeof(row));
    row.iteration = iter;
    /* exact_data_residual: distance(g, A x) (krylov.cpp:110-123) */
    orc_linop_apply(a, x, tr);
    for (size_t i = 0; i < m; ++i) tr[i] = g[i] - tr[i];
    row.res_data = sqrt(dotL(tr, tr, m, Ld));
    row.res_data_exact = 1;
    if (tau > 0.0) {
      orc_m_apply(gr, cx, cy, cz, eps, x, mx); /* SparseSpd::quadratic_form = sum x_i (Mx)_i */
      row.res_damped = sqrt(row.res_data * row.res_data + tau * dotL(x, mx, n, Ls));
    } else {
      row.res_damped = row.res_data;
    }
    row.s2_value = sqrt(rho_next) / nres0;
    row.anorm_est = nan;
    row.cond_est = nan;
    row.xnorm_est = nrm2L(x, n, Ls);
    if (trace) trace[iter - 1] = row;
    info->iterations = iter;
    if (stop->use_s4 && row.res_data <= stop->eta * stop->delta) {
      info->stop_reason = ORC_STOP_S4;
      break;
    }
    if (stop->use_s2 && row.s2_value <= stop->atol) {
      info->stop_reason = ORC_STOP_S2;
      break;
    }
    if (rho_next == 0.0) {
      info->stop_reason = ORC_STOP_BREAKDOWN;
      break;
    }
    if (iter >= stop->max_iters) break;
    xpby(r, rho_next / rho, d, n);
    rho = rho_next;
  }
done:
  if (f_out) memcpy(f_out, x, sizeof(double) * n);
  free(x); free(b); free(r); free(d); free(q); free(mx); free(tr);
  return status;
}

/* ======================================================================== */
/* krylov_basis (krylov.cpp:700-754): Gram-Schmidt with one reorthogonalization */
/* ======================================================================== */
int orc_krylov_basis(const orc_linop* a, const orc_map* msolver, const orc_grid* mg,
                     const double* cx, const double* cy, const double* cz, double eps, double tau,
                     const double* g, int k, double* out, int* count, int* rank_exhausted) {
  *count = 0;
  *rank_exhausted = 0;
  if (msolver && mg) return ORC_EINVAL;
  if (k < 1) return ORC_EINVAL;
  const size_t n = a->cols, L = a->sol_len;
  size_t mnx = 0, mny = 0, mnz = 0;
  if (mg) {
    grid_ext(mg, &mnx, &mny, &mnz);
    if (mnx * mny * mnz != n) return ORC_EDIM;
    if (mg->dims < 2) cy = NULL;
    if (mg->dims < 3) cz = NULL;
  }
  double* t = (double*)malloc(sizeof(double) * n);
  double* scratch = (double*)malloc(sizeof(double) * n);
  double* rows = (double*)malloc(sizeof(double) * a->rows);
  orc_linop_adjoint(a, g, t);
  if (msolver) {
    orc_map_solve(msolver, t, scratch);
    memcpy(t, scratch, sizeof(double) * n);
  }
  const double seed_norm = nrm2L(t, n, L);
  if (seed_norm == 0.0) {
    *rank_exhausted = 1;
  } else {
    for (int j = 0; j < k; ++j) {
      if (j > 0) {
        const double* prev = out + (size_t)(*count - 1) * n;
        orc_linop_apply(a, prev, rows);
        orc_linop_adjoint(a, rows, t);
        if (mg && tau > 0.0) {
          m_apply_ext(mnx, mny, mnz, cx, cy, cz, eps, prev, scratch);
          axpy(tau, scratch, t, n);
        }
        if (msolver) {
          orc_map_solve(msolver, t, scratch);
          memcpy(t, scratch, sizeof(double) * n);
        }
      }
      const double before = nrm2L(t, n, L);
      for (int pass = 0; pass < 2; ++pass)
        for (int q = 0; q < *count; ++q) {
          const double* qv = out + (size_t)q * n;
          axpy(-dotL(qv, t, n, L), qv, t, n);
        }
      const double after = nrm2L(t, n, L);
      if (after <= 1e-12 * (before > seed_norm ? before : seed_norm)) {
        *rank_exhausted = 1;
        break;
      }
      scal(1.0 / after, t, n);
      memcpy(out + (size_t)*count * n, t, sizeof(double) * n);
      ++*count;
    }
  }
  free(t);
  free(scratch);
  free(rows);
  return ORC_OK;
}
