/*
 * oracle/mlsqr_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference's priorconditioned-LSQR path
 * (arXiv 1308.6634 reference `mlsqr`, /root/reference/proj).  It is the
 * checker the CUDA product is compared against.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it; the product library never links or calls it.
 *
 * Pinning: the parts that exist in the reference (1D/2D Gaussian blur,
 * dense operator, penalty / diffusivity, edge-based M, mlsqr / lsqr,
 * LsqrRecurrence, stopping, nonlinear outer loop, GaussianSampler) are
 * checked against fixtures produced by the reference itself
 * (oracle/_ref/libmlsqr_ref.so built from /root/reference/proj/src, see
 * tests/golden/make_golden.py).  The parts the reference lacks (3D blur,
 * 3D edge grid, V-cycle SpdMap, fDOT-like generator, seeded phantoms,
 * relative noise, fixed-count outer driver) are restated in the reference's
 * conventions and are "parity unpinned" against the reference: they are
 * pinned by property tests (adjoint, Kronecker, SPD, constants) instead.
 */
#ifndef MLSQR_ORACLE_H
#define MLSQR_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirror include/mlsqr_b200.h) ---- */
#define ORC_OK 0
#define ORC_EDIM 1
#define ORC_EINVAL 2
#define ORC_EBREAKDOWN 3

/* ---- RNG: std::mt19937_64 + GaussianSampler (problems.cpp:12-28, rng.hpp:9-28) ---- */
typedef struct {
  uint64_t mt[312];
  int mti;
} orc_mt64;
void orc_mt64_seed(orc_mt64* s, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* s);
/* u = ((x >> 11) + 1) * 2^-53 in (0, 1]  (problems.cpp:17-18) */
double orc_uniform(orc_mt64* s);
void orc_gauss_fill(uint64_t seed, size_t n, double stddev, double* out);

/* ---- penalty (penalty.cpp:35-84) ---- */
enum { ORC_PEN_TIKHONOV = 0, ORC_PEN_TV = 1, ORC_PEN_PM_LOG = 2, ORC_PEN_PM_EXP = 3 };
double orc_r_value(int kind, double T, double t);
double orc_diffusivity(int kind, double T, double t);

/* ---- grid (grid.hpp:9-27, extended to 3D with edge weight h^3) ---- */
typedef struct {
  int dims;              /* 1, 2, 3 */
  size_t nx, ny, nz;     /* unused extents are 1 */
  double h;              /* spacing */
} orc_grid;

/* taps t_k = h * sqrt(2/(pi s^2)) * exp(-d^2/(2 s^2)), d = (k-R) h  (linop.cpp:93-102);
 * radius < 0 selects the reference radius ceil(6 s / h).  Returns the radius. */
int orc_taps(size_t n, double sigma_f, double domain_length, int radius, double* taps_out);

/* ---- linear operators (linop.hpp:21-126) ---- */
typedef struct orc_linop orc_linop;
orc_linop* orc_identity_new(size_t n);
orc_linop* orc_dense_new(size_t rows, size_t cols, const double* row_major); /* borrows */
orc_linop* orc_blur_new(int dims, size_t nx, size_t ny, size_t nz, int radius,
                        const double* taps); /* copies taps (same taps on every axis) */
void orc_linop_free(orc_linop* op);
size_t orc_linop_rows(const orc_linop* op);
size_t orc_linop_cols(const orc_linop* op);
void orc_linop_apply(const orc_linop* op, const double* x, double* y);
void orc_linop_adjoint(const orc_linop* op, const double* y, double* x);

/* ---- edge-based diffusion operator M (diffusion.cpp:27-106) ---- */
/* c_e = diffusivity(|(f_j - f_i)/h|) * w_e / h^2, one array per axis, zero where no edge. */
int orc_edge_coeffs(const orc_grid* g, const double* f, int pen_kind, double T,
                    double* cx, double* cy, double* cz);
double orc_max_diag(const orc_grid* g, const double* cx, const double* cy, const double* cz);
/* y = (M_unshifted + eps I) x with the CSR row order of sparse.cpp:65-74 */
void orc_m_apply(const orc_grid* g, const double* cx, const double* cy, const double* cz,
                 double eps, const double* x, double* y);
double orc_penalty_functional(const orc_grid* g, const double* f, int pen_kind, double T);

/* ---- SPD maps (spdsolve.hpp:11-33) ---- */
typedef struct orc_map orc_map;
orc_map* orc_identity_map_new(size_t n);
/* dense Cholesky solve of a row-major SPD matrix (tests/support/oracles.hpp:56-73 style) */
orc_map* orc_dense_chol_map_new(size_t n, const double* m_row_major);
/* V-cycle on the edge operator: aggregation coarsening, Galerkin edge sums,
 * omega-Jacobi pre/post sweeps, fixed coarse sweeps (SURVEY.md §7 hard part 2). */
orc_map* orc_vcycle_new(const orc_grid* g, int levels, int nu_pre, int nu_post, double omega,
                        int coarse_sweeps);
int orc_vcycle_set(orc_map* m, const double* cx, const double* cy, const double* cz, double eps);
/* hierarchy inspection: level l extents and edge coefficients */
int orc_vcycle_level(const orc_map* m, int l, size_t* dims3, double* cx, double* cy, double* cz,
                     double* eps);
typedef void (*orc_map_fn)(void* ctx, const double* p, double* v);
orc_map* orc_callback_map_new(size_t n, orc_map_fn fn, void* ctx);
/* SpdSolver::factorize (spdsolve.cpp:22-75): envelope Cholesky of M + eps I from edge
 * coefficients, reference operation order in both modes (sequential dots); NULL and
 * *pivot_row >= 0 on a nonpositive pivot (FactorizationError). */
orc_map* orc_env_chol_map_new(const orc_grid* g, const double* cx, const double* cy,
                              const double* cz, double eps, long long* pivot_row);
/* SpdSolver::inner_cg (spdsolve.cpp:77-85, 119-137): k_inner CG iterations from zero */
orc_map* orc_inner_cg_map_new(const orc_grid* g, const double* cx, const double* cy,
                              const double* cz, double eps, int k_inner);
void orc_map_free(orc_map* m);
void orc_map_solve(const orc_map* m, const double* p, double* v);

/* ---- Krylov (krylov.hpp:19-95, krylov.cpp:24-440) ---- */
typedef struct {
  double atol, btol, conlim, delta, eta;
  int max_iters;
  int use_s1, use_s2, use_s3, use_s4;
} orc_stop;

/* IterationRecord (krylov.hpp:41-52) */
typedef struct {
  int iteration;
  int res_data_exact;
  double res_damped, res_data, s2_value, anorm_est, cond_est, xnorm_est, alpha, beta;
} orc_iter_rec;

enum { ORC_STOP_S1 = 0, ORC_STOP_S2, ORC_STOP_S3, ORC_STOP_S4, ORC_STOP_MAX_ITERS,
       ORC_STOP_BREAKDOWN };

typedef struct {
  int iterations;
  int stop_reason;
  int n_alphas, n_betas;
  int breakdown_iteration; /* set when ORC_EBREAKDOWN is returned */
} orc_solve_info;

/* f_out[n]; trace[max_iters]; alphas[max_iters+1]; betas[max_iters+2]; any output may be NULL.
 * snapshots (optional, max_iters*n) receives f_i per iteration. */
int orc_mlsqr(const orc_linop* a, const orc_map* msolver, const double* g, double tau,
              const orc_stop* stop, double* f_out, orc_iter_rec* trace, double* alphas,
              double* betas, double* snapshots, orc_solve_info* info);
int orc_lsqr(const orc_linop* a, const double* g, double tau, const orc_stop* stop,
             double* f_out, orc_iter_rec* trace, double* alphas, double* betas,
             double* snapshots, orc_solve_info* info);
/* cg_normal (krylov.cpp:551-628): CG on the normal equation (A^T A + tau M) f = A^T g, the
 * unpriorconditioned baseline.  M = the edge operator (cx, cy, cz) + eps I on grid gr, applied
 * in CSR row order (sparse.cpp:65-74); its quadratic form is x . (M x) (sparse.cpp:82-93).
 * Returns ORC_EBREAKDOWN (info->breakdown_iteration) on nonpositive curvature. */
int orc_cg_normal(const orc_linop* a, const orc_grid* gr, const double* cx, const double* cy,
                  const double* cz, double eps, double tau, const double* g, const orc_stop* stop,
                  double* f_out, orc_iter_rec* trace, orc_solve_info* info);

/* ---- lagged-diffusivity outer loop (outer.cpp:31-100) with a V-cycle M^{-1} ---- */
typedef struct {
  double tau;
  int pen_kind;
  double T;
  orc_stop inner_stop;
  int inner_cap;
  double rel_decrease_threshold; /* <= 0: fixed count (no stagnation break) */
  int max_outer;
  double epsilon;                /* < 0: auto shift 1e-8 * max diag */
  int mg_levels, nu_pre, nu_post, coarse_sweeps;
  double omega;
  int spd_mode; /* 0: V-cycle (mg_levels > 0) or dense Cholesky (mg_levels == 0);
                   1: envelope Cholesky (SpdSolver::factorize); 2: inner CG (k_inner) */
  int k_inner;
} orc_outer_cfg;

typedef struct {
  int k;
  int inner_iterations;
  int inner_stop;
  double penalty_value;
  double final_residual;
  double eps_used;
} orc_outer_step;

/* steps[max_outer]; alphas/betas optional per-step blocks of (inner_cap+1)/(inner_cap+2);
 * iterates optional per-step blocks of n (f^k). Returns status. */
int orc_nonlinear(const orc_linop* a, const double* g, const orc_grid* grid,
                  const orc_outer_cfg* cfg, double* f_out, orc_outer_step* steps,
                  int* n_steps, int* stop_reason, int* triggered_at, double* alphas,
                  double* betas, double* iterates);

int orc_outer_stop_check(const double* history, int k, double threshold);

/* ---- seeded synthetic problems (new; reference conventions of problems.cpp) ---- */
/* C1: `count` axis-aligned rectangles, corners U^2 sorted, value U; painted in order */
void orc_phantom_rects2d(size_t nx, size_t ny, int count, uint64_t seed, double* out);
/* C2: discs or rectangles by coin flip; radius/half-widths 0.02 + 0.08 U; value U */
void orc_phantom_shapes2d(size_t nx, size_t ny, int count, uint64_t seed, double* out);
/* C3/C5: axis-aligned ellipsoids, centres U*n voxels, semi-axes U[lo,hi] voxels,
 * values U[vlo,vhi]; painted in order */
void orc_phantom_ellipsoids3d(size_t nx, size_t ny, size_t nz, int count, double semi_lo,
                              double semi_hi, double vlo, double vhi, uint64_t seed,
                              double* out);
/* fDOT-like Green tables: gs[s*N + x] = G(src_s, x), gd[d*N + x] = G(x, det_d),
 * G(a,x) = exp(-mu r)/(4 pi r), sources U on z=0 face, detectors U on z=n face. */
void orc_fdot_tables(size_t n, int n_src, int n_det, double mu, uint64_t seed, double* gs,
                     double* gd);
/* A[(s*n_det + d)*N + x] = gs[s,x] * gd[d,x] */
void orc_fdot_matrix(size_t N, int n_src, int n_det, const double* gs, const double* gd,
                     double* a);

/* DEVICE arithmetic order switch (see mlsqr_oracle.c "arithmetic order") */
/* krylov_basis (krylov.cpp:700-754): msolver XOR the stencil M (mg, cx, cy, cz, eps) or neither;
 * out: k x cols; *count vectors written */
int orc_krylov_basis(const orc_linop* a, const orc_map* msolver, const orc_grid* mg,
                     const double* cx, const double* cy, const double* cz, double eps, double tau,
                     const double* g, int k, double* out, int* count, int* rank_exhausted);
void orc_set_device_order(int on);
int orc_get_device_order(void);
double orc_canon_dot(const double* x, const double* y, size_t n, size_t row_len);
double orc_dhypot(double a, double b);
/* row lengths used by the canonical reductions in data / solution space */
void orc_linop_set_row_lengths(orc_linop* op, size_t data_len, size_t sol_len);

/* int-returning callback adapters (signature int(*)(void*, const double*, double*)) so the
 * reference's mlsqr can be driven by oracle operators / maps through ref_capi.cpp */
int orc_linop_apply_cb(void* op, const double* x, double* y);
int orc_linop_adjoint_cb(void* op, const double* y, double* x);
int orc_map_solve_cb(void* m, const double* p, double* v);

#ifdef __cplusplus
}
#endif
#endif
