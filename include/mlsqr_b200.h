/*
 * include/mlsqr_b200.h -- C-ABI of the B200-native priorconditioned-LSQR path.
 *
 * Drop-in boundary for the reference's hot path (arXiv 1308.6634 reference,
 * /root/reference/proj).  Every entry point below replaces one reference
 * interface; the file:line of that interface is cited.  No C++ or torch types
 * cross this boundary: plain pointers, sizes and int status codes.  Errors
 * never throw; they return a status and leave a thread-local message in
 * mlsqr_last_error().  include/mlsqr_b200.hpp rethrows them as the
 * reference's exception types (errors.hpp:9-41).
 *
 * Pointer kinds: MLSQR_HOST buffers are copied in/out around the call (the
 * reference's std::span contract, linop.hpp:33-36); MLSQR_DEVICE buffers are
 * cudaMalloc'ed memory on the context's device and stay resident.
 * Stream ordering of MLSQR_DEVICE buffers: the library reads and writes them on
 * the context's stream only.  A library-owned stream (NULL at mlsqr_ctx_create)
 * is created cudaStreamNonBlocking, so it does NOT wait for work the caller
 * queued elsewhere: either create the context on the stream that produces the
 * inputs, or synchronize that stream before the call.  Every call returns
 * after the context's stream has drained, so outputs are ready on return.
 *
 * Arithmetic: fp64 everywhere, in the canonical device order documented in
 * DESIGN.md (bit-exact with the oracle's DEVICE order).
 */
#ifndef MLSQR_B200_H
#define MLSQR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:9-41) ---- */
#define MLSQR_OK 0
#define MLSQR_EDIM 1        /* DimensionError            (errors.hpp:9-13)  */
#define MLSQR_EINVAL 2      /* std::invalid_argument     (krylov.cpp:219-226) */
#define MLSQR_EBREAKDOWN 3  /* BreakdownError(iteration) (errors.hpp:27-36) */
#define MLSQR_ECUDA 4       /* CUDA runtime failure / no device              */
#define MLSQR_ENCCL 5       /* collective failure                            */
#define MLSQR_ECALLBACK 6   /* a host callback (plugin SpdMap) failed        */
#define MLSQR_EFACTOR 7     /* FactorizationError(pivot_row) (errors.hpp:14-24) */

#define MLSQR_HOST 0
#define MLSQR_DEVICE 1

/* penalty kinds (penalty.hpp:6-12) */
#define MLSQR_PEN_TIKHONOV 0
#define MLSQR_PEN_TV 1
#define MLSQR_PEN_PM_LOG 2
#define MLSQR_PEN_PM_EXP 3

/* stop reasons (krylov.hpp:38) */
#define MLSQR_STOP_S1 0
#define MLSQR_STOP_S2 1
#define MLSQR_STOP_S3 2
#define MLSQR_STOP_S4 3
#define MLSQR_STOP_MAX_ITERS 4
#define MLSQR_STOP_BREAKDOWN 5

typedef struct mlsqr_ctx mlsqr_ctx;
typedef struct mlsqr_op mlsqr_op;
typedef struct mlsqr_pc mlsqr_pc;

/* thread-local message of the last failing call */
const char* mlsqr_last_error(void);
/* library/build identification, e.g. "mlsqr_b200 sm_100a fp64" */
const char* mlsqr_version(void);

/* ---- context: device + stream (+ optional communicator, see mlsqr_ctx_set_comm) ---- */
int mlsqr_ctx_create(int device, void* cuda_stream /* NULL: library-owned stream */,
                     mlsqr_ctx** out);
int mlsqr_ctx_destroy(mlsqr_ctx* ctx);
int mlsqr_ctx_synchronize(mlsqr_ctx* ctx);
/* device memory helpers for callers without their own allocator */
int mlsqr_dev_alloc(mlsqr_ctx* ctx, size_t bytes, void** ptr);
int mlsqr_dev_free(mlsqr_ctx* ctx, void* ptr);
int mlsqr_copy(mlsqr_ctx* ctx, void* dst, int dst_kind, const void* src, int src_kind,
               size_t bytes);
/* count of this library's kernel launches since the last reset (bench gpu_launches) */
uint64_t mlsqr_ctx_launch_count(mlsqr_ctx* ctx, int reset);
/* per-kernel-class device timing with CUDA events inside the solve (0 = off) */
int mlsqr_ctx_set_timing(mlsqr_ctx* ctx, int enable);
/* accumulated [ms, launches] for timing class `cls` (see MLSQR_TCLASS_*) */
int mlsqr_ctx_get_timing(mlsqr_ctx* ctx, int cls, double* ms, uint64_t* launches);
#define MLSQR_TCLASS_BLUR 0    /* A / A^T blur applications + fused epilogue   */
#define MLSQR_TCLASS_DENSE 1   /* dense GEMV / GEMV^T + fused epilogue          */
#define MLSQR_TCLASS_SMOOTH 2  /* V-cycle level-0 smoothing sweeps              */
#define MLSQR_TCLASS_MG 3      /* whole V-cycle (all levels)                    */
#define MLSQR_TCLASS_UPDATE 4  /* LSQR vector update (f, w, q) + w.q           */
#define MLSQR_TCLASS_ITER 5    /* whole LSQR iteration                          */
#define MLSQR_TCLASS_SWEEP_FN 6       /* level-0 pre-sweeps 1+2 (one fused kernel)    */
#define MLSQR_TCLASS_SWEEP_PROLONG 7  /* level-0 prolongation + post-sweep 1          */
#define MLSQR_TCLASS_SWEEP_LAST 8     /* level-0 plain sweep (last post-sweep)        */
#define MLSQR_TCLASS_RESTRICT 9       /* level-0 residual + restriction               */
#define MLSQR_TCLASS_HALO 10          /* z-slab ghost-plane exchanges (any stream)    */
#define MLSQR_TCLASS_COLL 11          /* allgathers / allreduces of the decomposition */
#define MLSQR_TCLASS_COUNT 12

/* ---- z-slab decomposition (multi-GPU) ----------------------
 * A context can own a slab of a global 3D grid: every grid object created on it with z
 * extent nz is the plane range [z_offset, z_offset + nz) of a grid with nz_global planes.
 * Ghost planes travel through the context's communicator: NCCL (one process per GPU) or
 * a loopback group (P virtual ranks of one process, each on its own thread/context --
 * used to verify sharded == unsharded bit for bit on a single GPU). */
int mlsqr_nccl_unique_id(void* out, size_t cap, size_t* len);
int mlsqr_ctx_set_comm_nccl(mlsqr_ctx* ctx, const void* unique_id, int rank, int size);
int mlsqr_loop_group_create(int size, void** group);
int mlsqr_loop_group_destroy(void* group);
int mlsqr_ctx_set_comm_loopback(mlsqr_ctx* ctx, void* group, int rank);
int mlsqr_ctx_set_slab(mlsqr_ctx* ctx, size_t nz_global, size_t z_offset);
/* Row shards (DenseOperator linop.hpp:59-71 with its rows split over ranks):
 * rank k holds data rows [row_offset, row_offset + rows_global / P) of every data-space vector
 * and of the dense operator (mlsqr_dense_create takes the local rows; the fDOT generator forms
 * them).  The solution space and the preconditioner are replicated.  A x is local; A^T u
 * allgathers the 8 canonical row-chunk partials and sums them in chunk order, and the data-space
 * norms allgather their segment partials -- so P in {1, 2, 4, 8} is bit-identical to P = 1.
 * Needs rows_global % 8 == 0 and whole 32-row segments per rank. */
int mlsqr_ctx_set_row_shard(mlsqr_ctx* ctx, size_t rows_global, size_t row_offset);

/* ---- LinearOperator (linop.hpp:21-47) ----------------------------------- */
/* Separable Gaussian blur with explicit taps (SeparableGaussianBlur2D, linop.hpp:110-126,
 * GaussianConvolution1D, linop.hpp:83-105; 3D = third z pass).  taps: 2*radius+1 host
 * values, identical on every axis; zero extension; self-adjoint. */
int mlsqr_blur_create(mlsqr_ctx* ctx, int dims, size_t nx, size_t ny, size_t nz,
                      const double* taps, int radius, mlsqr_op** out);
/* SeparableGaussianBlur2D (linop.hpp:110-126, linop.cpp:142-170) with one factor per axis,
 * kx_(nx) and ky_(ny) (linop.cpp:144-147): on a non-square grid the spacings 1/nx, 1/ny give
 * different taps and radii.  x pass then y pass, separate mul + add: bit-identical to the
 * reference's scalar backend. */
int mlsqr_blur2d_create_axes(mlsqr_ctx* ctx, size_t nx, size_t ny, const double* taps_x, int radius_x,
                             const double* taps_y, int radius_y, mlsqr_op** out);
/* DenseOperator (linop.hpp:59-71): row-major rows x cols.  a_kind HOST copies to device.
 * sol_row_len: row length of solution-space vectors for the canonical reductions
 * (the x-extent of the voxel grid; 0 = cols). */
int mlsqr_dense_create(mlsqr_ctx* ctx, size_t rows, size_t cols, const double* a, int a_kind,
                       size_t sol_row_len, mlsqr_op** out);
/* fDOT-like dense operator formed on the device: A[s*n_det+d, x] = gs[s,x] * gd[d,x]
 * (host tables from mlsqr_fdot_tables). */
int mlsqr_dense_create_fdot(mlsqr_ctx* ctx, size_t n_vox, int n_src, int n_det,
                            const double* gs, const double* gd, size_t sol_row_len,
                            mlsqr_op** out);
/* IdentityOperator (linop.hpp:49-56) */
int mlsqr_identity_create(mlsqr_ctx* ctx, size_t n, size_t row_len, mlsqr_op** out);
int mlsqr_op_destroy(mlsqr_op* op);
int mlsqr_op_shape(const mlsqr_op* op, size_t* rows, size_t* cols);
/* LinearOperator::apply / apply_adjoint (linop.cpp:30-40): EDIM on length mismatch */
int mlsqr_op_apply(mlsqr_op* op, const double* x, size_t x_len, double* y, size_t y_len,
                   int ptr_kind);
int mlsqr_op_apply_adjoint(mlsqr_op* op, const double* y, size_t y_len, double* x,
                           size_t x_len, int ptr_kind);

/* ---- SpdMap (spdsolve.hpp:11-33) ----------------------------------------- */
int mlsqr_identity_map_create(mlsqr_ctx* ctx, size_t n, mlsqr_pc** out);
/* Multigrid V-cycle on the edge-based diffusion operator M (diffusion.hpp:12-20):
 * 2^d aggregation, Galerkin edge sums, omega-Jacobi nu_pre/nu_post sweeps, fixed coarse
 * sweeps.  The SpdMap plug point named at spdsolve.hpp:13-14. */
int mlsqr_vcycle_create(mlsqr_ctx* ctx, int dims, size_t nx, size_t ny, size_t nz, double h,
                        int levels, int nu_pre, int nu_post, double omega, int coarse_sweeps,
                        mlsqr_pc** out);
/* explicit level-0 edge coefficients (one array per axis, zero where no edge) + shift */
int mlsqr_vcycle_set_coefficients(mlsqr_pc* pc, const double* cx, const double* cy,
                                  const double* cz, double eps, int ptr_kind);
/* assemble_m + auto_shift (diffusion.cpp:59-87) on the device from a field f:
 * c_e = diffusivity(|grad f|) w_e/h^2; eps < 0 selects 1e-8 * max diagonal. */
int mlsqr_vcycle_update(mlsqr_pc* pc, const double* f, int ptr_kind, int pen_kind, double T,
                        double eps, double* eps_used);
/* host plug-in SpdMap: fn(ctx, p, v) with host vectors (parity / test fakes) */
typedef int (*mlsqr_host_map_fn)(void* user, const double* p, double* v);
int mlsqr_callback_map_create(mlsqr_ctx* ctx, size_t n, mlsqr_host_map_fn fn, void* user,
                              mlsqr_pc** out);
/* SpdSolver::factorize (spdsolve.hpp:42-70, spdsolve.cpp:22-75) + solve_cholesky (:101-117):
 * envelope Cholesky of the level-0 M (+ shift) the V-cycle map `m` currently holds (set by
 * mlsqr_vcycle_set_coefficients / _update; a 1-level V-cycle is a plain holder of M).  Factor
 * and substitutions run on the device in the reference's operation order (sequential dots,
 * bit-identical to its scalar backend).  MLSQR_EFACTOR on a nonpositive pivot, its row in
 * *pivot_row (may be NULL).  For small grids: the envelope holds n * (bandwidth + 1) doubles. */
int mlsqr_chol_map_create(mlsqr_pc* m, mlsqr_pc** out, long long* pivot_row);
/* SpdSolver::inner_cg (spdsolve.cpp:77-85, solve_cg :119-137): exactly k_inner CG iterations
 * from zero on a snapshot of the level-0 M of `m`, canonical device dots, graph-capturable. */
int mlsqr_inner_cg_map_create(mlsqr_pc* m, int k_inner, mlsqr_pc** out);
int mlsqr_pc_destroy(mlsqr_pc* pc);
int mlsqr_pc_dimension(const mlsqr_pc* pc, size_t* n);
/* SpdMap::solve: v ~= M^{-1} p */
int mlsqr_pc_solve(mlsqr_pc* pc, const double* p, double* v, size_t n, int ptr_kind);
/* y = (M + eps I) x for the level-0 operator of a V-cycle (tests / R(f) gradient) */
int mlsqr_vcycle_m_apply(mlsqr_pc* pc, const double* x, double* y, size_t n, int ptr_kind);

/* ---- Krylov (krylov.hpp:19-95) ------------------------------------------- */
typedef struct {            /* StoppingConfig (krylov.hpp:19-36) */
  double atol, btol, conlim, delta, eta;
  int max_iters;
  int use_s1, use_s2, use_s3, use_s4;
} mlsqr_stop;

typedef struct {            /* IterationRecord (krylov.hpp:41-52) */
  int iteration;
  int res_data_exact;
  double res_damped, res_data, s2_value, anorm_est, cond_est, xnorm_est, alpha, beta;
} mlsqr_iter_rec;

typedef struct {
  int iterations;
  int stop_reason;          /* MLSQR_STOP_* */
  int n_alphas, n_betas;    /* BidiagEntries sizes after trim (krylov.cpp:182-186) */
  int breakdown_iteration;  /* BreakdownError::iteration() when MLSQR_EBREAKDOWN */
  int n_left_basis;         /* left basis vectors stored by mlsqr_solve_basis (else 0) */
} mlsqr_solve_info;

/* mlsqr (krylov.hpp:94-95, krylov.cpp:335-440): device-resident loop.
 * g: n_rows; f: n_cols; trace: max_iters rows; alphas: max_iters+1; betas: max_iters+2.
 * trace/alphas/betas/info are host arrays (may be NULL); g/f follow ptr_kind. */
int mlsqr_solve(mlsqr_op* op, mlsqr_pc* pc, const double* g, double tau,
                const mlsqr_stop* stop, double* f, mlsqr_iter_rec* trace, double* alphas,
                double* betas, mlsqr_solve_info* info, int ptr_kind);
/* lsqr (krylov.hpp:86-87): the M = I path without a preconditioner solve */
int mlsqr_lsqr_solve(mlsqr_op* op, const double* g, double tau, const mlsqr_stop* stop,
                     double* f, mlsqr_iter_rec* trace, double* alphas, double* betas,
                     mlsqr_solve_info* info, int ptr_kind);

/* mlsqr / lsqr with SolveOptions::store_basis (krylov.hpp:77-79): additionally writes the right
 * basis vtilde_1 .. vtilde_k (the scaled v of krylov.cpp:375-377, 421-423) as the rows of
 * basis[(max_iters + 1) * n_cols] and, when left_basis is non-NULL, the left basis u_1 .. u_{k+1}
 * (krylov.cpp:375-377, 421-425) as the rows of left_basis[(max_iters + 1) * n_rows]
 * (ptr_kind memory); info->n_alphas / info->n_left_basis rows are valid.  pc == NULL runs lsqr. */
int mlsqr_solve_basis(mlsqr_op* op, mlsqr_pc* pc, const double* g, double tau, const mlsqr_stop* stop,
                      double* f, mlsqr_iter_rec* trace, double* alphas, double* betas, double* basis,
                      double* left_basis, mlsqr_solve_info* info, int ptr_kind);
/* SolveOptions (krylov.hpp:77-80) and where their outputs go (ptr_kind memory of the call):
 *   record_snapshots -> snapshots[max_iters x n_cols]: f after each recorded iteration
 *                       (SolveTrace::snapshots, krylov.cpp:159-161); info->iterations rows valid
 *   store_basis      -> basis / left_basis as in mlsqr_solve_basis (left_basis may be NULL) */
typedef struct {
  int record_snapshots;
  int store_basis;
  double* snapshots;
  double* basis;
  double* left_basis;
} mlsqr_solve_opts;
/* mlsqr / lsqr (pc == NULL) with SolveOptions */
int mlsqr_solve_with(mlsqr_op* op, mlsqr_pc* pc, const double* g, double tau, const mlsqr_stop* stop,
                     const mlsqr_solve_opts* opts, double* f, mlsqr_iter_rec* trace, double* alphas,
                     double* betas, mlsqr_solve_info* info, int ptr_kind);
/* cg_normal with SolveOptions::record_snapshots (krylov.cpp:608); store_basis is ignored like
 * the reference (cg_normal has no bidiagonalization) */
int mlsqr_cg_normal_solve_with(mlsqr_op* op, mlsqr_pc* m, const double* g, double tau,
                               const mlsqr_stop* stop, const mlsqr_solve_opts* opts, double* f,
                               mlsqr_iter_rec* trace, mlsqr_solve_info* info, int ptr_kind);
/* solve_projected (krylov.hpp:124-127, krylov.cpp:631-678): y[k] minimising
 * |[B_k; sqrt(tau) I] y - beta1 e1| from k alphas and k+1 betas (host arithmetic; one
 * bidiagonalization serves every tau).  No device needed. */
int mlsqr_solve_projected(const double* alphas, size_t k, const double* betas, size_t n_betas,
                          double beta1, double tau, double* y);
/* reconstruct_from_basis (krylov.hpp:129-131): f = sum_j y_j basis_j for a basis stored by
 * mlsqr_solve_basis (rows of length n; ny <= rows).  y is a host array. */
int mlsqr_reconstruct_from_basis(mlsqr_ctx* ctx, const double* basis, size_t n, const double* y, size_t ny,
                                 double* f, int ptr_kind);

/* cg_normal (krylov.hpp:116-122, krylov.cpp:551-628): CG on (A^T A + tau M) f = A^T g, the
 * unpriorconditioned baseline of the paper's comparison.  M is the level-0 operator of the
 * V-cycle map m (as set by mlsqr_vcycle_set_coefficients / _update; m may be NULL when
 * tau == 0).  Trace rows follow the reference: exact res_data, s2 = |r_k| / |r_0|, NaN
 * anorm/cond estimates; no bidiagonal entries.  MLSQR_EBREAKDOWN on nonpositive curvature. */
int mlsqr_cg_normal_solve(mlsqr_op* op, mlsqr_pc* m, const double* g, double tau,
                          const mlsqr_stop* stop, double* f, mlsqr_iter_rec* trace,
                          mlsqr_solve_info* info, int ptr_kind);

/* krylov_basis (krylov.hpp:133-145, krylov.cpp:700-754): the first k orthonormalized vectors of
 * K^{A^T A} (msolver = m = NULL), K^{A^T A + tau M} (m: a V-cycle map holding M) or
 * K^{M^-1 A^T A} (msolver: any SpdMap), Gram-Schmidt with one reorthogonalization pass.
 * vectors: k x n_cols (ptr_kind memory); *count rows are valid; *rank_exhausted as KrylovBasis. */
int mlsqr_krylov_basis(mlsqr_op* op, mlsqr_pc* msolver, mlsqr_pc* m, double tau, const double* g,
                       int k, double* vectors, int* count, int* rank_exhausted, int ptr_kind);

/* ---- lagged-diffusivity outer loop (outer.hpp:13-62) --------------------- */
typedef struct {            /* OuterConfig (outer.hpp:13-28) with a V-cycle M^{-1} */
  double tau;
  int pen_kind;
  double T;
  mlsqr_stop inner_stop;
  int inner_cap;
  double rel_decrease_threshold;  /* <= 0: fixed outer count (no stagnation break) */
  int max_outer;
  double epsilon;                 /* < 0: auto shift */
  int mg_levels, nu_pre, nu_post, coarse_sweeps;
  double omega;
  int spd_mode;  /* M^{-1} per outer step: MLSQR_SPD_VCYCLE (mg_* fields), MLSQR_SPD_CHOLESKY or
                    MLSQR_SPD_INNER_CG (SpdSolverMode, spdsolve.hpp:35-38; outer.cpp:64-70) */
  int k_inner;   /* inner-CG iteration count */
} mlsqr_outer_cfg;
#define MLSQR_SPD_VCYCLE 0
#define MLSQR_SPD_CHOLESKY 1
#define MLSQR_SPD_INNER_CG 2

typedef struct {            /* OuterStep (outer.hpp:33-41) */
  int k;
  int inner_iterations;
  int inner_stop;
  double penalty_value;
  double final_residual;
  double eps_used;
} mlsqr_outer_step;

/* solve_nonlinear (outer.hpp:61-62, outer.cpp:40-100).  steps: max_outer; alphas/betas
 * optional host blocks (max_outer x (inner_cap+1) / (inner_cap+2)). */
int mlsqr_nonlinear_solve(mlsqr_op* op, const double* g, int dims, size_t nx, size_t ny,
                          size_t nz, double h, const mlsqr_outer_cfg* cfg, double* f_out,
                          mlsqr_outer_step* steps, int* n_steps, int* stop_reason,
                          int* triggered_at, double* alphas, double* betas, int ptr_kind);

/* Stateful driver for one outer step at a time (outer.cpp:59-87): D update at f_prev,
 * hierarchy + auto shift, mlsqr from zero (capped at inner_cap), R(f^k).  Keeps the
 * V-cycle and the Krylov workspace resident between steps (bench / serving loop).
 * With MLSQR_HOST buffers (pinned memory copies at full PCIe speed) f_prev is copied first,
 * g follows on the context's side stream while the hierarchy is built, and f_out returns
 * on the side stream as soon as the solve ends, next to R(f); the call still returns only
 * after every copy has completed. */
typedef struct mlsqr_outer mlsqr_outer;
int mlsqr_outer_create(mlsqr_op* op, int dims, size_t nx, size_t ny, size_t nz, double h,
                       const mlsqr_outer_cfg* cfg, mlsqr_outer** out);
int mlsqr_outer_advance(mlsqr_outer* o, const double* g, const double* f_prev, double* f_out,
                     mlsqr_outer_step* step, int ptr_kind);
/* the bidiagonalization of the last advanced step (BidiagEntries, krylov.hpp:62-67): alpha_1..,
 * beta_1.. into host buffers of capacity cap_a / cap_b (NULL: count only) */
int mlsqr_outer_last_bidiag(mlsqr_outer* o, double* alphas, size_t cap_a, double* betas, size_t cap_b,
                            int* n_alphas, int* n_betas);
int mlsqr_outer_destroy(mlsqr_outer* o);

/* ---- R(f) (diffusion.cpp:89-101) on the device --------------------------- */
int mlsqr_penalty_functional(mlsqr_ctx* ctx, int dims, size_t nx, size_t ny, size_t nz,
                             double h, const double* f, int ptr_kind, int pen_kind, double T,
                             double* value);

/* ---- seeded synthetic inputs (host; problems.cpp conventions) ------------ */
int mlsqr_taps(size_t n, double sigma_f, double domain_length, int radius, double* taps,
               int* radius_out);
int mlsqr_gauss_fill(uint64_t seed, size_t n, double stddev, double* out);
int mlsqr_phantom_rects2d(size_t nx, size_t ny, int count, uint64_t seed, double* out);
int mlsqr_phantom_shapes2d(size_t nx, size_t ny, int count, uint64_t seed, double* out);
int mlsqr_phantom_ellipsoids3d(size_t nx, size_t ny, size_t nz, int count, double semi_lo,
                               double semi_hi, double vlo, double vhi, uint64_t seed,
                               double* out);
int mlsqr_fdot_tables(size_t n, int n_src, int n_det, double mu, uint64_t seed, double* gs,
                      double* gd);

#ifdef __cplusplus
}
#endif
#endif
