// internal.cuh -- shared device helpers and host-side object model of the
// B200-native MLSQR path.  See DESIGN.md for the data layout and the
// "canonical arithmetic order" every kernel here implements (bit-exact with
// the oracle's DEVICE order).  Compiled with -fmad=false: no mul+add pair is
// ever contracted, exactly like the reference's scalar backend.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mlsqr_b200.h"

namespace mlsqr_b200 {

// ---------------------------------------------------------------------------
// errors: C++ exceptions inside the library, status codes at the C-ABI
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  int iteration;
  Error(int c, const std::string& m, int it = 0) : std::runtime_error(m), code(c), iteration(it) {}
};

#define MLSQR_CUDA(call)                                                                  \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::mlsqr_b200::Error(MLSQR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

inline void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw Error(code, msg);
}

// ---------------------------------------------------------------------------
// canonical reductions: segments of 32 consecutive row elements
// reduced by the shuffle-down tree; then tree-32 levels over partials.
// ---------------------------------------------------------------------------
constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// lane 0 receives v[0]+v[16] ... : the canonical tree32
__device__ __forceinline__ double tree32(double v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_down_sync(kFull, v, off);
  return v;
}

// serial emulation of tree32 over 32 values held by one thread
__device__ __forceinline__ double tree32_serial(double* v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
    for (int l = 0; l < off; ++l) v[l] = v[l] + v[l + off];
  return v[0];
}

// vector layout for reductions: `rows` rows of `len` elements, row-major
// gridDim.y for the (32, 8)-block row kernels: one block row per 8 rows, capped at CUDA's
// 65535 limit (those kernels loop over rows with a gridDim.y stride)
inline unsigned row_grid(size_t rows) {
  const size_t g = (rows + 7) / 8;
  return (unsigned)(g < 65535 ? (g ? g : 1) : 65535);
}

struct RowShape {
  size_t len;   // elements per row (x extent)
  size_t rows;  // number of rows (ny * nz)
  size_t chunks() const { return (len + 31) / 32; }
  size_t segments() const { return chunks() * rows; }
  size_t n() const { return len * rows; }
};

// deterministic hypot from IEEE basic operations (oracle orc_dhypot)
__host__ __device__ inline double dhypot(double a, double b) {
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

// penalty.cpp:60-84 with the device hypot
__host__ __device__ inline double diffusivity(int kind, double T, double t) {
  double c = 1.0;
  switch (kind) {
    case MLSQR_PEN_TIKHONOV: return 1.0;
    case MLSQR_PEN_TV: c = 1.0 / dhypot(T, t); break;
    case MLSQR_PEN_PM_LOG: {
      const double u = t / T;
      c = u > 1e8 ? (T / t) * (T / t) : 1.0 / (1.0 + u * u);
      break;
    }
    case MLSQR_PEN_PM_EXP: {
      const double u = t / T;
      c = exp(-u * u);
      break;
    }
  }
  const double dmin = 2.2250738585072014e-308;  // DBL_MIN (penalty.cpp:83)
  return c > dmin ? c : dmin;
}

// penalty.cpp:35-53
__host__ __device__ inline double r_value(int kind, double T, double t) {
  switch (kind) {
    case MLSQR_PEN_TIKHONOV: return 0.5 * t * t;
    case MLSQR_PEN_TV: return dhypot(T, t);
    case MLSQR_PEN_PM_LOG: {
      const double u = t / T;
      return 0.5 * T * T * log1p(u * u);
    }
    case MLSQR_PEN_PM_EXP: {
      const double u = t / T;
      return 0.5 * T * T * (1.0 - exp(-u * u));
    }
  }
  return 0.0;
}

// ---------------------------------------------------------------------------
// host object model
// ---------------------------------------------------------------------------
struct Ctx;

// Fused epilogue of an operator application:
//   out = A (x * sx)  [+ coef * (old * so)],  seg <- canonical segment partials of out^2
// All scalars are DEVICE pointers (the iteration never syncs with the host); a null
// pointer means "1" for sx/so and "no term" for old.  gate: skip when *gate == 0.
struct Epi {
  const double* sx = nullptr;
  const double* old = nullptr;
  const double* so = nullptr;
  const double* coef = nullptr;
  double* seg = nullptr;
  const int* gate = nullptr;
  bool in_guarded = false;  // the input carries halo_planes_needed() zero/ghost planes per side
  bool ghosts_ready = false; // (z-sharded) the caller already filled the input's ghost planes
};

class Op {
 public:
  virtual ~Op() = default;
  Ctx* ctx = nullptr;
  size_t rows = 0, cols = 0;
  RowShape data_shape{}, sol_shape{};
  // ghost planes the operator needs on its input when z-sharded (0: none)
  virtual int halo_planes_needed() const { return 0; }
  virtual size_t plane_size() const { return 0; }
  virtual void apply(const double* x, double* y, const Epi& e) = 0;
  virtual void adjoint(const double* y, double* x, const Epi& e) = 0;
  virtual int tclass() const { return MLSQR_TCLASS_BLUR; }
};

class Pc {
 public:
  virtual ~Pc() = default;
  Ctx* ctx = nullptr;
  size_t n = 0;
  // (z-sharded) the caller's input p carries at least one writable guard plane per side, so the
  // map may fill ghost planes of p in place (the Krylov workspace's guarded p does)
  bool in_guarded = false;
  // v = B p on the device; seg (optional) <- segment partials of v*p laid out over
  // `shape` (the operator's solution space); gate as in Epi
  virtual void solve(const double* p, double* v, double* seg, const int* gate, RowShape shape) = 0;
  virtual bool host_callback() const { return false; }
  // row length the map's reduction partials are laid out with (0: follows the caller)
  virtual size_t row_len() const { return 0; }
};

// communicator of the z-slab decomposition (comm.cu)
class Comm {
 public:
  virtual ~Comm() = default;
  int rank = 0, size = 1;
  virtual bool capturable() const = 0;
  // recv_lo <- (rank-1).send_hi ; recv_hi <- (rank+1).send_lo ; missing neighbours: untouched
  virtual void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi,
                    size_t count, cudaStream_t s) = 0;
  // recv[k*count .. (k+1)*count) <- rank k's send
  virtual void allgather(const double* send, size_t count, double* recv, cudaStream_t s) = 0;
  virtual void allreduce_max_u64(unsigned long long* buf, cudaStream_t s) = 0;
};
struct LoopGroup;
Comm* make_nccl_comm(const void* uid, int rank, int size);
int nccl_unique_id(void* out128);
LoopGroup* make_loop_group(int p);
void free_loop_group(LoopGroup* g);
Comm* make_loop_comm(LoopGroup* g, int rank);

struct Ctx {
  int device = 0;
  // z-slab decomposition: grids built on this context with z extent nz are the planes
  // [zoff, zoff + nz) of a global grid with nzg planes (nzg == 0: not sharded)
  Comm* comm = nullptr;
  long zoff = 0, nzg = 0;
  // side stream + fork/join events for exchanges overlapped with main-stream work
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;    // the Krylov loop's vtilde exchange
  cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;  // an operator's own input exchange
  cudaEvent_t ev_copy = nullptr, ev_copy2 = nullptr;   // HOST-buffer copies overlapped with main-stream work
  cudaStream_t side_stream() {
    if (!side) {
      MLSQR_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      MLSQR_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      MLSQR_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
      MLSQR_CUDA(cudaEventCreateWithFlags(&ev_fork2, cudaEventDisableTiming));
      MLSQR_CUDA(cudaEventCreateWithFlags(&ev_join2, cudaEventDisableTiming));
      MLSQR_CUDA(cudaEventCreateWithFlags(&ev_copy, cudaEventDisableTiming));
      MLSQR_CUDA(cudaEventCreateWithFlags(&ev_copy2, cudaEventDisableTiming));
    }
    return side;
  }
  void release_side() {
    if (side) {
      cudaStreamDestroy(side);
      cudaEventDestroy(ev_fork);
      cudaEventDestroy(ev_join);
      cudaEventDestroy(ev_fork2);
      cudaEventDestroy(ev_join2);
      cudaEventDestroy(ev_copy);
      cudaEventDestroy(ev_copy2);
      side = nullptr;
    }
  }
  // row-shard decomposition (dense operators): data-space vectors hold the rows
  // [row0, row0 + rows_g / P) of a global data space with rows_g rows; the solution space and any
  // preconditioner are replicated (so sharded() -- the z-slab predicate -- is false)
  bool row_mode = false;
  long row0 = 0, rows_g = 0;
  // an explicit mlsqr_ctx_set_slab / _set_row_shard runs the decomposed code path even on a
  // one-rank communicator (ghost exchanges with no neighbours, one-rank collectives): that is
  // how the NCCL transport and the sharded graph are exercised on a single GPU
  bool decomposed = false;
  bool multi() const { return comm != nullptr && (comm->size > 1 || decomposed); }
  bool sharded() const { return multi() && !row_mode; }
  bool row_sharded() const { return multi() && row_mode; }
  // data-space reductions span ranks in both decompositions
  bool data_distributed() const { return multi(); }
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint64_t launches = 0;
  bool timing = false;
  double t_ms[MLSQR_TCLASS_COUNT] = {};
  uint64_t t_n[MLSQR_TCLASS_COUNT] = {};
  int sm_count = 148;
  size_t l2_bytes = 0;
  // grow-only staging buffers for HOST-pointer calls (no cudaMalloc/cudaFree per call)
  void* stage[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t stage_bytes[4] = {0, 0, 0, 0};
  int stage_next = 0;
  void* staging(size_t bytes) {
    const int k = stage_next;
    stage_next = (stage_next + 1) & 3;
    if (stage_bytes[k] < bytes) {
      if (stage[k]) cudaFree(stage[k]);
      stage[k] = nullptr;
      stage_bytes[k] = 0;
      if (cudaMalloc(&stage[k], bytes) != cudaSuccess)
        throw Error(MLSQR_ECUDA, "staging allocation failed");
      stage_bytes[k] = bytes;
    }
    return stage[k];
  }
  void release_staging() {
    for (int k = 0; k < 4; ++k)
      if (stage[k]) cudaFree(stage[k]);
    if (ws_cache) ws_free(ws_cache);
    ws_cache = nullptr;
  }
  // last Krylov workspace, reused by repeated solves of the same shape
  void* ws_cache = nullptr;
  void (*ws_free)(void*) = nullptr;

  void count(int k = 1) { launches += (uint64_t)k; }
  void check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(MLSQR_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  }
};

// scoped timing of one kernel class (CUDA events on the context stream)
class TimedRegion {
 public:
  TimedRegion(Ctx* c, int cls, cudaStream_t s = nullptr) : c_(c), cls_(cls), s_(s ? s : c->stream) {
    if (!c_->timing || cls_ < 0) return;
    cudaEventCreate(&a_);
    cudaEventCreate(&b_);
    cudaEventRecord(a_, s_);
  }
  ~TimedRegion() {
    if (!c_->timing || cls_ < 0) return;
    cudaEventRecord(b_, s_);
    pending().push_back({a_, b_, cls_});
  }
  struct Pending {
    cudaEvent_t a, b;
    int cls;
  };
  static std::vector<Pending>& pending() {
    static thread_local std::vector<Pending> p;
    return p;
  }
  static void collect(Ctx* c) {
    auto& p = pending();
    if (p.empty()) return;
    for (auto& e : p) {
      float ms = 0.f;
      cudaEventSynchronize(e.b);  // (regions may sit on the side stream too)
      cudaEventElapsedTime(&ms, e.a, e.b);
      c->t_ms[e.cls] += ms;
      c->t_n[e.cls] += 1;
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    p.clear();
  }

 private:
  Ctx* c_;
  int cls_;
  cudaStream_t s_;
  cudaEvent_t a_{}, b_{};
};

// device buffer (RAII)
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  void alloc(size_t count) {
    release();
    if (count) MLSQR_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
};

// ---------------------------------------------------------------------------
// kernels shared across translation units (defined in reduce.cu / vec.cu)
// ---------------------------------------------------------------------------
// canonical reduction of `nseg` segment partials -> out (device scalar)
void reduce_segments(Ctx* c, const double* seg, size_t nseg, double* scratch, double* out,
                     const int* gate);
size_t reduce_scratch_size(size_t nseg);
// all passes but the last: returns the <= 1024 partials left (count in *J_out) for a final
// one-warp pass that the caller may fuse with its scalar epilogue (vec.cuh reduce_final_fin)
const double* reduce_segments_to_warp(Ctx* c, const double* seg, size_t nseg, double* scratch, const int* gate,
                                      size_t* J_out);
// segment partials of (x .* y) over a row shape (both unscaled)
void seg_dot(Ctx* c, const double* x, const double* y, RowShape s, double* seg, const int* gate);
// out = x * sx + coef * (old * so) elementwise (identity operator / copies), with seg of out^2
void axpby_epi(Ctx* c, const double* x, double* out, RowShape s, const Epi& e);
// z-slab halo: fill k ghost planes below/above a guarded local vector from the neighbours
void halo_planes(Ctx* c, double* v, size_t plane, long nz_loc, int k);
void halo_planes(Ctx* c, double* v, size_t plane, long nz_loc, int k, cudaStream_t s);
// canonical reduction of this rank's segments of a z-sharded vector: bit-identical to the
// unsharded reduction (block-aligned tree partials or raw segments are allgathered)
// dist: the segments are this rank's share of a distributed vector (else: a local / replicated one)
void reduce_segments_dist(Ctx* c, const double* seg, size_t nseg, double* scratch, double* gathered,
                          double* out, const int* gate, bool dist);
void reduce_segments_dist(Ctx* c, const double* seg, size_t nseg, double* scratch, double* gathered,
                          double* out, const int* gate);
// the distributed reductions' first half: this rank's block-aligned level-3 partials (or its raw
// segments), allgathered in rank order; returns the gathered list and its length
const double* dist_gather_partials(Ctx* c, const double* seg, size_t nseg, double* scratch, double* gathered,
                                   const int* gate, size_t* count);
// scratch sizes of reduce_segments_dist
size_t dist_gather_size(Ctx* c, size_t nseg);

// ---------------------------------------------------------------------------
// operator / map factories (blur.cu, dense.cu, vcycle.cu)
// ---------------------------------------------------------------------------
Op* make_blur(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, const double* taps, int radius);
Op* make_blur2d_axes(Ctx* c, size_t nx, size_t ny, const double* tx, int rx, const double* ty, int ry);
Op* make_dense(Ctx* c, size_t rows, size_t cols, const double* a, bool a_on_device,
               size_t sol_row_len);
Op* make_dense_fdot(Ctx* c, size_t nvox, int nsrc, int ndet, const double* gs, const double* gd,
                    size_t sol_row_len);
Op* make_identity(Ctx* c, size_t n, size_t row_len);

class VCycle;
Pc* make_identity_map(Ctx* c, size_t n);
VCycle* make_vcycle(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, double h, int levels,
                    int nu_pre, int nu_post, double omega, int coarse_sweeps);
void vcycle_set_coefficients(VCycle* v, const double* cx, const double* cy, const double* cz,
                             double eps);  // device pointers
double vcycle_update(VCycle* v, const double* f_dev, int pen_kind, double T, double eps);
void vcycle_m_apply(VCycle* v, const double* x, double* y);
void vcycle_update_async(VCycle* v, const double* f_dev, int pen_kind, double T, double eps);
const double* vcycle_eps_dev(VCycle* v);
Pc* vcycle_as_pc(VCycle* v);
size_t vcycle_sol_len(VCycle* v);
void penalty_functional_async(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, double h,
                              const double* f, int kind, double T, double* seg, double* scratch,
                              double* gathered, double* fguard, double* out);
Pc* make_callback_map(Ctx* c, size_t n, mlsqr_host_map_fn fn, void* user);
// SpdSolver::factorize / inner_cg over the level-0 M (+ shift) of a V-cycle map (spdmaps.cu)
Pc* make_chol_map(VCycle* src, long long* pivot_row);
Pc* make_inner_cg_map(VCycle* src, int k_inner);
double penalty_functional_dev(Ctx* c, int dims, size_t nx, size_t ny, size_t nz, double h,
                              const double* f, int pen_kind, double T);

// solvers (lsqr.cu)
struct Workspace;  // per-solve device buffers, reusable across outer steps
Workspace* workspace_new(Ctx* c, size_t rows, size_t cols, RowShape data, RowShape sol,
                         int max_iters, size_t guard = 0);
// guard elements per side the Krylov vectors need for an operator's ghost planes
inline size_t op_guard(const Op* o) {
  const int k = o->halo_planes_needed();
  return k > 0 ? (size_t)k * o->plane_size() + 64 : 0;
}
void workspace_free(Workspace* w);
// Runs mlsqr (or lsqr when pc == nullptr) fully on the device.  Outputs to host arrays
// when non-null.  `sync_out`: copy results back and return status; when false the solve
// stays queued (outer loop) and results must be fetched with solve_fetch().
int solve_mlsqr(Op* op, Pc* pc, const double* g_dev, double tau, const mlsqr_stop& stop,
                double* f_dev, mlsqr_iter_rec* trace, double* alphas, double* betas,
                mlsqr_solve_info* info, Workspace* ws = nullptr, bool use_graph = true,
                double* basis_dev = nullptr, double* left_dev = nullptr, double* snap_dev = nullptr);
// solve_projected (krylov.cpp:631-678), host arithmetic (projected.cu)
std::vector<double> solve_projected(const double* alphas, size_t k, const double* betas, size_t nb,
                                    double beta1, double tau);
void reconstruct_from_basis(Ctx* c, const double* basis, size_t n, const double* y, size_t ny, double* f);
void validate_stop(const mlsqr_stop& s);
// cg_normal (krylov.cpp:551-628) on the device; M = the V-cycle's level-0 operator (cgn.cu)
void solve_cg_normal(Op* op, VCycle* m, const double* g, double tau, const mlsqr_stop& stop,
                     double* f_dev, mlsqr_iter_rec* trace, mlsqr_solve_info* info,
                     double* snap_dev = nullptr);
// krylov_basis (krylov.cpp:700-754) on the device (basis.cu); returns the vector count
int krylov_basis(Op* op, Pc* msolver, VCycle* m, double tau, const double* g, int k, double* vecs,
                 int* rank_exhausted);
// stateful outer step (outer.cu)
class OuterSolver {
 public:
  OuterSolver(Op* o, int dims, size_t nx, size_t ny, size_t nz, double h, const mlsqr_outer_cfg& cfg);
  ~OuterSolver();
  OuterSolver(const OuterSolver&) = delete;
  OuterSolver& operator=(const OuterSolver&) = delete;
  void step(const double* g, const double* f_prev, double* f_out, mlsqr_outer_step* st, int k);
  // HOST-buffer calls (mlsqr_outer_advance): g may still be on its way on the side stream while
  // the hierarchy is built from f_prev (g_ready, waited for before the solve), and f_out goes
  // back to out_host on the side stream as soon as the solve is done, next to R(f)
  cudaEvent_t g_ready = nullptr;
  double* out_host = nullptr;
  Op* op;
  mlsqr_solve_info last_info{};
  std::vector<double> al_, be_;

 private:
  int dims_;
  size_t nx_, ny_, nz_;
  double h_;
  mlsqr_outer_cfg cfg_;
  mlsqr_stop inner_{};
  VCycle* vc_ = nullptr;
  Workspace* ws_ = nullptr;
  DevBuf<double> pseg_, pscr_, pval_, pgat_, pfg_;
  std::vector<mlsqr_iter_rec> trace_;
};

// solve_nonlinear (outer.cu)
void nonlinear_solve(Op* o, const double* g_dev, int dims, size_t nx, size_t ny, size_t nz,
                     double h, const mlsqr_outer_cfg& cfg, double* f_dev, mlsqr_outer_step* steps,
                     int* n_steps, int* stop_reason, int* triggered_at, double* alphas,
                     double* betas);

}  // namespace mlsqr_b200

struct mlsqr_ctx {
  mlsqr_b200::Ctx impl;
};
struct mlsqr_op {
  mlsqr_b200::Op* impl;
};
struct mlsqr_pc {
  mlsqr_b200::Pc* impl;
  mlsqr_b200::VCycle* vc;  // non-null for V-cycle maps
};
