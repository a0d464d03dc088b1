// capi.cu -- the extern "C" boundary (include/mlsqr_b200.h).  Every entry
// point converts C++ exceptions into status codes + a thread-local message,
// validates lengths like LinearOperator::apply (linop.cpp:15-40), and moves
// host buffers in/out when ptr_kind == MLSQR_HOST.
#include <cstring>
#include <memory>

#include "internal.cuh"

using namespace mlsqr_b200;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& fn) {
  try {
    g_err.clear();
    fn();
    return MLSQR_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return MLSQR_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MLSQR_EINVAL;
  }
}

void check_len(size_t got, size_t want, const char* what) {
  if (got != want)
    throw Error(MLSQR_EDIM, std::string(what) + ": expected length " + std::to_string(want) +
                                ", got " + std::to_string(got));
}

void set_device(Ctx* c) { MLSQR_CUDA(cudaSetDevice(c->device)); }

// stage a host or device input as a device pointer (host data goes through the
// context's grow-only staging buffers: every HOST call completes before returning)
struct In {
  const double* d = nullptr;
  In(Ctx* c, const double* p, size_t n, int kind) {
    if (kind == MLSQR_DEVICE || n == 0) {
      d = p;
      return;
    }
    double* s = static_cast<double*>(c->staging(sizeof(double) * n));
    MLSQR_CUDA(cudaMemcpyAsync(s, p, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    d = s;
  }
};

struct Out {
  double* d = nullptr;
  double* host = nullptr;
  size_t n;
  Ctx* c;
  Out(Ctx* cc, double* p, size_t nn, int kind) : n(nn), c(cc) {
    if (kind == MLSQR_DEVICE) {
      d = p;
      return;
    }
    host = p;
    d = static_cast<double*>(c->staging(sizeof(double) * n));
  }
  void finish() {
    if (host) MLSQR_CUDA(cudaMemcpyAsync(host, d, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    MLSQR_CUDA(cudaStreamSynchronize(c->stream));
  }
};

}  // namespace

// ---------------------------------------------------------------------------
// host plug-in SpdMap (spdsolve.hpp:15-22 implemented by the caller)
// ---------------------------------------------------------------------------
namespace mlsqr_b200 {
class CallbackMap final : public Pc {
 public:
  CallbackMap(Ctx* c, size_t nn, mlsqr_host_map_fn fn, void* user) : fn_(fn), user_(user) {
    ctx = c;
    n = nn;
    hp_.resize(n);
    hv_.resize(n);
  }
  bool host_callback() const override { return true; }
  void solve(const double* p, double* v, double* seg, const int* gate, RowShape shape) override {
    int on = 1;
    if (gate) MLSQR_CUDA(cudaMemcpyAsync(&on, gate, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    MLSQR_CUDA(cudaMemcpyAsync(hp_.data(), p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    MLSQR_CUDA(cudaStreamSynchronize(ctx->stream));
    if (!on) return;
    if (fn_(user_, hp_.data(), hv_.data()) != 0) throw Error(MLSQR_ECALLBACK, "host SpdMap callback failed");
    MLSQR_CUDA(cudaMemcpyAsync(v, hv_.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    if (seg) seg_dot(ctx, v, p, shape, seg, gate);
  }

 private:
  mlsqr_host_map_fn fn_;
  void* user_;
  std::vector<double> hp_, hv_;
};
Pc* make_callback_map(Ctx* c, size_t n, mlsqr_host_map_fn fn, void* user) {
  return new CallbackMap(c, n, fn, user);
}
}  // namespace mlsqr_b200

extern "C" {

const char* mlsqr_last_error(void) { return g_err.c_str(); }

const char* mlsqr_version(void) { return "mlsqr_b200 0.1 sm_100a fp64 canonical-order"; }

int mlsqr_ctx_create(int device, void* stream, mlsqr_ctx** out) {
  return guard([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      throw Error(MLSQR_ECUDA, "no CUDA device visible: the B200 path has no CPU fallback");
    require(device >= 0 && device < n, MLSQR_EINVAL, "device index out of range");
    auto* c = new mlsqr_ctx();
    c->impl.device = device;
    MLSQR_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    MLSQR_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
      delete c;
      throw Error(MLSQR_ECUDA, std::string("device ") + prop.name + " is not sm_100-class (this build targets sm_100a)");
    }
    c->impl.sm_count = prop.multiProcessorCount;
    c->impl.l2_bytes = (size_t)prop.l2CacheSize;
    if (stream) {
      c->impl.stream = (cudaStream_t)stream;
    } else {
      MLSQR_CUDA(cudaStreamCreateWithFlags(&c->impl.stream, cudaStreamNonBlocking));
      c->impl.own_stream = true;
    }
    *out = c;
  });
}

int mlsqr_ctx_destroy(mlsqr_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->impl.device);
    cudaStreamSynchronize(ctx->impl.stream);
    ctx->impl.release_staging();
    if (ctx->impl.side) cudaStreamSynchronize(ctx->impl.side);
    ctx->impl.release_side();
    delete ctx->impl.comm;
    ctx->impl.comm = nullptr;
    if (ctx->impl.own_stream) cudaStreamDestroy(ctx->impl.stream);
    delete ctx;
  });
}

int mlsqr_ctx_synchronize(mlsqr_ctx* ctx) {
  return guard([&] { MLSQR_CUDA(cudaStreamSynchronize(ctx->impl.stream)); });
}

int mlsqr_dev_alloc(mlsqr_ctx* ctx, size_t bytes, void** ptr) {
  return guard([&] {
    set_device(&ctx->impl);
    MLSQR_CUDA(cudaMalloc(ptr, bytes));
  });
}

int mlsqr_dev_free(mlsqr_ctx* ctx, void* ptr) {
  return guard([&] {
    set_device(&ctx->impl);
    MLSQR_CUDA(cudaFree(ptr));
  });
}

int mlsqr_copy(mlsqr_ctx* ctx, void* dst, int dk, const void* src, int sk, size_t bytes) {
  return guard([&] {
    set_device(&ctx->impl);
    cudaMemcpyKind k = dk == MLSQR_DEVICE ? (sk == MLSQR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice)
                                          : (sk == MLSQR_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost);
    MLSQR_CUDA(cudaMemcpyAsync(dst, src, bytes, k, ctx->impl.stream));
    MLSQR_CUDA(cudaStreamSynchronize(ctx->impl.stream));
  });
}

uint64_t mlsqr_ctx_launch_count(mlsqr_ctx* ctx, int reset) {
  const uint64_t n = ctx->impl.launches;
  if (reset) ctx->impl.launches = 0;
  return n;
}

int mlsqr_ctx_set_timing(mlsqr_ctx* ctx, int enable) {
  return guard([&] {
    ctx->impl.timing = enable != 0;
    for (int i = 0; i < MLSQR_TCLASS_COUNT; ++i) {
      ctx->impl.t_ms[i] = 0.0;
      ctx->impl.t_n[i] = 0;
    }
  });
}

int mlsqr_ctx_get_timing(mlsqr_ctx* ctx, int cls, double* ms, uint64_t* launches) {
  return guard([&] {
    require(cls >= 0 && cls < MLSQR_TCLASS_COUNT, MLSQR_EINVAL, "bad timing class");
    TimedRegion::collect(&ctx->impl);
    *ms = ctx->impl.t_ms[cls];
    *launches = ctx->impl.t_n[cls];
  });
}

// ---- z-slab decomposition ----
int mlsqr_nccl_unique_id(void* out, size_t cap, size_t* len) {
  return guard([&] {
    require(cap >= 128, MLSQR_EINVAL, "unique id buffer must hold 128 bytes");
    const int n = nccl_unique_id(out);
    if (len) *len = (size_t)n;
  });
}

int mlsqr_ctx_set_comm_nccl(mlsqr_ctx* ctx, const void* uid, int rank, int size) {
  return guard([&] {
    set_device(&ctx->impl);
    require(size >= 1 && rank >= 0 && rank < size, MLSQR_EINVAL, "bad rank / size");
    delete ctx->impl.comm;
    ctx->impl.comm = nullptr;
    ctx->impl.comm = make_nccl_comm(uid, rank, size);
  });
}

int mlsqr_loop_group_create(int size, void** group) {
  return guard([&] {
    require(size >= 1, MLSQR_EINVAL, "group size must be >= 1");
    *group = make_loop_group(size);
  });
}

int mlsqr_loop_group_destroy(void* group) {
  return guard([&] { free_loop_group(static_cast<LoopGroup*>(group)); });
}

int mlsqr_ctx_set_comm_loopback(mlsqr_ctx* ctx, void* group, int rank) {
  return guard([&] {
    delete ctx->impl.comm;
    ctx->impl.comm = nullptr;
    ctx->impl.comm = make_loop_comm(static_cast<LoopGroup*>(group), rank);
  });
}

int mlsqr_ctx_set_slab(mlsqr_ctx* ctx, size_t nz_global, size_t z_offset) {
  return guard([&] {
    require(z_offset < nz_global, MLSQR_EINVAL, "slab offset outside the global grid");
    ctx->impl.row_mode = false;
    ctx->impl.decomposed = true;
    ctx->impl.nzg = (long)nz_global;
    ctx->impl.zoff = (long)z_offset;
  });
}

int mlsqr_ctx_set_row_shard(mlsqr_ctx* ctx, size_t rows_global, size_t row_offset) {
  return guard([&] {
    require(row_offset < rows_global, MLSQR_EINVAL, "row shard offset outside the data space");
    ctx->impl.row_mode = true;
    ctx->impl.decomposed = true;
    ctx->impl.rows_g = (long)rows_global;
    ctx->impl.row0 = (long)row_offset;
  });
}

// ---- operators ----
int mlsqr_blur2d_create_axes(mlsqr_ctx* ctx, size_t nx, size_t ny, const double* tx, int rx, const double* ty,
                             int ry, mlsqr_op** out) {
  return guard([&] {
    require(ctx && tx && ty && out, MLSQR_EINVAL, "blur2d_create_axes: null argument");
    set_device(&ctx->impl);
    *out = new mlsqr_op{make_blur2d_axes(&ctx->impl, nx, ny, tx, rx, ty, ry)};
  });
}

int mlsqr_blur_create(mlsqr_ctx* ctx, int dims, size_t nx, size_t ny, size_t nz,
                      const double* taps, int radius, mlsqr_op** out) {
  return guard([&] {
    set_device(&ctx->impl);
    require(taps != nullptr, MLSQR_EINVAL, "taps must not be null");
    require(!ctx->impl.row_sharded(), MLSQR_EINVAL, "a blur is z-sharded, not row-sharded (mlsqr_ctx_set_slab)");
    *out = new mlsqr_op{make_blur(&ctx->impl, dims, nx, ny, nz, taps, radius)};
  });
}

int mlsqr_dense_create(mlsqr_ctx* ctx, size_t rows, size_t cols, const double* a, int a_kind,
                       size_t sol_row_len, mlsqr_op** out) {
  return guard([&] {
    set_device(&ctx->impl);
    require(!ctx->impl.sharded(), MLSQR_EINVAL, "dense operators are row-sharded, not z-sharded (mlsqr_ctx_set_row_shard)");
    *out = new mlsqr_op{make_dense(&ctx->impl, rows, cols, a, a_kind == MLSQR_DEVICE, sol_row_len)};
  });
}

int mlsqr_dense_create_fdot(mlsqr_ctx* ctx, size_t n_vox, int n_src, int n_det, const double* gs,
                            const double* gd, size_t sol_row_len, mlsqr_op** out) {
  return guard([&] {
    set_device(&ctx->impl);
    require(n_src >= 1 && n_det >= 1 && n_vox >= 1, MLSQR_EDIM, "fDOT operator needs sources, detectors and voxels");
    *out = new mlsqr_op{make_dense_fdot(&ctx->impl, n_vox, n_src, n_det, gs, gd, sol_row_len)};
  });
}

int mlsqr_identity_create(mlsqr_ctx* ctx, size_t n, size_t row_len, mlsqr_op** out) {
  return guard([&] {
    set_device(&ctx->impl);
    *out = new mlsqr_op{make_identity(&ctx->impl, n, row_len)};
  });
}

int mlsqr_op_destroy(mlsqr_op* op) {
  return guard([&] {
    if (!op) return;
    delete op->impl;
    delete op;
  });
}

int mlsqr_op_shape(const mlsqr_op* op, size_t* rows, size_t* cols) {
  return guard([&] {
    *rows = op->impl->rows;
    *cols = op->impl->cols;
  });
}

int mlsqr_op_apply(mlsqr_op* op, const double* x, size_t x_len, double* y, size_t y_len, int kind) {
  return guard([&] {
    Op* o = op->impl;
    Ctx* c = o->ctx;
    set_device(c);
    check_len(x_len, o->cols, "apply input");
    check_len(y_len, o->rows, "apply output");
    In in(c, x, x_len, kind);
    Out out(c, y, y_len, kind);
    o->apply(in.d, out.d, Epi{});
    out.finish();
    TimedRegion::collect(c);
  });
}

int mlsqr_op_apply_adjoint(mlsqr_op* op, const double* y, size_t y_len, double* x, size_t x_len,
                           int kind) {
  return guard([&] {
    Op* o = op->impl;
    Ctx* c = o->ctx;
    set_device(c);
    check_len(y_len, o->rows, "apply_adjoint input");
    check_len(x_len, o->cols, "apply_adjoint output");
    In in(c, y, y_len, kind);
    Out out(c, x, x_len, kind);
    o->adjoint(in.d, out.d, Epi{});
    out.finish();
    TimedRegion::collect(c);
  });
}

// ---- maps ----
int mlsqr_identity_map_create(mlsqr_ctx* ctx, size_t n, mlsqr_pc** out) {
  return guard([&] {
    set_device(&ctx->impl);
    require(n >= 1, MLSQR_EDIM, "map dimension must be at least 1");
    *out = new mlsqr_pc{make_identity_map(&ctx->impl, n), nullptr};
  });
}

int mlsqr_vcycle_create(mlsqr_ctx* ctx, int dims, size_t nx, size_t ny, size_t nz, double h,
                        int levels, int nu_pre, int nu_post, double omega, int coarse_sweeps,
                        mlsqr_pc** out) {
  return guard([&] {
    set_device(&ctx->impl);
    VCycle* v = make_vcycle(&ctx->impl, dims, nx, ny, nz, h, levels, nu_pre, nu_post, omega, coarse_sweeps);
    *out = new mlsqr_pc{vcycle_as_pc(v), v};
  });
}

int mlsqr_chol_map_create(mlsqr_pc* m, mlsqr_pc** out, long long* pivot_row) {
  if (pivot_row) *pivot_row = -1;
  return guard([&] {
    require(m && m->vc && out, MLSQR_EINVAL, "the Cholesky map is built from the M of a V-cycle map");
    set_device(m->impl->ctx);
    *out = new mlsqr_pc{make_chol_map(m->vc, pivot_row), nullptr};
  });
}

int mlsqr_inner_cg_map_create(mlsqr_pc* m, int k_inner, mlsqr_pc** out) {
  return guard([&] {
    require(m && m->vc && out, MLSQR_EINVAL, "the inner-CG map is built from the M of a V-cycle map");
    set_device(m->impl->ctx);
    *out = new mlsqr_pc{make_inner_cg_map(m->vc, k_inner), nullptr};
  });
}

int mlsqr_vcycle_set_coefficients(mlsqr_pc* pc, const double* cx, const double* cy,
                                  const double* cz, double eps, int kind) {
  return guard([&] {
    require(pc && pc->vc, MLSQR_EINVAL, "not a V-cycle map");
    Ctx* c = pc->impl->ctx;
    set_device(c);
    require(eps >= 0.0, MLSQR_EINVAL, "diagonal shift must be nonnegative");
    const size_t n = pc->impl->n;
    In a(c, cx, n, kind), b(c, cy, cy ? n : 0, kind), d(c, cz, cz ? n : 0, kind);
    vcycle_set_coefficients(pc->vc, a.d, b.d, d.d, eps);
    MLSQR_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int mlsqr_vcycle_update(mlsqr_pc* pc, const double* f, int kind, int pen_kind, double T, double eps,
                        double* eps_used) {
  return guard([&] {
    require(pc && pc->vc, MLSQR_EINVAL, "not a V-cycle map");
    require(pen_kind >= 0 && pen_kind <= 3, MLSQR_EINVAL, "unknown penalty kind");
    require(pen_kind == MLSQR_PEN_TIKHONOV || T > 0.0, MLSQR_EINVAL, "penalty threshold T must be positive");
    Ctx* c = pc->impl->ctx;
    set_device(c);
    In in(c, f, pc->impl->n, kind);
    const double e = vcycle_update(pc->vc, in.d, pen_kind, T, eps);
    if (eps_used) *eps_used = e;
  });
}

int mlsqr_callback_map_create(mlsqr_ctx* ctx, size_t n, mlsqr_host_map_fn fn, void* user,
                              mlsqr_pc** out) {
  return guard([&] {
    set_device(&ctx->impl);
    require(fn != nullptr, MLSQR_EINVAL, "callback must not be null");
    *out = new mlsqr_pc{make_callback_map(&ctx->impl, n, fn, user), nullptr};
  });
}

int mlsqr_pc_destroy(mlsqr_pc* pc) {
  return guard([&] {
    if (!pc) return;
    delete pc->impl;
    delete pc;
  });
}

int mlsqr_pc_dimension(const mlsqr_pc* pc, size_t* n) {
  return guard([&] { *n = pc->impl->n; });
}

int mlsqr_pc_solve(mlsqr_pc* pc, const double* p, double* v, size_t n, int kind) {
  return guard([&] {
    Ctx* c = pc->impl->ctx;
    set_device(c);
    check_len(n, pc->impl->n, "solve");
    In in(c, p, n, kind);
    Out out(c, v, n, kind);
    pc->impl->solve(in.d, out.d, nullptr, nullptr, RowShape{n, 1});
    out.finish();
    TimedRegion::collect(c);
  });
}

int mlsqr_vcycle_m_apply(mlsqr_pc* pc, const double* x, double* y, size_t n, int kind) {
  return guard([&] {
    require(pc && pc->vc, MLSQR_EINVAL, "not a V-cycle map");
    Ctx* c = pc->impl->ctx;
    set_device(c);
    check_len(n, pc->impl->n, "M apply");
    In in(c, x, n, kind);
    Out out(c, y, n, kind);
    vcycle_m_apply(pc->vc, in.d, out.d);
    out.finish();
  });
}

// ---- solvers ----
static int run_solve(mlsqr_op* op, mlsqr_pc* pc, const double* g, double tau, const mlsqr_stop* stop,
                     double* f, mlsqr_iter_rec* trace, double* alphas, double* betas,
                     mlsqr_solve_info* info, int kind, bool plain) {
  int bd_iter = 0;
  if (info) std::memset(info, 0, sizeof(*info));
  const int st = guard([&] {
    require(op && stop, MLSQR_EINVAL, "operator and stopping config are required");
    Op* o = op->impl;
    Ctx* c = o->ctx;
    set_device(c);
    In gin(c, g, o->rows, kind);
    Out fout(c, f, o->cols, kind);
    try {
      solve_mlsqr(o, plain ? nullptr : pc->impl, gin.d, tau, *stop, fout.d, trace, alphas, betas, info);
    } catch (const Error& e) {
      if (e.code == MLSQR_EBREAKDOWN) bd_iter = e.iteration;
      throw;
    }
    fout.finish();
  });
  if (st == MLSQR_EBREAKDOWN && info) info->breakdown_iteration = bd_iter;
  return st;
}

int mlsqr_solve(mlsqr_op* op, mlsqr_pc* pc, const double* g, double tau, const mlsqr_stop* stop,
                double* f, mlsqr_iter_rec* trace, double* alphas, double* betas,
                mlsqr_solve_info* info, int ptr_kind) {
  if (!pc) {
    g_err = "mlsqr needs a preconditioner map (use mlsqr_identity_map_create for M = I)";
    return MLSQR_EINVAL;
  }
  return run_solve(op, pc, g, tau, stop, f, trace, alphas, betas, info, ptr_kind, false);
}

int mlsqr_lsqr_solve(mlsqr_op* op, const double* g, double tau, const mlsqr_stop* stop, double* f,
                     mlsqr_iter_rec* trace, double* alphas, double* betas, mlsqr_solve_info* info,
                     int ptr_kind) {
  return run_solve(op, nullptr, g, tau, stop, f, trace, alphas, betas, info, ptr_kind, true);
}

// mlsqr / lsqr with SolveOptions: basis, left basis and snapshots staged for HOST calls
static int solve_with_impl(mlsqr_op* op, mlsqr_pc* pc, const double* g, double tau, const mlsqr_stop* stop,
                           double* f, mlsqr_iter_rec* trace, double* alphas, double* betas, double* basis,
                           double* left_basis, double* snaps, mlsqr_solve_info* info, int kind) {
  int bd_iter = 0;
  if (info) std::memset(info, 0, sizeof(*info));
  const int st = guard([&] {
    require(op && stop, MLSQR_EINVAL, "operator and stopping config are required");
    Op* o = op->impl;
    Ctx* c = o->ctx;
    set_device(c);
    In gin(c, g, o->rows, kind);
    Out fout(c, f, o->cols, kind);
    const size_t nb = ((size_t)stop->max_iters + 1) * o->cols;
    const size_t nl = ((size_t)stop->max_iters + 1) * o->rows;
    const size_t ns = (size_t)stop->max_iters * o->cols;
    DevBuf<double> staged, staged_l, staged_s;
    double* bd = basis;
    double* ld = left_basis;
    double* sd = snaps;
    if (kind != MLSQR_DEVICE) {
      if (basis) {
        staged.alloc(nb);
        bd = staged.p;
      }
      if (left_basis) {
        staged_l.alloc(nl);
        ld = staged_l.p;
      }
      if (snaps) {
        staged_s.alloc(ns);
        sd = staged_s.p;
      }
    }
    mlsqr_solve_info inf{};
    try {
      solve_mlsqr(o, pc ? pc->impl : nullptr, gin.d, tau, *stop, fout.d, trace, alphas, betas, &inf, nullptr, true, bd,
                  ld, sd);
    } catch (const Error& e) {
      if (e.code == MLSQR_EBREAKDOWN) bd_iter = e.iteration;
      if (info) *info = inf;
      throw;
    }
    if (info) *info = inf;
    if (kind != MLSQR_DEVICE && basis && inf.n_alphas > 0)
      MLSQR_CUDA(cudaMemcpyAsync(basis, bd, sizeof(double) * (size_t)inf.n_alphas * o->cols, cudaMemcpyDeviceToHost,
                                 c->stream));
    if (kind != MLSQR_DEVICE && left_basis && inf.n_left_basis > 0)
      MLSQR_CUDA(cudaMemcpyAsync(left_basis, ld, sizeof(double) * (size_t)inf.n_left_basis * o->rows,
                                 cudaMemcpyDeviceToHost, c->stream));
    if (kind != MLSQR_DEVICE && snaps && inf.iterations > 0)
      MLSQR_CUDA(cudaMemcpyAsync(snaps, sd, sizeof(double) * (size_t)inf.iterations * o->cols,
                                 cudaMemcpyDeviceToHost, c->stream));
    fout.finish();
  });
  if (st == MLSQR_EBREAKDOWN && info) info->breakdown_iteration = bd_iter;
  return st;
}

int mlsqr_solve_basis(mlsqr_op* op, mlsqr_pc* pc, const double* g, double tau, const mlsqr_stop* stop,
                      double* f, mlsqr_iter_rec* trace, double* alphas, double* betas, double* basis,
                      double* left_basis, mlsqr_solve_info* info, int kind) {
  if (!basis) {
    g_err = "operator, stopping config and basis are required";
    if (info) std::memset(info, 0, sizeof(*info));
    return MLSQR_EINVAL;
  }
  return solve_with_impl(op, pc, g, tau, stop, f, trace, alphas, betas, basis, left_basis, nullptr, info, kind);
}

int mlsqr_solve_with(mlsqr_op* op, mlsqr_pc* pc, const double* g, double tau, const mlsqr_stop* stop,
                     const mlsqr_solve_opts* opts, double* f, mlsqr_iter_rec* trace, double* alphas,
                     double* betas, mlsqr_solve_info* info, int kind) {
  mlsqr_solve_opts o{};
  if (opts) o = *opts;
  if ((o.record_snapshots && !o.snapshots) || (o.store_basis && !o.basis)) {
    g_err = "SolveOptions requests an output without a buffer";
    if (info) std::memset(info, 0, sizeof(*info));
    return MLSQR_EINVAL;
  }
  return solve_with_impl(op, pc, g, tau, stop, f, trace, alphas, betas, o.store_basis ? o.basis : nullptr,
                         o.store_basis ? o.left_basis : nullptr, o.record_snapshots ? o.snapshots : nullptr,
                         info, kind);
}

int mlsqr_solve_projected(const double* alphas, size_t k, const double* betas, size_t n_betas, double beta1,
                          double tau, double* y) {
  return guard([&] {
    require(alphas && betas && y, MLSQR_EINVAL, "solve_projected: null argument");
    const std::vector<double> v = solve_projected(alphas, k, betas, n_betas, beta1, tau);
    std::memcpy(y, v.data(), sizeof(double) * k);
  });
}

int mlsqr_reconstruct_from_basis(mlsqr_ctx* ctx, const double* basis, size_t n, const double* y, size_t ny,
                                 double* f, int kind) {
  return guard([&] {
    require(ctx && basis && y && f, MLSQR_EINVAL, "reconstruct_from_basis: null argument");
    require(ny >= 1, MLSQR_EINVAL, "no basis vectors were stored");
    Ctx* c = &ctx->impl;
    set_device(c);
    In bin(c, basis, ny * n, kind);
    DevBuf<double> yd(ny);
    MLSQR_CUDA(cudaMemcpyAsync(yd.p, y, sizeof(double) * ny, cudaMemcpyHostToDevice, c->stream));
    Out fout(c, f, n, kind);
    reconstruct_from_basis(c, bin.d, n, yd.p, ny, fout.d);
    fout.finish();
  });
}

static int cg_normal_impl(mlsqr_op* op, mlsqr_pc* m, const double* g, double tau, const mlsqr_stop* stop,
                          double* f, mlsqr_iter_rec* trace, mlsqr_solve_info* info, double* snaps, int kind) {
  int bd_iter = 0;
  if (info) std::memset(info, 0, sizeof(*info));
  const int st = guard([&] {
    require(op && stop, MLSQR_EINVAL, "operator and stopping config are required");
    require(m == nullptr || m->vc != nullptr, MLSQR_EINVAL, "cg_normal's M comes from a V-cycle map");
    Op* o = op->impl;
    Ctx* c = o->ctx;
    set_device(c);
    In gin(c, g, o->rows, kind);
    Out fout(c, f, o->cols, kind);
    try {
      DevBuf<double> staged;
      double* sd = snaps;
      if (snaps && kind != MLSQR_DEVICE) {
        staged.alloc((size_t)stop->max_iters * o->cols);
        sd = staged.p;
      }
      mlsqr_solve_info inf{};
      solve_cg_normal(o, m ? m->vc : nullptr, gin.d, tau, *stop, fout.d, trace, &inf, sd);
      if (info) *info = inf;
      if (snaps && kind != MLSQR_DEVICE && inf.iterations > 0)
        MLSQR_CUDA(cudaMemcpyAsync(snaps, sd, sizeof(double) * (size_t)inf.iterations * o->cols,
                                   cudaMemcpyDeviceToHost, c->stream));
      fout.finish();
    } catch (const Error& e) {
      if (e.code == MLSQR_EBREAKDOWN) bd_iter = e.iteration;
      throw;
    }
  });
  if (st == MLSQR_EBREAKDOWN && info) info->breakdown_iteration = bd_iter;
  return st;
}

int mlsqr_cg_normal_solve(mlsqr_op* op, mlsqr_pc* m, const double* g, double tau, const mlsqr_stop* stop,
                          double* f, mlsqr_iter_rec* trace, mlsqr_solve_info* info, int kind) {
  return cg_normal_impl(op, m, g, tau, stop, f, trace, info, nullptr, kind);
}

int mlsqr_cg_normal_solve_with(mlsqr_op* op, mlsqr_pc* m, const double* g, double tau, const mlsqr_stop* stop,
                               const mlsqr_solve_opts* opts, double* f, mlsqr_iter_rec* trace,
                               mlsqr_solve_info* info, int kind) {
  if (opts && opts->record_snapshots && !opts->snapshots) {
    g_err = "SolveOptions requests snapshots without a buffer";
    if (info) std::memset(info, 0, sizeof(*info));
    return MLSQR_EINVAL;
  }
  return cg_normal_impl(op, m, g, tau, stop, f, trace, info,
                        opts && opts->record_snapshots ? opts->snapshots : nullptr, kind);
}

int mlsqr_krylov_basis(mlsqr_op* op, mlsqr_pc* msolver, mlsqr_pc* m, double tau, const double* g, int k,
                       double* vectors, int* count, int* rank_exhausted, int kind) {
  if (count) *count = 0;
  if (rank_exhausted) *rank_exhausted = 0;
  return guard([&] {
    require(op && g && vectors && count && rank_exhausted, MLSQR_EINVAL, "krylov_basis: null argument");
    require(m == nullptr || m->vc != nullptr, MLSQR_EINVAL, "krylov_basis's M comes from a V-cycle map");
    require(k >= 1, MLSQR_EINVAL, "need at least one basis vector");
    Op* o = op->impl;
    Ctx* c = o->ctx;
    set_device(c);
    In gin(c, g, o->rows, kind);
    DevBuf<double> staged;
    double* vd = vectors;
    if (kind != MLSQR_DEVICE) {
      staged.alloc((size_t)k * o->cols);
      vd = staged.p;
    }
    const int cnt = krylov_basis(o, msolver ? msolver->impl : nullptr, m ? m->vc : nullptr, tau, gin.d, k, vd,
                                 rank_exhausted);
    *count = cnt;
    if (kind != MLSQR_DEVICE && cnt > 0)
      MLSQR_CUDA(cudaMemcpy(vectors, vd, sizeof(double) * (size_t)cnt * o->cols, cudaMemcpyDeviceToHost));
  });
}

int mlsqr_nonlinear_solve(mlsqr_op* op, const double* g, int dims, size_t nx, size_t ny,
                          size_t nz, double h, const mlsqr_outer_cfg* cfg, double* f_out,
                          mlsqr_outer_step* steps, int* n_steps, int* stop_reason,
                          int* triggered_at, double* alphas, double* betas, int kind) {
  return guard([&] {
    require(op && cfg && steps && n_steps && stop_reason && triggered_at, MLSQR_EINVAL,
            "nonlinear_solve: null argument");
    Op* o = op->impl;
    Ctx* c = o->ctx;
    set_device(c);
    In gin(c, g, o->rows, kind);
    Out fout(c, f_out, o->cols, kind);
    nonlinear_solve(o, gin.d, dims, nx, ny, nz, h, *cfg, fout.d, steps, n_steps, stop_reason,
                    triggered_at, alphas, betas);
    fout.finish();
  });
}

}  // extern "C"

struct mlsqr_outer {
  std::unique_ptr<OuterSolver> impl;
  int k = 0;
};

extern "C" {

int mlsqr_outer_create(mlsqr_op* op, int dims, size_t nx, size_t ny, size_t nz, double h,
                       const mlsqr_outer_cfg* cfg, mlsqr_outer** out) {
  return guard([&] {
    require(op && cfg && out, MLSQR_EINVAL, "outer_create: null argument");
    set_device(op->impl->ctx);
    auto* o = new mlsqr_outer();
    try {
      o->impl.reset(new OuterSolver(op->impl, dims, nx, ny, nz, h, *cfg));
    } catch (...) {
      delete o;
      throw;
    }
    *out = o;
  });
}

int mlsqr_outer_advance(mlsqr_outer* o, const double* g, const double* f_prev, double* f_out,
                     mlsqr_outer_step* step, int kind) {
  return guard([&] {
    Op* op = o->impl->op;
    Ctx* c = op->ctx;
    set_device(c);
    if (kind == MLSQR_DEVICE) {
      o->impl->step(g, f_prev, f_out, step, ++o->k);
      return;
    }
    // HOST buffers: f_prev first on the main stream (the hierarchy build needs only it), then g on
    // the side stream behind it (the same PCIe direction: no sharing), joined before the solve;
    // f_out returns on the side stream from inside step(), overlapped with R(f)
    In fin(c, f_prev, op->cols, kind);
    double* gd = static_cast<double*>(c->staging(sizeof(double) * op->rows));
    double* fd = static_cast<double*>(c->staging(sizeof(double) * op->cols));
    cudaStream_t side = c->side_stream();
    MLSQR_CUDA(cudaEventRecord(c->ev_copy, c->stream));
    MLSQR_CUDA(cudaStreamWaitEvent(side, c->ev_copy, 0));
    MLSQR_CUDA(cudaMemcpyAsync(gd, g, sizeof(double) * op->rows, cudaMemcpyHostToDevice, side));
    MLSQR_CUDA(cudaEventRecord(c->ev_copy, side));
    struct Reset {  // also on an error path: no copy may still touch the caller's buffers
      OuterSolver* s;
      cudaStream_t side;
      ~Reset() {
        s->g_ready = nullptr;
        s->out_host = nullptr;
        cudaStreamSynchronize(side);
      }
    } reset{o->impl.get(), side};
    o->impl->g_ready = c->ev_copy;
    o->impl->out_host = f_out;
    o->impl->step(gd, fin.d, fd, step, ++o->k);
  });
}

int mlsqr_outer_last_bidiag(mlsqr_outer* o, double* alphas, size_t cap_a, double* betas, size_t cap_b,
                            int* n_alphas, int* n_betas) {
  return guard([&] {
    require(o && n_alphas && n_betas, MLSQR_EINVAL, "outer_last_bidiag: null argument");
    const OuterSolver& s = *o->impl;
    const size_t na = (size_t)s.last_info.n_alphas, nb = (size_t)s.last_info.n_betas;
    require((!alphas || cap_a >= na) && (!betas || cap_b >= nb), MLSQR_EDIM, "outer_last_bidiag: buffer too short");
    if (alphas) std::memcpy(alphas, s.al_.data(), sizeof(double) * na);
    if (betas) std::memcpy(betas, s.be_.data(), sizeof(double) * nb);
    *n_alphas = (int)na;
    *n_betas = (int)nb;
  });
}

int mlsqr_outer_destroy(mlsqr_outer* o) {
  return guard([&] { delete o; });
}

int mlsqr_penalty_functional(mlsqr_ctx* ctx, int dims, size_t nx, size_t ny, size_t nz, double h,
                             const double* f, int kind, int pen_kind, double T, double* value) {
  return guard([&] {
    Ctx* c = &ctx->impl;
    set_device(c);
    require(dims >= 1 && dims <= 3, MLSQR_EINVAL, "grid must be 1D, 2D or 3D");
    const size_t n = nx * (dims >= 2 ? ny : 1) * (dims >= 3 ? nz : 1);
    In in(c, f, n, kind);
    *value = penalty_functional_dev(c, dims, nx, ny, nz, h, in.d, pen_kind, T);
  });
}

}  // extern "C"
