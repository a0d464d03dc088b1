"""paper_1308_6634_b200 -- B200-native priorconditioned LSQR (arXiv 1308.6634 hot path).

A Python mirror of the reference's C++ interface for this path
(/root/reference/proj/include/mlsqr): LinearOperator (linop.hpp:21-47),
SpdMap (spdsolve.hpp:11-22), StoppingConfig / mlsqr / lsqr (krylov.hpp),
OuterConfig / solve_nonlinear (outer.hpp), PenaltySpec (penalty.hpp) -- same
names, argument meaning and error types -- over the C-ABI library
libmlsqr_b200.so (include/mlsqr_b200.h).  All arithmetic runs in the CUDA
kernels of that library; there is no CPU fallback: without the built
extension or without a B200 the calls raise.

Vectors may be numpy arrays (host; copied around the call, the reference's
std::span contract) or CUDA torch tensors (device-resident, no copies).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MLSQR_LIB_PATH") or os.path.join(HERE, "libmlsqr_b200.so")  # override: A/B builds

__all__ = [
    "DimensionError", "BreakdownError", "CudaError", "Context", "default_context",
    "LinearOperator", "SeparableGaussianBlur", "DenseOperator", "FdotOperator",
    "IdentityOperator", "SpdMap", "IdentityMap", "VCycleMap", "CallbackMap", "CholeskyMap",
    "InnerCgMap", "FactorizationError", "krylov_basis", "cg_normal",
    "StoppingConfig", "IterationRecord", "SolveResult", "mlsqr", "lsqr", "PenaltySpec",
    "OuterConfig", "OuterStep", "OuterReport", "solve_nonlinear", "penalty_functional",
    "gaussian_taps", "gaussian_noise", "phantom_rects2d", "phantom_shapes2d",
    "phantom_ellipsoids3d", "fdot_tables", "lib",
]


# ---------------------------------------------------------------------------
# errors (errors.hpp:9-41)
# ---------------------------------------------------------------------------
class DimensionError(ValueError):
    """Caller passed a vector whose length does not match (errors.hpp:9-13)."""


class BreakdownError(RuntimeError):
    """Nonpositive M-weighted square norm: the map is not SPD (errors.hpp:27-36)."""

    def __init__(self, msg: str, iteration: int):
        super().__init__(msg)
        self.iteration = iteration


class CudaError(RuntimeError):
    """CUDA failure or no B200 visible (the product has no CPU fallback)."""


class FactorizationError(RuntimeError):
    """Cholesky hit a nonpositive pivot (errors.hpp:14-24)."""

    def __init__(self, msg: str, pivot_row: int):
        super().__init__(msg)
        self.pivot_row = pivot_row


OK, EDIM, EINVAL, EBREAKDOWN, ECUDA, ENCCL, ECALLBACK, EFACTOR = 0, 1, 2, 3, 4, 5, 6, 7
HOST, DEVICE = 0, 1
STOP_NAMES = ["S1", "S2", "S3", "S4", "max_iters", "breakdown"]
SPD_MODES = {"vcycle": 0, "cholesky": 1, "inner_cg": 2}
PEN_KINDS = {"tikhonov": 0, "tv": 1, "tv_smoothed": 1, "pm_log": 2, "perona_malik_log": 2,
             "pm_exp": 3, "perona_malik_exp": 3}
dp = C.POINTER(C.c_double)
HOST_MAP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, dp, dp)


# ---------------------------------------------------------------------------
# C structs (include/mlsqr_b200.h)
# ---------------------------------------------------------------------------
class _Stop(C.Structure):
    _fields_ = [("atol", C.c_double), ("btol", C.c_double), ("conlim", C.c_double),
                ("delta", C.c_double), ("eta", C.c_double), ("max_iters", C.c_int),
                ("use_s1", C.c_int), ("use_s2", C.c_int), ("use_s3", C.c_int), ("use_s4", C.c_int)]


class _IterRec(C.Structure):
    _fields_ = [("iteration", C.c_int), ("res_data_exact", C.c_int), ("res_damped", C.c_double),
                ("res_data", C.c_double), ("s2_value", C.c_double), ("anorm_est", C.c_double),
                ("cond_est", C.c_double), ("xnorm_est", C.c_double), ("alpha", C.c_double),
                ("beta", C.c_double)]


class _Info(C.Structure):
    _fields_ = [("iterations", C.c_int), ("stop_reason", C.c_int), ("n_alphas", C.c_int),
                ("n_betas", C.c_int), ("breakdown_iteration", C.c_int), ("n_left_basis", C.c_int)]


class _OuterCfg(C.Structure):
    _fields_ = [("tau", C.c_double), ("pen_kind", C.c_int), ("T", C.c_double), ("inner_stop", _Stop),
                ("inner_cap", C.c_int), ("rel_decrease_threshold", C.c_double), ("max_outer", C.c_int),
                ("epsilon", C.c_double), ("mg_levels", C.c_int), ("nu_pre", C.c_int),
                ("nu_post", C.c_int), ("coarse_sweeps", C.c_int), ("omega", C.c_double),
                ("spd_mode", C.c_int), ("k_inner", C.c_int)]


class _OuterStep(C.Structure):
    _fields_ = [("k", C.c_int), ("inner_iterations", C.c_int), ("inner_stop", C.c_int),
                ("penalty_value", C.c_double), ("final_residual", C.c_double), ("eps_used", C.c_double)]


# exported symbols and their signatures (tests check every one is present)
SIGNATURES = {
    "mlsqr_last_error": (C.c_char_p, []),
    "mlsqr_version": (C.c_char_p, []),
    "mlsqr_ctx_create": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "mlsqr_ctx_destroy": (C.c_int, [C.c_void_p]),
    "mlsqr_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "mlsqr_dev_alloc": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "mlsqr_dev_free": (C.c_int, [C.c_void_p, C.c_void_p]),
    "mlsqr_copy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_size_t]),
    "mlsqr_ctx_launch_count": (C.c_uint64, [C.c_void_p, C.c_int]),
    "mlsqr_ctx_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "mlsqr_ctx_get_timing": (C.c_int, [C.c_void_p, C.c_int, dp, C.POINTER(C.c_uint64)]),
    "mlsqr_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "mlsqr_ctx_set_comm_nccl": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "mlsqr_loop_group_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "mlsqr_loop_group_destroy": (C.c_int, [C.c_void_p]),
    "mlsqr_ctx_set_comm_loopback": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "mlsqr_ctx_set_slab": (C.c_int, [C.c_void_p, C.c_size_t, C.c_size_t]),
    "mlsqr_ctx_set_row_shard": (C.c_int, [C.c_void_p, C.c_size_t, C.c_size_t]),
    "mlsqr_blur_create": (C.c_int, [C.c_void_p, C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, dp,
                                    C.c_int, C.POINTER(C.c_void_p)]),
    "mlsqr_blur2d_create_axes": (C.c_int, [C.c_void_p, C.c_size_t, C.c_size_t, dp, C.c_int, dp, C.c_int,
                                           C.POINTER(C.c_void_p)]),
    "mlsqr_dense_create": (C.c_int, [C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p, C.c_int,
                                     C.c_size_t, C.POINTER(C.c_void_p)]),
    "mlsqr_dense_create_fdot": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, C.c_int, dp, dp,
                                          C.c_size_t, C.POINTER(C.c_void_p)]),
    "mlsqr_identity_create": (C.c_int, [C.c_void_p, C.c_size_t, C.c_size_t, C.POINTER(C.c_void_p)]),
    "mlsqr_op_destroy": (C.c_int, [C.c_void_p]),
    "mlsqr_op_shape": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "mlsqr_op_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int]),
    "mlsqr_op_apply_adjoint": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                         C.c_int]),
    "mlsqr_identity_map_create": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "mlsqr_vcycle_create": (C.c_int, [C.c_void_p, C.c_int, C.c_size_t, C.c_size_t, C.c_size_t,
                                      C.c_double, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                      C.POINTER(C.c_void_p)]),
    "mlsqr_vcycle_set_coefficients": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_double, C.c_int]),
    "mlsqr_vcycle_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_double,
                                      C.c_double, dp]),
    "mlsqr_callback_map_create": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                            C.POINTER(C.c_void_p)]),
    "mlsqr_chol_map_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_longlong)]),
    "mlsqr_inner_cg_map_create": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "mlsqr_pc_destroy": (C.c_int, [C.c_void_p]),
    "mlsqr_pc_dimension": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "mlsqr_pc_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]),
    "mlsqr_vcycle_m_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]),
    "mlsqr_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.POINTER(_Stop),
                              C.c_void_p, C.POINTER(_IterRec), dp, dp, C.POINTER(_Info), C.c_int]),
    "mlsqr_lsqr_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.POINTER(_Stop), C.c_void_p,
                                   C.POINTER(_IterRec), dp, dp, C.POINTER(_Info), C.c_int]),
    "mlsqr_solve_basis": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.POINTER(_Stop), C.c_void_p,
                                    C.POINTER(_IterRec), dp, dp, C.c_void_p, C.c_void_p, C.POINTER(_Info),
                                    C.c_int]),
    "mlsqr_solve_with": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.POINTER(_Stop),
                                   C.c_void_p, C.c_void_p, C.POINTER(_IterRec), dp, dp, C.POINTER(_Info),
                                   C.c_int]),
    "mlsqr_cg_normal_solve_with": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.POINTER(_Stop),
                                             C.c_void_p, C.c_void_p, C.POINTER(_IterRec), C.POINTER(_Info),
                                             C.c_int]),
    "mlsqr_krylov_basis": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_int,
                                     C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int]),
    "mlsqr_solve_projected": (C.c_int, [dp, C.c_size_t, dp, C.c_size_t, C.c_double, C.c_double, dp]),
    "mlsqr_reconstruct_from_basis": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, dp, C.c_size_t, C.c_void_p,
                                               C.c_int]),
    "mlsqr_cg_normal_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.POINTER(_Stop),
                                        C.c_void_p, C.POINTER(_IterRec), C.POINTER(_Info), C.c_int]),
    "mlsqr_nonlinear_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_size_t, C.c_size_t,
                                        C.c_size_t, C.c_double, C.POINTER(_OuterCfg), C.c_void_p,
                                        C.POINTER(_OuterStep), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), dp, dp, C.c_int]),
    "mlsqr_outer_create": (C.c_int, [C.c_void_p, C.c_int, C.c_size_t, C.c_size_t, C.c_size_t,
                                     C.c_double, C.POINTER(_OuterCfg), C.POINTER(C.c_void_p)]),
    "mlsqr_outer_advance": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.POINTER(_OuterStep), C.c_int]),
    "mlsqr_outer_last_bidiag": (C.c_int, [C.c_void_p, dp, C.c_size_t, dp, C.c_size_t, C.POINTER(C.c_int),
                                         C.POINTER(C.c_int)]),
    "mlsqr_outer_destroy": (C.c_int, [C.c_void_p]),
    "mlsqr_penalty_functional": (C.c_int, [C.c_void_p, C.c_int, C.c_size_t, C.c_size_t, C.c_size_t,
                                           C.c_double, C.c_void_p, C.c_int, C.c_int, C.c_double, dp]),
    "mlsqr_taps": (C.c_int, [C.c_size_t, C.c_double, C.c_double, C.c_int, dp, C.POINTER(C.c_int)]),
    "mlsqr_gauss_fill": (C.c_int, [C.c_uint64, C.c_size_t, C.c_double, dp]),
    "mlsqr_phantom_rects2d": (C.c_int, [C.c_size_t, C.c_size_t, C.c_int, C.c_uint64, dp]),
    "mlsqr_phantom_shapes2d": (C.c_int, [C.c_size_t, C.c_size_t, C.c_int, C.c_uint64, dp]),
    "mlsqr_phantom_ellipsoids3d": (C.c_int, [C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.c_double,
                                             C.c_double, C.c_double, C.c_double, C.c_uint64, dp]),
    "mlsqr_fdot_tables": (C.c_int, [C.c_size_t, C.c_int, C.c_int, C.c_double, C.c_uint64, dp, dp]),
}

_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Load libmlsqr_b200.so (fails loudly when the extension is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_1308_6634_b200.build` "
                              "(there is no CPU fallback for this path)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int, info: Optional[_Info] = None) -> None:
    if status == OK:
        return
    msg = lib().mlsqr_last_error().decode(errors="replace")
    if status == EDIM:
        raise DimensionError(msg)
    if status == EINVAL:
        raise ValueError(msg)
    if status == EBREAKDOWN:
        raise BreakdownError(msg, info.breakdown_iteration if info is not None else -1)
    if status == EFACTOR:
        raise FactorizationError(msg, int(msg.rsplit(" ", 1)[-1]) if msg[-1:].isdigit() else -1)
    raise CudaError(f"[status {status}] {msg}")


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(dp) if a is not None else None


def _is_dev(t) -> bool:
    return hasattr(t, "data_ptr") and getattr(t, "is_cuda", False)


def _vec_in(x):
    """(pointer, length, kind, keepalive) for a host array or a CUDA tensor.

    Stream ordering (mlsqr_b200.h, MLSQR_DEVICE): a context's stream does not wait for
    torch's streams, so before the library reads a CUDA tensor (or writes into memory that
    torch work still pending may use) torch's current stream on that device is drained."""
    if _is_dev(x):
        assert str(x.dtype) == "torch.float64" and x.is_contiguous(), "device vectors must be contiguous float64"
        import torch
        torch.cuda.current_stream(x.device).synchronize()
        return C.c_void_p(x.data_ptr()), x.numel(), DEVICE, x
    a = _f64(x).ravel()
    return C.c_void_p(a.ctypes.data), a.size, HOST, a


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------
class Context:
    """Device + CUDA stream.  `stream` (an int cudaStream_t, e.g.
    torch.cuda.current_stream().cuda_stream) lets torch events time our kernels."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = C.c_void_p()
        _check(lib().mlsqr_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h
        self.device = device

    def synchronize(self) -> None:
        _check(lib().mlsqr_ctx_synchronize(self.h))

    # ---- z-slab decomposition
    def set_slab(self, nz_global: int, z_offset: int) -> None:
        """Objects built on this context with z extent nz are planes [z_offset, z_offset+nz)
        of a global grid with nz_global planes."""
        _check(lib().mlsqr_ctx_set_slab(self.h, nz_global, z_offset))

    def set_row_shard(self, rows_global: int, row_offset: int) -> None:
        """Dense operators built on this context hold data rows [row_offset, row_offset +
        rows_global / P); solution-space vectors and preconditioners are replicated."""
        _check(lib().mlsqr_ctx_set_row_shard(self.h, rows_global, row_offset))

    def set_comm_nccl(self, unique_id: bytes, rank: int, size: int) -> None:
        _nccl_first()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(lib().mlsqr_ctx_set_comm_nccl(self.h, buf, rank, size))

    def set_comm_loopback(self, group: "LoopGroup", rank: int) -> None:
        _check(lib().mlsqr_ctx_set_comm_loopback(self.h, group.h, rank))
        self._group = group  # keep the group alive

    def launch_count(self, reset: bool = False) -> int:
        return int(lib().mlsqr_ctx_launch_count(self.h, int(reset)))

    def set_timing(self, on: bool) -> None:
        _check(lib().mlsqr_ctx_set_timing(self.h, int(on)))

    def timing(self, cls: int):
        ms, n = C.c_double(), C.c_uint64()
        _check(lib().mlsqr_ctx_get_timing(self.h, cls, C.byref(ms), C.byref(n)))
        return ms.value, int(n.value)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().mlsqr_ctx_destroy(self.h)
        except Exception:
            pass


def _nccl_first():
    """Load torch's bundled NCCL before the library dlopens libnccl.so.2: torch binds to the
    first libnccl.so.2 in the process, so a system NCCL loaded first would break `import torch`."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    """An ncclUniqueId (128 bytes) for Context.set_comm_nccl; broadcast it from rank 0."""
    _nccl_first()
    buf = C.create_string_buffer(128)
    n = C.c_size_t()
    _check(lib().mlsqr_nccl_unique_id(buf, 128, C.byref(n)))
    return buf.raw[:n.value]


class LoopGroup:
    """P virtual ranks of one process on one GPU (each with its own Context and thread)."""

    def __init__(self, size: int):
        h = C.c_void_p()
        _check(lib().mlsqr_loop_group_create(size, C.byref(h)))
        self.h, self.size = h, size

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().mlsqr_loop_group_destroy(self.h)
        except Exception:
            pass


TCLASS = {"blur": 0, "dense": 1, "smooth": 2, "mg": 3, "update": 4, "iter": 5, "sweep_fn": 6,
          "sweep_prolong": 7, "sweep_last": 8, "restrict": 9, "halo": 10, "coll": 11}
_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


# ---------------------------------------------------------------------------
# LinearOperator (linop.hpp:21-47)
# ---------------------------------------------------------------------------
class LinearOperator:
    """A : R^{n_cols} -> R^{n_rows}; apply / apply_adjoint raise DimensionError on
    length mismatch (linop.cpp:15-40)."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx
        r, c = C.c_size_t(), C.c_size_t()
        _check(lib().mlsqr_op_shape(self.h, C.byref(r), C.byref(c)))
        self.n_rows, self.n_cols = r.value, c.value

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    def apply(self, x, y=None):
        xp, xn, kind, keep = _vec_in(x)
        if kind == DEVICE:
            import torch
            y = torch.empty(self.n_rows, dtype=torch.float64, device=x.device) if y is None else y
            _check(lib().mlsqr_op_apply(self.h, xp, xn, C.c_void_p(y.data_ptr()), y.numel(), DEVICE))
            return y
        out = np.zeros(self.n_rows) if y is None else y
        _check(lib().mlsqr_op_apply(self.h, xp, xn, C.c_void_p(out.ctypes.data), out.size, HOST))
        return out

    def apply_adjoint(self, y, x=None):
        yp, yn, kind, keep = _vec_in(y)
        if kind == DEVICE:
            import torch
            x = torch.empty(self.n_cols, dtype=torch.float64, device=y.device) if x is None else x
            _check(lib().mlsqr_op_apply_adjoint(self.h, yp, yn, C.c_void_p(x.data_ptr()), x.numel(), DEVICE))
            return x
        out = np.zeros(self.n_cols) if x is None else x
        _check(lib().mlsqr_op_apply_adjoint(self.h, yp, yn, C.c_void_p(out.ctypes.data), out.size, HOST))
        return out

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().mlsqr_op_destroy(self.h)
        except Exception:
            pass


class SeparableGaussianBlur(LinearOperator):
    """Separable Gaussian blur on a 1D/2D/3D grid (SeparableGaussianBlur2D,
    linop.hpp:110-126, + z pass).  `taps` (2R+1 values) or (sigma_f, radius):
    taps = gaussian_taps(shape[0], sigma_f, radius); radius=None is the
    reference's ceil(6 sigma / h)."""

    def __init__(self, shape, sigma_f: Optional[float] = None, radius: Optional[int] = None,
                 taps=None, ctx: Optional[Context] = None, taps_y=None):
        ctx = ctx or default_context()
        shape = tuple(int(s) for s in shape)
        dims = len(shape)
        if taps is None:
            taps = gaussian_taps(shape[0], sigma_f, -1 if radius is None else radius)
        taps = _f64(taps)
        nx, ny, nz = (list(shape) + [1, 1])[:3]
        h = C.c_void_p()
        if taps_y is None and dims == 2 and nx != ny and sigma_f is not None and radius is None:
            # the reference's 2D operator builds ky_(ny, sigma_f) on its own spacing (linop.cpp:144-147)
            taps_y = gaussian_taps(ny, sigma_f, -1)
        if taps_y is not None:
            ty = _f64(taps_y)
            _check(lib().mlsqr_blur2d_create_axes(ctx.h, nx, ny, _ptr(taps), (taps.size - 1) // 2, _ptr(ty),
                                                  (ty.size - 1) // 2, C.byref(h)))
        else:
            _check(lib().mlsqr_blur_create(ctx.h, dims, nx, ny, nz, _ptr(taps), (taps.size - 1) // 2,
                                           C.byref(h)))
        self.grid_shape, self.taps, self.taps_y = shape, taps, taps_y
        super().__init__(h, ctx)


class DenseOperator(LinearOperator):
    """Row-major dense matrix (DenseOperator, linop.hpp:59-71)."""

    def __init__(self, a, sol_row_len: int = 0, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        h = C.c_void_p()
        if _is_dev(a):
            rows, cols = a.shape
            _check(lib().mlsqr_dense_create(ctx.h, rows, cols, C.c_void_p(a.data_ptr()), DEVICE, sol_row_len, C.byref(h)))
        else:
            a = _f64(a)
            rows, cols = a.shape
            _check(lib().mlsqr_dense_create(ctx.h, rows, cols, C.c_void_p(a.ctypes.data), HOST, sol_row_len, C.byref(h)))
        super().__init__(h, ctx)


class FdotOperator(LinearOperator):
    """fDOT-like dense sensitivity operator A[(s,d), x] = G(s,x) G(x,d) formed on the device."""

    def __init__(self, n: int, n_src: int, n_det: int, mu: float = 1.0, seed: int = 0,
                 tables=None, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        gs, gd = tables if tables is not None else fdot_tables(n, n_src, n_det, mu, seed)
        gs, gd = _f64(gs), _f64(gd)
        h = C.c_void_p()
        _check(lib().mlsqr_dense_create_fdot(ctx.h, n ** 3, n_src, n_det, _ptr(gs), _ptr(gd), n, C.byref(h)))
        super().__init__(h, ctx)


class IdentityOperator(LinearOperator):
    def __init__(self, n: int, row_len: int = 0, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(lib().mlsqr_identity_create(ctx.h, n, row_len, C.byref(h)))
        super().__init__(h, ctx)


# ---------------------------------------------------------------------------
# SpdMap (spdsolve.hpp:11-33)
# ---------------------------------------------------------------------------
class SpdMap:
    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx
        n = C.c_size_t()
        _check(lib().mlsqr_pc_dimension(self.h, C.byref(n)))
        self.n = n.value

    def dimension(self) -> int:
        return self.n

    def solve(self, p, v=None):
        pp, pn, kind, keep = _vec_in(p)
        if kind == DEVICE:
            import torch
            v = torch.empty(self.n, dtype=torch.float64, device=p.device) if v is None else v
            _check(lib().mlsqr_pc_solve(self.h, pp, C.c_void_p(v.data_ptr()), pn, DEVICE))
            return v
        out = np.zeros(self.n) if v is None else v
        _check(lib().mlsqr_pc_solve(self.h, pp, C.c_void_p(out.ctypes.data), pn, HOST))
        return out

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().mlsqr_pc_destroy(self.h)
        except Exception:
            pass


class IdentityMap(SpdMap):
    def __init__(self, n: int, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(lib().mlsqr_identity_map_create(ctx.h, n, C.byref(h)))
        super().__init__(h, ctx)


class VCycleMap(SpdMap):
    """Multigrid V-cycle approximating M^{-1} for the edge-based diffusion
    operator M_f (diffusion.hpp:12-20): 2^d aggregation, Galerkin coarse edges,
    omega-Jacobi nu_pre/nu_post sweeps, fixed coarse sweeps -- a fixed SPD map."""

    def __init__(self, shape, h: float, levels: int, nu_pre: int = 2, nu_post: int = 2,
                 omega: float = 2.0 / 3.0, coarse_sweeps: int = 4, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        shape = tuple(int(s) for s in shape)
        nx, ny, nz = (list(shape) + [1, 1])[:3]
        hh = C.c_void_p()
        _check(lib().mlsqr_vcycle_create(ctx.h, len(shape), nx, ny, nz, h, levels, nu_pre, nu_post,
                                         omega, coarse_sweeps, C.byref(hh)))
        self.grid_shape = shape
        super().__init__(hh, ctx)

    def set_coefficients(self, cx, cy=None, cz=None, eps: float = 0.0) -> None:
        arrs = [None if a is None else _f64(a) for a in (cx, cy, cz)]
        ptrs = [None if a is None else C.c_void_p(a.ctypes.data) for a in arrs]
        _check(lib().mlsqr_vcycle_set_coefficients(self.h, ptrs[0], ptrs[1], ptrs[2], eps, HOST))

    def update(self, f, penalty: "PenaltySpec", eps: Optional[float] = None) -> float:
        """assemble_m + auto_shift at field f (diffusion.cpp:59-87); returns eps used."""
        fp, fn, kind, keep = _vec_in(f)
        e = C.c_double()
        _check(lib().mlsqr_vcycle_update(self.h, fp, kind, penalty.kind_code, penalty.threshold,
                                         -1.0 if eps is None else eps, C.byref(e)))
        return e.value

    def m_apply(self, x):
        xp, xn, kind, keep = _vec_in(x)
        out = np.zeros(self.n)
        _check(lib().mlsqr_vcycle_m_apply(self.h, xp, C.c_void_p(out.ctypes.data), xn, HOST))
        return out


class CholeskyMap(SpdMap):
    """SpdSolver::factorize (spdsolve.cpp:22-75): envelope Cholesky of the M (+ shift) a
    V-cycle map holds (VCycleMap(levels=1) is a plain holder of M), factorized and applied on
    the device in the reference's operation order.  FactorizationError on a nonpositive pivot."""

    def __init__(self, m: "VCycleMap"):
        h = C.c_void_p()
        row = C.c_longlong(-1)
        _check(lib().mlsqr_chol_map_create(m.h, C.byref(h), C.byref(row)))
        self.grid_shape = m.grid_shape
        super().__init__(h, m.ctx)


class InnerCgMap(SpdMap):
    """SpdSolver::inner_cg (spdsolve.cpp:77-85, 119-137): k_inner CG iterations from zero on a
    snapshot of the M a V-cycle map holds; device-resident (graph-capturable)."""

    def __init__(self, m: "VCycleMap", k_inner: int):
        h = C.c_void_p()
        _check(lib().mlsqr_inner_cg_map_create(m.h, int(k_inner), C.byref(h)))
        self.grid_shape = m.grid_shape
        super().__init__(h, m.ctx)


class CallbackMap(SpdMap):
    """A host SpdMap plug-in: fn(p: np.ndarray) -> v (test fakes, parity maps)."""

    def __init__(self, n: int, fn, ctx: Optional[Context] = None):
        ctx = ctx or default_context()

        def tramp(user, p, v):
            try:
                pa = np.ctypeslib.as_array(p, shape=(n,))
                va = np.ctypeslib.as_array(v, shape=(n,))
                va[:] = fn(pa.copy())
                return 0
            except Exception:
                return 1

        self._cb = HOST_MAP_FN(tramp)
        h = C.c_void_p()
        _check(lib().mlsqr_callback_map_create(ctx.h, n, C.cast(self._cb, C.c_void_p), None, C.byref(h)))
        super().__init__(h, ctx)


# ---------------------------------------------------------------------------
# Krylov (krylov.hpp)
# ---------------------------------------------------------------------------
@dataclass
class StoppingConfig:
    """StoppingConfig (krylov.hpp:19-36)."""
    atol: float = 1e-8
    btol: float = 1e-8
    conlim: float = 1e8
    delta: float = 0.0
    eta: float = 1.1
    max_iters: int = 100
    use_s1: bool = False
    use_s2: bool = False
    use_s3: bool = False
    use_s4: bool = False

    @staticmethod
    def max_iterations(n: int) -> "StoppingConfig":
        c = StoppingConfig(max_iters=n)
        c.validate()
        return c

    @staticmethod
    def discrepancy(delta: float, eta: float, max_iters: int) -> "StoppingConfig":
        c = StoppingConfig(delta=delta, eta=eta, max_iters=max_iters, use_s4=True)
        c.validate()
        return c

    @staticmethod
    def lsqr_classic(atol: float, btol: float, conlim: float, max_iters: int) -> "StoppingConfig":
        c = StoppingConfig(atol=atol, btol=btol, conlim=conlim, max_iters=max_iters, use_s1=True,
                           use_s2=True, use_s3=True)
        c.validate()
        return c

    def validate(self) -> None:  # krylov.cpp:219-226
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if self.use_s4 and not self.eta > 1.0:
            raise ValueError("discrepancy stopping needs a safety factor eta > 1")
        if self.use_s4 and not self.delta >= 0.0:
            raise ValueError("noise level delta must be >= 0")
        if not (self.atol >= 0.0 and self.btol >= 0.0):
            raise ValueError("tolerances must be >= 0")

    def _c(self) -> _Stop:
        return _Stop(self.atol, self.btol, self.conlim, self.delta, self.eta, self.max_iters,
                     int(self.use_s1), int(self.use_s2), int(self.use_s3), int(self.use_s4))


@dataclass
class IterationRecord:
    iteration: int
    res_damped: float
    res_data: float
    res_data_exact: bool
    s2_value: float
    anorm_est: float
    cond_est: float
    xnorm_est: float
    alpha: float
    beta: float


@dataclass
class SolveResult:
    solution: object
    iterations: int
    stop_reason: str
    trace: list
    alphas: np.ndarray
    betas: np.ndarray
    basis: object = None       # [n_alphas, n] right basis when store_basis was requested
    left_basis: object = None  # [n_left, m] left basis u_1 .. u_{k+1}
    snapshots: object = None   # [iterations, n] f after each iteration (record_snapshots)


class _SolveOpts(C.Structure):  # mlsqr_solve_opts (SolveOptions, krylov.hpp:77-80)
    _fields_ = [("record_snapshots", C.c_int), ("store_basis", C.c_int), ("snapshots", C.c_void_p),
                ("basis", C.c_void_p), ("left_basis", C.c_void_p)]


def _run(op: LinearOperator, pc: Optional[SpdMap], g, tau: float, stop: StoppingConfig,
         f_out=None, cgn: bool = False, store_basis: bool = False,
         record_snapshots: bool = False) -> SolveResult:
    stop.validate()
    if not tau >= 0.0:
        raise ValueError("tau must be nonnegative")
    gp, gn, kind, keep = _vec_in(g)
    if gn != op.n_rows:
        raise DimensionError("right-hand side length mismatch")
    if pc is not None and pc.n != op.n_cols:
        raise DimensionError("preconditioner dimension does not match operator columns")
    k = stop.max_iters
    tr = (_IterRec * k)()
    al = np.zeros(k + 1)
    be = np.zeros(k + 2)
    info = _Info()

    def buf(count):
        if kind == DEVICE:
            import torch
            t = torch.empty(count, dtype=torch.float64, device=g.device)
            return t, C.c_void_p(t.data_ptr())
        a = np.zeros(count)
        return a, C.c_void_p(a.ctypes.data)

    if f_out is None:
        f, fptr = buf(op.n_cols)
    else:
        f = f_out
        fptr = C.c_void_p(f.data_ptr() if kind == DEVICE else f.ctypes.data)
    sc = stop._c()
    opts = _SolveOpts()
    basis = left = snaps = None
    if store_basis and not cgn:
        basis, opts.basis = buf((k + 1) * op.n_cols)
        left, opts.left_basis = buf((k + 1) * op.n_rows)
        opts.store_basis = 1
    if record_snapshots:
        snaps, opts.snapshots = buf(k * op.n_cols)
        opts.record_snapshots = 1
    pch = pc.h if pc is not None else None
    if cgn:
        st = lib().mlsqr_cg_normal_solve_with(op.h, pch, gp, tau, C.byref(sc), C.byref(opts), fptr, tr,
                                              C.byref(info), kind)
    elif opts.store_basis or opts.record_snapshots:
        st = lib().mlsqr_solve_with(op.h, pch, gp, tau, C.byref(sc), C.byref(opts), fptr, tr, _ptr(al),
                                    _ptr(be), C.byref(info), kind)
    elif pc is None:
        st = lib().mlsqr_lsqr_solve(op.h, gp, tau, C.byref(sc), fptr, tr, _ptr(al), _ptr(be), C.byref(info), kind)
    else:
        st = lib().mlsqr_solve(op.h, pc.h, gp, tau, C.byref(sc), fptr, tr, _ptr(al), _ptr(be), C.byref(info), kind)
    _check(st, info)
    trace = [IterationRecord(t.iteration, t.res_damped, t.res_data, bool(t.res_data_exact), t.s2_value,
                             t.anorm_est, t.cond_est, t.xnorm_est, t.alpha, t.beta)
             for t in tr[:info.iterations]]
    left_basis = None
    if basis is not None:
        basis = basis[:info.n_alphas * op.n_cols].reshape(info.n_alphas, op.n_cols)
        left_basis = left[:info.n_left_basis * op.n_rows].reshape(info.n_left_basis, op.n_rows)
    if snaps is not None:
        snaps = snaps[:info.iterations * op.n_cols].reshape(info.iterations, op.n_cols)
    if cgn:
        al, be = np.zeros(0), np.zeros(0)
        info.n_alphas = info.n_betas = 0
    return SolveResult(f, info.iterations, STOP_NAMES[info.stop_reason], trace,
                       al[:info.n_alphas].copy(), be[:info.n_betas].copy(), basis, left_basis, snaps)


def mlsqr(a: LinearOperator, msolver: SpdMap, g, tau: float, stop: StoppingConfig, f_out=None,
          store_basis: bool = False, record_snapshots: bool = False) -> SolveResult:
    """Factorization-free priorconditioned LSQR (krylov.hpp:89-95).  SolveOptions (krylov.hpp:77-80):
    store_basis also returns the right basis vtilde_1..k as `.basis`; record_snapshots the iterate
    after every iteration as `.snapshots`."""
    return _run(a, msolver, g, tau, stop, f_out, store_basis=store_basis, record_snapshots=record_snapshots)


def lsqr(a: LinearOperator, g, tau: float, stop: StoppingConfig, f_out=None,
         store_basis: bool = False, record_snapshots: bool = False) -> SolveResult:
    """Damped LSQR (krylov.hpp:80-87)."""
    return _run(a, None, g, tau, stop, f_out, store_basis=store_basis, record_snapshots=record_snapshots)


def solve_projected(alphas, betas, beta1: float, tau: float) -> np.ndarray:
    """solve_projected (krylov.hpp:124-127): y minimising |[B_k; sqrt(tau) I] y - beta1 e1|
    from a bidiagonalization's k alphas and k+1 betas -- one solve serves every tau."""
    a = np.ascontiguousarray(alphas, dtype=np.float64)
    b = np.ascontiguousarray(betas, dtype=np.float64)
    y = np.zeros(max(a.size, 1))
    _check(lib().mlsqr_solve_projected(_ptr(a), a.size, _ptr(b), b.size, beta1, tau, _ptr(y)))
    return y[:a.size]


def reconstruct_from_basis(basis, y, ctx: Optional[Context] = None, f_out=None):
    """reconstruct_from_basis (krylov.hpp:129-131): f = sum_j y_j basis[j]."""
    ctx = ctx or default_context()
    y = np.ascontiguousarray(y, dtype=np.float64)
    if y.size == 0:
        raise ValueError("no basis vectors were stored")
    if y.size > basis.shape[0]:
        raise DimensionError("more coefficients than basis vectors")
    n = basis.shape[1]
    if _is_dev(basis):
        import torch
        b = basis[:y.size].contiguous()
        f = torch.empty(n, dtype=torch.float64, device=basis.device) if f_out is None else f_out
        _check(lib().mlsqr_reconstruct_from_basis(ctx.h, C.c_void_p(b.data_ptr()), n, _ptr(y), y.size,
                                                  C.c_void_p(f.data_ptr()), DEVICE))
    else:
        b = np.ascontiguousarray(basis[:y.size], dtype=np.float64)
        f = np.zeros(n) if f_out is None else f_out
        _check(lib().mlsqr_reconstruct_from_basis(ctx.h, C.c_void_p(b.ctypes.data), n, _ptr(y), y.size,
                                                  C.c_void_p(f.ctypes.data), HOST))
    return f


def cg_normal(a: LinearOperator, m: Optional["VCycleMap"], tau: float, g, stop: StoppingConfig,
              f_out=None, record_snapshots: bool = False) -> SolveResult:
    """CG on the normal equation (A^T A + tau M) f = A^T g (krylov.hpp:116-122), the
    unpriorconditioned baseline.  M is the level-0 operator of the V-cycle map `m` (None when
    tau == 0).  Argument order follows the reference: (a, m, tau, g, stop)."""
    if m is not None and not isinstance(m, VCycleMap):
        raise ValueError("cg_normal's M comes from a VCycleMap (its level-0 edge operator)")
    return _run(a, m, g, tau, stop, f_out, cgn=True, record_snapshots=record_snapshots)


def krylov_basis(a: LinearOperator, msolver: Optional[SpdMap], m: Optional["VCycleMap"], tau: float, g,
                 k: int):
    """krylov_basis (krylov.hpp:133-145): (vectors [count, n] host array, rank_exhausted) for
    K^{A^T A} (msolver = m = None), K^{A^T A + tau M} (m) or K^{M^-1 A^T A} (msolver)."""
    if m is not None and not isinstance(m, VCycleMap):
        raise ValueError("krylov_basis's M comes from a VCycleMap (its level-0 edge operator)")
    gp, gn, kind, keep = _vec_in(g)
    if gn != a.n_rows:
        raise DimensionError("right-hand side length mismatch")
    out = np.zeros(max(int(k), 1) * a.n_cols)
    cnt, ex = C.c_int(), C.c_int()
    if kind == DEVICE:
        gp = C.c_void_p(np.ascontiguousarray(g.cpu().numpy()).ctypes.data)
    _check(lib().mlsqr_krylov_basis(a.h, msolver.h if msolver is not None else None,
                                    m.h if m is not None else None, tau, gp, int(k),
                                    C.c_void_p(out.ctypes.data), C.byref(cnt), C.byref(ex), HOST))
    return out[:cnt.value * a.n_cols].reshape(cnt.value, a.n_cols), bool(ex.value)


# ---------------------------------------------------------------------------
# penalty / outer loop (penalty.hpp, outer.hpp)
# ---------------------------------------------------------------------------
@dataclass
class PenaltySpec:
    """PenaltySpec (penalty.hpp:14-27)."""
    kind: str = "tikhonov"
    threshold: float = 1.0
    tau: float = 0.0

    @staticmethod
    def tikhonov(tau: float = 0.0):
        return PenaltySpec("tikhonov", 1.0, tau)

    @staticmethod
    def tv_smoothed(threshold: float, tau: float = 0.0):
        return PenaltySpec("tv", threshold, tau)

    @staticmethod
    def perona_malik_log(threshold: float, tau: float = 0.0):
        return PenaltySpec("pm_log", threshold, tau)

    @staticmethod
    def perona_malik_exp(threshold: float, tau: float = 0.0):
        return PenaltySpec("pm_exp", threshold, tau)

    @property
    def kind_code(self) -> int:
        return PEN_KINDS[self.kind]

    def validate(self) -> None:  # penalty.cpp:27-32
        if self.kind_code != 0 and not self.threshold > 0.0:
            raise ValueError("penalty threshold T must be positive")
        if not self.tau >= 0.0:
            raise ValueError("penalty strength tau must be nonnegative")


@dataclass
class OuterConfig:
    """OuterConfig (outer.hpp:13-28) with the V-cycle M^{-1}; rel_decrease_threshold <= 0
    runs a fixed number of outer steps (BASELINE's "K outer x I inner")."""
    tau: float = 0.0
    penalty: PenaltySpec = field(default_factory=PenaltySpec)
    inner_stop: StoppingConfig = field(default_factory=StoppingConfig)
    inner_cap: int = 20
    rel_decrease_threshold: float = 0.15
    max_outer: int = 25
    epsilon: Optional[float] = None
    mg_levels: int = 3
    nu_pre: int = 2
    nu_post: int = 2
    coarse_sweeps: int = 4
    omega: float = 2.0 / 3.0
    spd_mode: str = "vcycle"  # SpdSolverMode: "vcycle" | "cholesky" | "inner_cg" (outer.cpp:64-70)
    k_inner: int = 30

    def _c(self) -> _OuterCfg:
        return _OuterCfg(self.tau, self.penalty.kind_code, self.penalty.threshold, self.inner_stop._c(),
                         self.inner_cap, self.rel_decrease_threshold, self.max_outer,
                         -1.0 if self.epsilon is None else self.epsilon, self.mg_levels, self.nu_pre,
                         self.nu_post, self.coarse_sweeps, self.omega, SPD_MODES[self.spd_mode], self.k_inner)


@dataclass
class OuterStep:
    k: int
    penalty_value: float
    inner_iterations: int
    final_residual: float
    inner_stop: str
    eps_used: float
    alphas: np.ndarray
    betas: np.ndarray


@dataclass
class OuterReport:
    solution: object
    steps: list
    stop_reason: str
    triggered_at: int


def solve_nonlinear(a: LinearOperator, g, grid_shape, h: float, cfg: OuterConfig, f_out=None) -> OuterReport:
    """Lagged-diffusivity fixed point, priorconditioned (outer.hpp:52-62)."""
    cfg.penalty.validate()
    gp, gn, kind, keep = _vec_in(g)
    if gn != a.n_rows:
        raise DimensionError("data length mismatch")
    shape = tuple(int(s) for s in grid_shape)
    nx, ny, nz = (list(shape) + [1, 1])[:3]
    steps = (_OuterStep * cfg.max_outer)()
    ns, sr, trig = C.c_int(), C.c_int(), C.c_int()
    al = np.zeros(cfg.max_outer * (cfg.inner_cap + 1))
    be = np.zeros(cfg.max_outer * (cfg.inner_cap + 2))
    if kind == DEVICE:
        import torch
        f = torch.empty(a.n_cols, dtype=torch.float64, device=g.device) if f_out is None else f_out
        fptr = C.c_void_p(f.data_ptr())
    else:
        f = np.zeros(a.n_cols) if f_out is None else f_out
        fptr = C.c_void_p(f.ctypes.data)
    c = cfg._c()
    _check(lib().mlsqr_nonlinear_solve(a.h, gp, len(shape), nx, ny, nz, h, C.byref(c), fptr, steps,
                                       C.byref(ns), C.byref(sr), C.byref(trig), _ptr(al), _ptr(be), kind))
    al = al.reshape(cfg.max_outer, cfg.inner_cap + 1)
    be = be.reshape(cfg.max_outer, cfg.inner_cap + 2)
    out = []
    for i in range(ns.value):
        s = steps[i]
        out.append(OuterStep(s.k, s.penalty_value, s.inner_iterations, s.final_residual,
                             STOP_NAMES[s.inner_stop], s.eps_used, al[i].copy(), be[i].copy()))
    return OuterReport(f, out, "stagnation" if sr.value == 0 else "max_outer", trig.value)


class OuterSolver:
    """One lagged-diffusivity outer step per call (outer.cpp:59-87) with the V-cycle
    hierarchy and Krylov workspace kept resident: step(g, f_prev, f_out)."""

    def __init__(self, a: LinearOperator, grid_shape, h: float, cfg: OuterConfig):
        cfg.penalty.validate()
        shape = tuple(int(s) for s in grid_shape)
        nx, ny, nz = (list(shape) + [1, 1])[:3]
        self._cfg = cfg._c()
        hh = C.c_void_p()
        _check(lib().mlsqr_outer_create(a.h, len(shape), nx, ny, nz, h, C.byref(self._cfg), C.byref(hh)))
        self.h, self.op = hh, a

    def step(self, g, f_prev, f_out) -> OuterStep:
        gp, gn, kind, k1 = _vec_in(g)
        pp, pn, kind2, k2 = _vec_in(f_prev)
        op_, on, kind3, k3 = _vec_in(f_out)
        assert kind == kind2 == kind3, "g, f_prev, f_out must all be host or all device"
        if kind == HOST:  # the C-ABI writes f_out in place
            op_ = C.c_void_p(f_out.ctypes.data)
        s = _OuterStep()
        _check(lib().mlsqr_outer_advance(self.h, gp, pp, op_, C.byref(s), kind))
        cap = self._cfg.inner_cap + 2
        al, be = np.zeros(cap), np.zeros(cap)
        na, nb = C.c_int(), C.c_int()
        _check(lib().mlsqr_outer_last_bidiag(self.h, _ptr(al), cap, _ptr(be), cap, C.byref(na), C.byref(nb)))
        return OuterStep(s.k, s.penalty_value, s.inner_iterations, s.final_residual,
                         STOP_NAMES[s.inner_stop], s.eps_used, al[:na.value].copy(), be[:nb.value].copy())

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().mlsqr_outer_destroy(self.h)
        except Exception:
            pass


def penalty_functional(f, grid_shape, h: float, penalty: PenaltySpec, ctx: Optional[Context] = None) -> float:
    """R(f) = sum_e w_e r(|d_e|) on the device (diffusion.cpp:89-101)."""
    ctx = ctx or default_context()
    fp, fn, kind, keep = _vec_in(f)
    shape = tuple(int(s) for s in grid_shape)
    nx, ny, nz = (list(shape) + [1, 1])[:3]
    v = C.c_double()
    _check(lib().mlsqr_penalty_functional(ctx.h, len(shape), nx, ny, nz, h, fp, kind, penalty.kind_code,
                                          penalty.threshold, C.byref(v)))
    return v.value


# ---------------------------------------------------------------------------
# seeded inputs (host generators of the library)
# ---------------------------------------------------------------------------
def gaussian_taps(n: int, sigma_f: float, radius: int = -1, domain_length: float = 1.0) -> np.ndarray:
    R = C.c_int()
    _check(lib().mlsqr_taps(n, sigma_f, domain_length, radius, None, C.byref(R)))
    t = np.zeros(2 * R.value + 1)
    _check(lib().mlsqr_taps(n, sigma_f, domain_length, R.value, _ptr(t), C.byref(R)))
    return t


def gaussian_noise(seed: int, n: int, stddev: float = 1.0) -> np.ndarray:
    out = np.zeros(n)
    _check(lib().mlsqr_gauss_fill(seed, n, stddev, _ptr(out)))
    return out


def phantom_rects2d(nx, ny, count, seed):
    out = np.zeros(nx * ny)
    _check(lib().mlsqr_phantom_rects2d(nx, ny, count, seed, _ptr(out)))
    return out


def phantom_shapes2d(nx, ny, count, seed):
    out = np.zeros(nx * ny)
    _check(lib().mlsqr_phantom_shapes2d(nx, ny, count, seed, _ptr(out)))
    return out


def phantom_ellipsoids3d(nx, ny, nz, count, semi_lo, semi_hi, vlo, vhi, seed):
    out = np.zeros(nx * ny * nz)
    _check(lib().mlsqr_phantom_ellipsoids3d(nx, ny, nz, count, semi_lo, semi_hi, vlo, vhi, seed, _ptr(out)))
    return out


def fdot_tables(n, n_src, n_det, mu, seed):
    N = n ** 3
    gs, gd = np.zeros(n_src * N), np.zeros(n_det * N)
    _check(lib().mlsqr_fdot_tables(n, n_src, n_det, mu, seed, _ptr(gs), _ptr(gd)))
    return gs, gd
