"""oracle/pyoracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes bindings for the C restatement (oracle/liborc.so) and for the
reference shim (oracle/_ref/libmlsqr_ref.so, the unmodified reference core).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libmlsqr_ref.so")

dp = C.POINTER(C.c_double)
VEC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, dp, dp)

PEN = {"tikhonov": 0, "tv": 1, "pm_log": 2, "pm_exp": 3}
STOP_NAMES = ["S1", "S2", "S3", "S4", "max_iters", "breakdown"]


def build(ref: bool = True) -> None:
    targets = ["all"] + (["ref"] if ref and os.path.isdir("/root/reference/proj/src") else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _ptr(a):
    return a.ctypes.data_as(dp) if a is not None else None


class Stop(C.Structure):
    _fields_ = [("atol", C.c_double), ("btol", C.c_double), ("conlim", C.c_double),
                ("delta", C.c_double), ("eta", C.c_double), ("max_iters", C.c_int),
                ("use_s1", C.c_int), ("use_s2", C.c_int), ("use_s3", C.c_int),
                ("use_s4", C.c_int)]


def stop(max_iters=100, atol=1e-8, btol=1e-8, conlim=1e8, delta=0.0, eta=1.1, s1=False,
         s2=False, s3=False, s4=False) -> Stop:
    return Stop(atol, btol, conlim, delta, eta, max_iters, int(s1), int(s2), int(s3), int(s4))


class IterRec(C.Structure):
    _fields_ = [("iteration", C.c_int), ("res_data_exact", C.c_int), ("res_damped", C.c_double),
                ("res_data", C.c_double), ("s2_value", C.c_double), ("anorm_est", C.c_double),
                ("cond_est", C.c_double), ("xnorm_est", C.c_double), ("alpha", C.c_double),
                ("beta", C.c_double)]


class SolveInfo(C.Structure):
    _fields_ = [("iterations", C.c_int), ("stop_reason", C.c_int), ("n_alphas", C.c_int),
                ("n_betas", C.c_int), ("breakdown_iteration", C.c_int)]


class Grid(C.Structure):
    _fields_ = [("dims", C.c_int), ("nx", C.c_size_t), ("ny", C.c_size_t), ("nz", C.c_size_t),
                ("h", C.c_double)]


class OuterCfg(C.Structure):
    _fields_ = [("tau", C.c_double), ("pen_kind", C.c_int), ("T", C.c_double),
                ("inner_stop", Stop), ("inner_cap", C.c_int),
                ("rel_decrease_threshold", C.c_double), ("max_outer", C.c_int),
                ("epsilon", C.c_double), ("mg_levels", C.c_int), ("nu_pre", C.c_int),
                ("nu_post", C.c_int), ("coarse_sweeps", C.c_int), ("omega", C.c_double),
                ("spd_mode", C.c_int), ("k_inner", C.c_int)]


class OuterStep(C.Structure):
    _fields_ = [("k", C.c_int), ("inner_iterations", C.c_int), ("inner_stop", C.c_int),
                ("penalty_value", C.c_double), ("final_residual", C.c_double),
                ("eps_used", C.c_double)]


@dataclass
class SolveOut:
    f: np.ndarray
    iterations: int
    stop_reason: str
    alphas: np.ndarray
    betas: np.ndarray
    trace: list
    status: int = 0
    breakdown_iteration: int = 0
    snapshots: np.ndarray | None = None


def _trace_list(arr, k):
    return [{f[0]: getattr(arr[i], f[0]) for f in IterRec._fields_} for i in range(k)]


# ---------------------------------------------------------------------------
# restatement (liborc.so)
# ---------------------------------------------------------------------------
class Oracle:
    def __init__(self, path: str = ORC_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_uniform.restype = C.c_double
        L.orc_mt64_next.restype = C.c_uint64
        L.orc_r_value.restype = C.c_double
        L.orc_r_value.argtypes = [C.c_int, C.c_double, C.c_double]
        L.orc_diffusivity.restype = C.c_double
        L.orc_diffusivity.argtypes = [C.c_int, C.c_double, C.c_double]
        L.orc_taps.argtypes = [C.c_size_t, C.c_double, C.c_double, C.c_int, dp]
        L.orc_gauss_fill.argtypes = [C.c_uint64, C.c_size_t, C.c_double, dp]
        for name in ("orc_identity_new",):
            getattr(L, name).restype = C.c_void_p
            getattr(L, name).argtypes = [C.c_size_t]
        L.orc_dense_new.restype = C.c_void_p
        L.orc_dense_new.argtypes = [C.c_size_t, C.c_size_t, dp]
        L.orc_blur_new.restype = C.c_void_p
        L.orc_blur_new.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, dp]
        L.orc_linop_free.argtypes = [C.c_void_p]
        L.orc_linop_apply.argtypes = [C.c_void_p, dp, dp]
        L.orc_linop_adjoint.argtypes = [C.c_void_p, dp, dp]
        L.orc_edge_coeffs.argtypes = [C.POINTER(Grid), dp, C.c_int, C.c_double, dp, dp, dp]
        L.orc_max_diag.restype = C.c_double
        L.orc_max_diag.argtypes = [C.POINTER(Grid), dp, dp, dp]
        L.orc_m_apply.argtypes = [C.POINTER(Grid), dp, dp, dp, C.c_double, dp, dp]
        L.orc_penalty_functional.restype = C.c_double
        L.orc_penalty_functional.argtypes = [C.POINTER(Grid), dp, C.c_int, C.c_double]
        L.orc_identity_map_new.restype = C.c_void_p
        L.orc_identity_map_new.argtypes = [C.c_size_t]
        L.orc_dense_chol_map_new.restype = C.c_void_p
        L.orc_dense_chol_map_new.argtypes = [C.c_size_t, dp]
        L.orc_env_chol_map_new.restype = C.c_void_p
        L.orc_env_chol_map_new.argtypes = [C.POINTER(Grid), dp, dp, dp, C.c_double, C.POINTER(C.c_longlong)]
        L.orc_inner_cg_map_new.restype = C.c_void_p
        L.orc_inner_cg_map_new.argtypes = [C.POINTER(Grid), dp, dp, dp, C.c_double, C.c_int]
        L.orc_krylov_basis.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(Grid), dp, dp, dp, C.c_double,
                                        C.c_double, dp, C.c_int, dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_vcycle_new.restype = C.c_void_p
        L.orc_vcycle_new.argtypes = [C.POINTER(Grid), C.c_int, C.c_int, C.c_int, C.c_double, C.c_int]
        L.orc_vcycle_set.argtypes = [C.c_void_p, dp, dp, dp, C.c_double]
        L.orc_map_free.argtypes = [C.c_void_p]
        L.orc_vcycle_level.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_size_t), dp, dp, dp, dp]
        L.orc_set_device_order.argtypes = [C.c_int]
        L.orc_canon_dot.restype = C.c_double
        L.orc_canon_dot.argtypes = [dp, dp, C.c_size_t, C.c_size_t]
        L.orc_dhypot.restype = C.c_double
        L.orc_dhypot.argtypes = [C.c_double, C.c_double]
        L.orc_linop_set_row_lengths.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t]
        L.orc_map_solve.argtypes = [C.c_void_p, dp, dp]
        L.orc_mlsqr.argtypes = [C.c_void_p, C.c_void_p, dp, C.c_double, C.POINTER(Stop), dp,
                                C.POINTER(IterRec), dp, dp, dp, C.POINTER(SolveInfo)]
        L.orc_cg_normal.argtypes = [C.c_void_p, C.POINTER(Grid), dp, dp, dp, C.c_double, C.c_double, dp,
                                    C.POINTER(Stop), dp, C.POINTER(IterRec), C.POINTER(SolveInfo)]
        L.orc_lsqr.argtypes = [C.c_void_p, dp, C.c_double, C.POINTER(Stop), dp,
                               C.POINTER(IterRec), dp, dp, dp, C.POINTER(SolveInfo)]
        L.orc_nonlinear.argtypes = [C.c_void_p, dp, C.POINTER(Grid), C.POINTER(OuterCfg), dp,
                                    C.POINTER(OuterStep), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int), dp, dp, dp]
        L.orc_outer_stop_check.argtypes = [dp, C.c_int, C.c_double]
        L.orc_phantom_rects2d.argtypes = [C.c_size_t, C.c_size_t, C.c_int, C.c_uint64, dp]
        L.orc_phantom_shapes2d.argtypes = [C.c_size_t, C.c_size_t, C.c_int, C.c_uint64, dp]
        L.orc_phantom_ellipsoids3d.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, C.c_int,
                                               C.c_double, C.c_double, C.c_double, C.c_double,
                                               C.c_uint64, dp]
        L.orc_fdot_tables.argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_double, C.c_uint64, dp, dp]
        L.orc_fdot_matrix.argtypes = [C.c_size_t, C.c_int, C.c_int, dp, dp, dp]
        self.apply_cb = C.cast(L.orc_linop_apply_cb, C.c_void_p).value
        self.adjoint_cb = C.cast(L.orc_linop_adjoint_cb, C.c_void_p).value
        self.solve_cb = C.cast(L.orc_map_solve_cb, C.c_void_p).value

    # -- arithmetic order
    def set_device_order(self, on: bool) -> None:
        self.lib.orc_set_device_order(int(on))

    def device_order(self):
        return _DeviceOrder(self)

    def canon_dot(self, x, y, row_len):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        return self.lib.orc_canon_dot(_ptr(x), _ptr(y), x.size, row_len)

    # -- generators
    def taps(self, n, sigma_f, radius=-1, domain_length=1.0):
        R = self.lib.orc_taps(n, sigma_f, domain_length, radius, None)
        t = np.zeros(2 * R + 1)
        self.lib.orc_taps(n, sigma_f, domain_length, R, _ptr(t))
        return t

    def gauss(self, seed, n, stddev=1.0):
        out = np.zeros(n)
        self.lib.orc_gauss_fill(seed, n, stddev, _ptr(out))
        return out

    def uniforms(self, seed, n):
        st = (C.c_uint64 * 313)()
        self.lib.orc_mt64_seed(C.byref(st), C.c_uint64(seed))
        return np.array([self.lib.orc_uniform(C.byref(st)) for _ in range(n)])

    def rects2d(self, nx, ny, count, seed):
        out = np.zeros(nx * ny)
        self.lib.orc_phantom_rects2d(nx, ny, count, seed, _ptr(out))
        return out

    def shapes2d(self, nx, ny, count, seed):
        out = np.zeros(nx * ny)
        self.lib.orc_phantom_shapes2d(nx, ny, count, seed, _ptr(out))
        return out

    def ellipsoids3d(self, nx, ny, nz, count, semi_lo, semi_hi, vlo, vhi, seed):
        out = np.zeros(nx * ny * nz)
        self.lib.orc_phantom_ellipsoids3d(nx, ny, nz, count, semi_lo, semi_hi, vlo, vhi, seed,
                                          _ptr(out))
        return out

    def fdot(self, n, n_src, n_det, mu, seed):
        N = n ** 3
        gs = np.zeros(n_src * N)
        gd = np.zeros(n_det * N)
        self.lib.orc_fdot_tables(n, n_src, n_det, mu, seed, _ptr(gs), _ptr(gd))
        a = np.zeros(n_src * n_det * N)
        self.lib.orc_fdot_matrix(N, n_src, n_det, _ptr(gs), _ptr(gd), _ptr(a))
        return gs, gd, a.reshape(n_src * n_det, N)

    # -- penalty
    def diffusivity(self, kind, T, t):
        return self.lib.orc_diffusivity(PEN.get(kind, kind), T, t)

    def r_value(self, kind, T, t):
        return self.lib.orc_r_value(PEN.get(kind, kind), T, t)

    # -- operators
    def blur(self, dims, shape, taps):
        nx, ny, nz = (list(shape) + [1, 1])[:3]
        taps = np.ascontiguousarray(taps, dtype=np.float64)
        return OrcOp(self, self.lib.orc_blur_new(dims, nx, ny, nz, (len(taps) - 1) // 2, _ptr(taps)),
                     nx * ny * nz, nx * ny * nz)

    def dense(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        op = OrcOp(self, self.lib.orc_dense_new(a.shape[0], a.shape[1], _ptr(a)), a.shape[0], a.shape[1])
        op._keep = a
        return op

    def identity(self, n):
        return OrcOp(self, self.lib.orc_identity_new(n), n, n)

    # -- M
    @staticmethod
    def grid(dims, shape, h):
        nx, ny, nz = (list(shape) + [1, 1])[:3]
        return Grid(dims, nx, ny, nz, h)

    def edge_coeffs(self, grid, f, kind, T):
        n = grid.nx * grid.ny * grid.nz
        cx, cy, cz = np.zeros(n), np.zeros(n), np.zeros(n)
        f = np.ascontiguousarray(f, dtype=np.float64)
        st = self.lib.orc_edge_coeffs(C.byref(grid), _ptr(f), PEN.get(kind, kind), T, _ptr(cx), _ptr(cy), _ptr(cz))
        assert st == 0, st
        return cx, cy, cz

    def max_diag(self, grid, cx, cy, cz):
        return self.lib.orc_max_diag(C.byref(grid), _ptr(cx), _ptr(cy), _ptr(cz))

    def m_apply(self, grid, cx, cy, cz, eps, x):
        y = np.zeros_like(x)
        self.lib.orc_m_apply(C.byref(grid), _ptr(cx), _ptr(cy), _ptr(cz), eps,
                             _ptr(np.ascontiguousarray(x)), _ptr(y))
        return y

    def penalty_functional(self, grid, f, kind, T):
        return self.lib.orc_penalty_functional(C.byref(grid), _ptr(np.ascontiguousarray(f)),
                                               PEN.get(kind, kind), T)

    # -- maps
    def vcycle(self, grid, levels, nu_pre=2, nu_post=2, omega=2.0 / 3.0, coarse_sweeps=4):
        h = self.lib.orc_vcycle_new(C.byref(grid), levels, nu_pre, nu_post, omega, coarse_sweeps)
        if not h:
            raise ValueError("invalid V-cycle configuration")
        return OrcMap(self, h, grid.nx * grid.ny * grid.nz)

    def identity_map(self, n):
        return OrcMap(self, self.lib.orc_identity_map_new(n), n)

    def chol_map(self, m_dense):
        m_dense = np.ascontiguousarray(m_dense, dtype=np.float64)
        h = self.lib.orc_dense_chol_map_new(m_dense.shape[0], _ptr(m_dense))
        if not h:
            raise ValueError("matrix not SPD")
        return OrcMap(self, h, m_dense.shape[0])

    def env_chol_map(self, grid, cx, cy, cz, eps):
        """SpdSolver::factorize over the stencil M (spdsolve.cpp:22-75); ValueError(pivot row)."""
        row = C.c_longlong(-1)
        n = grid.nx * grid.ny * grid.nz
        h = self.lib.orc_env_chol_map_new(C.byref(grid), _ptr(cx), _ptr(cy), _ptr(cz), eps, C.byref(row))
        if not h:
            raise ValueError(f"nonpositive pivot at row {row.value}")
        return OrcMap(self, h, n)

    def inner_cg_map(self, grid, cx, cy, cz, eps, k_inner):
        """SpdSolver::inner_cg (spdsolve.cpp:77-85, 119-137)."""
        n = grid.nx * grid.ny * grid.nz
        h = self.lib.orc_inner_cg_map_new(C.byref(grid), _ptr(cx), _ptr(cy), _ptr(cz), eps, k_inner)
        if not h:
            raise ValueError("invalid inner-CG configuration")
        return OrcMap(self, h, n)

    def krylov_basis(self, op, msolver, k, g, tau=0.0, m=None):
        """krylov_basis (krylov.cpp:700-754); m = (grid, cx, cy, cz, eps) for K^{A^T A + tau M}."""
        g = np.ascontiguousarray(g, dtype=np.float64)
        out = np.zeros(k * op.cols)
        cnt, ex = C.c_int(), C.c_int()
        if m is not None:
            grid, cx, cy, cz, eps = m
            st = self.lib.orc_krylov_basis(op.h, None, C.byref(grid), _ptr(cx), _ptr(cy), _ptr(cz), eps, tau,
                                           _ptr(g), k, _ptr(out), C.byref(cnt), C.byref(ex))
        else:
            st = self.lib.orc_krylov_basis(op.h, msolver.h if msolver is not None else None, None, None, None,
                                           None, 0.0, tau, _ptr(g), k, _ptr(out), C.byref(cnt), C.byref(ex))
        assert st == 0, st
        return out[:cnt.value * op.cols].reshape(cnt.value, op.cols), bool(ex.value)

    # -- solvers
    def mlsqr(self, op, pc, g, tau, st, snapshots=False, lsqr=False):
        g = np.ascontiguousarray(g, dtype=np.float64)
        n = op.cols
        k = st.max_iters
        f = np.zeros(n)
        tr = (IterRec * k)()
        al = np.zeros(k + 1)
        be = np.zeros(k + 2)
        snap = np.zeros(k * n) if snapshots else None
        info = SolveInfo()
        if lsqr:
            status = self.lib.orc_lsqr(op.h, _ptr(g), tau, C.byref(st), _ptr(f), tr, _ptr(al),
                                       _ptr(be), _ptr(snap), C.byref(info))
        else:
            status = self.lib.orc_mlsqr(op.h, pc.h, _ptr(g), tau, C.byref(st), _ptr(f), tr,
                                        _ptr(al), _ptr(be), _ptr(snap), C.byref(info))
        return SolveOut(f, info.iterations, STOP_NAMES[info.stop_reason], al[:info.n_alphas].copy(),
                        be[:info.n_betas].copy(), _trace_list(tr, info.iterations), status,
                        info.breakdown_iteration,
                        snap.reshape(k, n)[:info.iterations] if snapshots else None)

    def cg_normal(self, op, grid, cx, cy, cz, eps, tau, g, st):
        """orc_cg_normal (krylov.cpp:551-628); M = edge operator (cx, cy, cz) + eps I."""
        g = np.ascontiguousarray(g, dtype=np.float64)
        k = st.max_iters
        f = np.zeros(op.cols)
        tr = (IterRec * k)()
        info = SolveInfo()
        z = np.zeros(op.cols)
        cy = z if cy is None else cy
        cz = z if cz is None else cz
        status = self.lib.orc_cg_normal(op.h, C.byref(grid), _ptr(cx), _ptr(cy), _ptr(cz), eps, tau, _ptr(g),
                                        C.byref(st), _ptr(f), tr, C.byref(info))
        return SolveOut(f, info.iterations, STOP_NAMES[info.stop_reason], np.zeros(0), np.zeros(0),
                        _trace_list(tr, info.iterations), status, info.breakdown_iteration, None)

    def nonlinear(self, op, g, grid, *, tau, pen, T, inner_stop, inner_cap, max_outer,
                  threshold=0.0, epsilon=-1.0, levels=3, nu_pre=2, nu_post=2, coarse_sweeps=4,
                  omega=2.0 / 3.0, keep=False, spd_mode=0, k_inner=30):
        cfg = OuterCfg(tau, PEN.get(pen, pen), T, inner_stop, inner_cap, threshold, max_outer,
                       epsilon, levels, nu_pre, nu_post, coarse_sweeps, omega, spd_mode, k_inner)
        n = op.cols
        f = np.zeros(n)
        steps = (OuterStep * max_outer)()
        ns, sr, trig = C.c_int(), C.c_int(), C.c_int()
        al = np.zeros(max_outer * (inner_cap + 1))
        be = np.zeros(max_outer * (inner_cap + 2))
        it = np.zeros(max_outer * n) if keep else None
        g = np.ascontiguousarray(g, dtype=np.float64)
        status = self.lib.orc_nonlinear(op.h, _ptr(g), C.byref(grid), C.byref(cfg), _ptr(f), steps,
                                        C.byref(ns), C.byref(sr), C.byref(trig), _ptr(al), _ptr(be),
                                        _ptr(it))
        return {
            "status": status, "f": f, "n_steps": ns.value,
            "stop_reason": "stagnation" if sr.value == 0 else "max_outer",
            "triggered_at": trig.value,
            "steps": [{fl[0]: getattr(steps[i], fl[0]) for fl in OuterStep._fields_} for i in range(ns.value)],
            "alphas": al.reshape(max_outer, inner_cap + 1)[:ns.value],
            "betas": be.reshape(max_outer, inner_cap + 2)[:ns.value],
            "iterates": it.reshape(max_outer, n)[:ns.value] if keep else None,
        }


class _DeviceOrder:
    def __init__(self, orc):
        self.orc = orc

    def __enter__(self):
        self.orc.set_device_order(True)
        return self.orc

    def __exit__(self, *a):
        self.orc.set_device_order(False)


class OrcOp:
    def __init__(self, orc, h, rows, cols):
        self.orc, self.h, self.rows, self.cols = orc, h, rows, cols

    def set_row_lengths(self, data_len, sol_len):
        self.orc.lib.orc_linop_set_row_lengths(self.h, data_len, sol_len)
        return self

    def apply(self, x):
        y = np.zeros(self.rows)
        self.orc.lib.orc_linop_apply(self.h, _ptr(np.ascontiguousarray(x, dtype=np.float64)), _ptr(y))
        return y

    def adjoint(self, y):
        x = np.zeros(self.cols)
        self.orc.lib.orc_linop_adjoint(self.h, _ptr(np.ascontiguousarray(y, dtype=np.float64)), _ptr(x))
        return x

    def __del__(self):
        try:
            self.orc.lib.orc_linop_free(self.h)
        except Exception:
            pass


class OrcMap:
    def __init__(self, orc, h, n):
        self.orc, self.h, self.n = orc, h, n

    def set(self, cx, cy, cz, eps):
        st = self.orc.lib.orc_vcycle_set(self.h, _ptr(cx), _ptr(cy), _ptr(cz), eps)
        assert st == 0

    def level(self, l):
        d = (C.c_size_t * 3)()
        self.orc.lib.orc_vcycle_level(self.h, l, d, None, None, None, None)
        n = d[0] * d[1] * d[2]
        cx, cy, cz, e = np.zeros(n), np.zeros(n), np.zeros(n), C.c_double()
        self.orc.lib.orc_vcycle_level(self.h, l, d, _ptr(cx), _ptr(cy), _ptr(cz), C.byref(e))
        return (d[0], d[1], d[2]), cx, cy, cz, e.value

    def solve(self, p):
        v = np.zeros(self.n)
        self.orc.lib.orc_map_solve(self.h, _ptr(np.ascontiguousarray(p, dtype=np.float64)), _ptr(v))
        return v

    def __del__(self):
        try:
            self.orc.lib.orc_map_free(self.h)
        except Exception:
            pass


# ---------------------------------------------------------------------------
# the reference itself (oracle/_ref/libmlsqr_ref.so)
# ---------------------------------------------------------------------------
class RefOp(C.Structure):
    _fields_ = [("kind", C.c_int), ("rows", C.c_size_t), ("cols", C.c_size_t), ("a", dp),
                ("nx", C.c_size_t), ("ny", C.c_size_t), ("sigma", C.c_double),
                ("apply", C.c_void_p), ("adjoint", C.c_void_p), ("ctx", C.c_void_p)]


class RefMap(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_size_t), ("m", dp), ("dims", C.c_int),
                ("nx", C.c_size_t), ("ny", C.c_size_t), ("h", C.c_double), ("f", dp),
                ("pen_kind", C.c_int), ("T", C.c_double), ("eps", C.c_double),
                ("k_inner", C.c_int), ("solve", C.c_void_p), ("ctx", C.c_void_p)]


class RefOuterCfg(C.Structure):
    _fields_ = [("tau", C.c_double), ("pen_kind", C.c_int), ("T", C.c_double),
                ("inner_stop", Stop), ("inner_cap", C.c_int),
                ("rel_decrease_threshold", C.c_double), ("max_outer", C.c_int),
                ("spd_mode", C.c_int), ("k_inner", C.c_int), ("epsilon", C.c_double)]


class Reference:
    """The unmodified reference core (needs oracle/_ref, built from /root/reference)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle ref` where /root/reference exists)")
        L = self.lib = C.CDLL(path)
        L.ref_taps.argtypes = [C.c_size_t, C.c_double, dp, C.POINTER(C.c_int)]
        L.ref_op_apply.argtypes = [C.POINTER(RefOp), dp, dp]
        L.ref_op_adjoint.argtypes = [C.POINTER(RefOp), dp, dp]
        L.ref_diffusivity.restype = C.c_double
        L.ref_diffusivity.argtypes = [C.c_int, C.c_double, C.c_double]
        L.ref_r_value.restype = C.c_double
        L.ref_r_value.argtypes = [C.c_int, C.c_double, C.c_double]
        L.ref_assemble_m_dense.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_double, dp, C.c_int,
                                           C.c_double, C.c_double, dp, dp]
        L.ref_m_multiply.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_double, dp, C.c_int,
                                     C.c_double, C.c_double, dp, dp]
        L.ref_penalty_functional.restype = C.c_double
        L.ref_penalty_functional.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_double, dp, C.c_int, C.c_double]
        L.ref_gauss_fill.argtypes = [C.c_uint64, C.c_size_t, C.c_double, dp]
        L.ref_mlsqr.argtypes = [C.POINTER(RefOp), C.POINTER(RefMap), dp, C.c_double, C.POINTER(Stop),
                                C.c_int, dp, C.POINTER(IterRec), dp, dp, dp, C.POINTER(SolveInfo)]
        L.ref_solve_projected.argtypes = [dp, C.c_size_t, dp, C.c_size_t, C.c_double, C.c_double, dp]
        L.ref_cg_normal.argtypes = [C.POINTER(RefOp), C.c_int, C.c_size_t, C.c_size_t, C.c_double, dp, C.c_int,
                                    C.c_double, C.c_double, C.c_double, dp, C.POINTER(Stop), dp,
                                    C.POINTER(IterRec), C.POINTER(SolveInfo)]
        L.ref_lsqr.argtypes = [C.POINTER(RefOp), dp, C.c_double, C.POINTER(Stop), C.c_int, dp,
                               C.POINTER(IterRec), dp, dp, dp, C.POINTER(SolveInfo)]
        L.ref_solve_nonlinear.argtypes = [C.POINTER(RefOp), dp, C.c_int, C.c_size_t, C.c_size_t,
                                          C.c_double, C.POINTER(RefOuterCfg), dp, C.POINTER(OuterStep),
                                          C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), dp]
        L.ref_mlsqr_timed.argtypes = [C.POINTER(RefOp), C.POINTER(RefMap), dp, C.c_double,
                                      C.POINTER(Stop), C.c_int, dp, dp, C.POINTER(SolveInfo)]
        L.ref_select_backend.argtypes = [C.c_int]
        L.ref_krylov_basis.argtypes = [C.POINTER(RefOp), C.POINTER(RefMap), C.c_int, C.c_int, C.c_size_t,
                                       C.c_size_t, C.c_double, dp, C.c_int, C.c_double, C.c_double, C.c_double,
                                       dp, C.c_int, dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_map_solve.argtypes = [C.POINTER(RefMap), dp, dp]
        L.ref_kernel_backend.restype = C.c_char_p
        self._keep = []

    def select_backend(self, scalar: bool) -> bool:
        return self.lib.ref_select_backend(int(scalar)) == 0

    def backend(self) -> str:
        return self.lib.ref_kernel_backend().decode()

    # operator descriptors
    def op_identity(self, n):
        return RefOp(0, n, n, None, 0, 0, 0.0, None, None, None)

    def op_dense(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        self._keep.append(a)
        return RefOp(1, a.shape[0], a.shape[1], _ptr(a), 0, 0, 0.0, None, None, None)

    def op_conv1d(self, n, sigma):
        return RefOp(2, n, n, None, n, 1, sigma, None, None, None)

    def op_blur2d(self, nx, ny, sigma):
        return RefOp(3, nx * ny, nx * ny, None, nx, ny, sigma, None, None, None)

    def op_callback(self, rows, cols, apply_fn, adjoint_fn, ctx):
        return RefOp(4, rows, cols, None, 0, 0, 0.0, apply_fn, adjoint_fn, ctx)

    # maps
    def map_identity(self, n):
        return RefMap(kind=0, n=n)

    def map_chol_dense(self, m):
        m = np.ascontiguousarray(m, dtype=np.float64)
        self._keep.append(m)
        return RefMap(kind=1, n=m.shape[0], m=_ptr(m))

    def map_assembled(self, dims, shape, h, f, pen, T, eps=-1.0, inner_cg=0):
        f = np.ascontiguousarray(f, dtype=np.float64)
        self._keep.append(f)
        nx, ny = (list(shape) + [1])[:2]
        return RefMap(kind=3 if inner_cg else 2, n=nx * ny, dims=dims, nx=nx, ny=ny, h=h, f=_ptr(f),
                      pen_kind=PEN.get(pen, pen), T=T, eps=eps, k_inner=inner_cg)

    def map_callback(self, n, fn, ctx):
        return RefMap(kind=4, n=n, solve=fn, ctx=ctx)

    def krylov_basis(self, od, cols, k, g, tau=0.0, md=None, m=None):
        """krylov_basis; md: a map descriptor (priorconditioned space); m = (dims, shape, h, f, pen,
        T, eps) for K^{A^T A + tau M}."""
        g = np.ascontiguousarray(g, dtype=np.float64)
        out = np.zeros(k * cols)
        cnt, ex = C.c_int(), C.c_int()
        if m is not None:
            dims, shape, h, f, pen, T, eps = m
            nx, ny = (list(shape) + [1])[:2]
            f = np.ascontiguousarray(f, dtype=np.float64)
            args = (None, 1, dims, nx, ny, h, _ptr(f), PEN.get(pen, pen), T, eps)
        else:
            args = (C.byref(md) if md is not None else None, 0, 1, 0, 0, 0.0, None, 0, 0.0, -1.0)
        st = self.lib.ref_krylov_basis(C.byref(od), *args, tau, _ptr(g), k, _ptr(out), C.byref(cnt), C.byref(ex))
        assert st == 0, st
        return out[:cnt.value * cols].reshape(cnt.value, cols), bool(ex.value)

    def map_solve(self, md, p):
        """One SpdMap::solve of a freshly built reference map."""
        v = np.zeros(md.n)
        st = self.lib.ref_map_solve(C.byref(md), _ptr(np.ascontiguousarray(p, dtype=np.float64)), _ptr(v))
        assert st == 0, st
        return v

    def taps(self, n, sigma):
        R = C.c_int()
        self.lib.ref_taps(n, sigma, None, C.byref(R))
        t = np.zeros(2 * R.value + 1)
        self.lib.ref_taps(n, sigma, _ptr(t), C.byref(R))
        return t

    def apply(self, od, x, rows):
        y = np.zeros(rows)
        st = self.lib.ref_op_apply(C.byref(od), _ptr(np.ascontiguousarray(x, dtype=np.float64)), _ptr(y))
        assert st == 0, st
        return y

    def adjoint(self, od, y, cols):
        x = np.zeros(cols)
        st = self.lib.ref_op_adjoint(C.byref(od), _ptr(np.ascontiguousarray(y, dtype=np.float64)), _ptr(x))
        assert st == 0, st
        return x

    def diffusivity(self, kind, T, t):
        return self.lib.ref_diffusivity(PEN.get(kind, kind), T, t)

    def r_value(self, kind, T, t):
        return self.lib.ref_r_value(PEN.get(kind, kind), T, t)

    def assemble_dense(self, dims, shape, h, f, kind, T, eps=-1.0):
        nx, ny = (list(shape) + [1])[:2]
        n = nx * ny
        out = np.zeros(n * n)
        e = C.c_double()
        st = self.lib.ref_assemble_m_dense(dims, nx, ny, h, _ptr(np.ascontiguousarray(f)), PEN.get(kind, kind),
                                           T, eps, _ptr(out), C.byref(e))
        assert st == 0, st
        return out.reshape(n, n), e.value

    def penalty_functional(self, dims, shape, h, f, kind, T):
        nx, ny = (list(shape) + [1])[:2]
        return self.lib.ref_penalty_functional(dims, nx, ny, h, _ptr(np.ascontiguousarray(f)),
                                               PEN.get(kind, kind), T)

    def gauss(self, seed, n, stddev=1.0):
        out = np.zeros(n)
        self.lib.ref_gauss_fill(seed, n, stddev, _ptr(out))
        return out

    def mlsqr(self, od, md, g, tau, st, cols, snapshots=False, lsqr=False):
        g = np.ascontiguousarray(g, dtype=np.float64)
        k = st.max_iters
        f = np.zeros(cols)
        tr = (IterRec * k)()
        al = np.zeros(k + 1)
        be = np.zeros(k + 2)
        snap = np.zeros(k * cols) if snapshots else None
        info = SolveInfo()
        if lsqr:
            status = self.lib.ref_lsqr(C.byref(od), _ptr(g), tau, C.byref(st), int(snapshots), _ptr(f),
                                       tr, _ptr(al), _ptr(be), _ptr(snap), C.byref(info))
        else:
            status = self.lib.ref_mlsqr(C.byref(od), C.byref(md), _ptr(g), tau, C.byref(st),
                                        int(snapshots), _ptr(f), tr, _ptr(al), _ptr(be), _ptr(snap),
                                        C.byref(info))
        return SolveOut(f, info.iterations, STOP_NAMES[info.stop_reason], al[:info.n_alphas].copy(),
                        be[:info.n_betas].copy(), _trace_list(tr, info.iterations), status,
                        info.breakdown_iteration,
                        snap.reshape(k, cols)[:info.iterations] if snapshots else None)

    def solve_projected(self, alphas, betas, beta1, tau):
        a = np.ascontiguousarray(alphas, dtype=np.float64)
        b = np.ascontiguousarray(betas, dtype=np.float64)
        y = np.zeros(a.size)
        st = self.lib.ref_solve_projected(_ptr(a), a.size, _ptr(b), b.size, beta1, tau, _ptr(y))
        assert st == 0, st
        return y

    def cg_normal(self, od, dims, shape, h, fM, pen, T, eps, tau, g, st, cols):
        """The reference's own cg_normal with M assembled at fM (eps < 0: auto shift)."""
        nx, ny = (list(shape) + [1])[:2]
        k = st.max_iters
        f = np.zeros(cols)
        tr = (IterRec * k)()
        info = SolveInfo()
        status = self.lib.ref_cg_normal(C.byref(od), dims, nx, ny, h, _ptr(np.ascontiguousarray(fM)),
                                        PEN.get(pen, pen), T, eps, tau, _ptr(np.ascontiguousarray(g)),
                                        C.byref(st), _ptr(f), tr, C.byref(info))
        return SolveOut(f, info.iterations, STOP_NAMES[info.stop_reason], np.zeros(0), np.zeros(0),
                        _trace_list(tr, info.iterations), status, info.breakdown_iteration, None)

    def mlsqr_timed(self, od, md, g, tau, iters, warm, cols):
        """Reference mlsqr for warm+iters iterations; returns (seconds of the last
        `iters` iterations, iterations done, f)."""
        f = np.zeros(cols)
        secs = C.c_double()
        info = SolveInfo()
        st = stop(warm + iters)
        status = self.lib.ref_mlsqr_timed(C.byref(od), C.byref(md), _ptr(np.ascontiguousarray(g)), tau,
                                          C.byref(st), warm, _ptr(f), C.byref(secs), C.byref(info))
        assert status == 0, status
        return secs.value, info.iterations, f

    def solve_nonlinear(self, od, g, dims, shape, h, *, tau, pen, T, inner_stop, inner_cap,
                        threshold, max_outer, spd_mode=0, k_inner=30, epsilon=-1.0, keep=False):
        nx, ny = (list(shape) + [1])[:2]
        n = nx * ny
        cfg = RefOuterCfg(tau, PEN.get(pen, pen), T, inner_stop, inner_cap, threshold, max_outer,
                          spd_mode, k_inner, epsilon)
        f = np.zeros(n)
        steps = (OuterStep * max_outer)()
        ns, sr, trig = C.c_int(), C.c_int(), C.c_int()
        it = np.zeros(max_outer * n) if keep else None
        status = self.lib.ref_solve_nonlinear(C.byref(od), _ptr(np.ascontiguousarray(g)), dims, nx, ny, h,
                                              C.byref(cfg), _ptr(f), steps, C.byref(ns), C.byref(sr),
                                              C.byref(trig), _ptr(it))
        return {
            "status": status, "f": f, "n_steps": ns.value,
            "stop_reason": "stagnation" if sr.value == 0 else "max_outer",
            "triggered_at": trig.value,
            "steps": [{fl[0]: getattr(steps[i], fl[0]) for fl in OuterStep._fields_} for i in range(ns.value)],
            "iterates": it.reshape(max_outer, n)[:ns.value] if keep else None,
        }
