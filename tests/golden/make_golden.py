"""Generate tests/golden/*.npz from the REFERENCE ITSELF.

Runs the unmodified reference core (oracle/_ref/libmlsqr_ref.so, compiled
from /root/reference/proj/src by oracle/Makefile) on small seeded inputs and
stores inputs + outputs.  Two backends are recorded where it matters:
`scalar` (MLSQR_KERNELS=scalar, kernels_scalar.cpp) which the C restatement
must reproduce bit-for-bit, and `avx2` (the reference default,
kernels_avx2.cpp) whose spread against scalar is the rounding floor
(SURVEY.md §8c "noise floor").

Usage (in the build container, where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from pyoracle import Reference, stop, VEC_FN  # noqa: E402

KINDS = [("tikhonov", 1.0), ("tv", 0.5), ("pm_log", 0.25), ("pm_exp", 0.75)]


def phantom1d(n):
    # Phantom1D::default_phantom (problems.cpp:35-44), realized at cell centres
    jumps = [(0.00, 0.0), (0.10, 1.0), (0.28, 0.0), (0.40, 1.5), (0.62, 0.2), (0.76, 2.0),
             (0.80, 0.2), (0.90, 0.0)]
    x = (np.arange(n) + 0.5) / n
    f = np.zeros(n)
    for i, xi in enumerate(x):
        lev = jumps[0][1]
        for pos, l in jumps:
            if pos <= xi:
                lev = l
        f[i] = lev
    return f


def main():
    r = Reference()
    out = {}
    rng = np.random.default_rng(20131308)

    # --- sampler + taps
    out["gauss_seed7_n1001_sd0.3"] = r.gauss(7, 1001, 0.3)
    for n, s in [(128, 2 / 128), (1024, 3 / 1024), (64, 0.03), (128, 0.03)]:
        out[f"taps_n{n}_s{s!r}"] = r.taps(n, s)

    # --- penalty KATs
    t = np.concatenate([[0.0], np.logspace(-6, 9, 61)])
    out["pen_t"] = t
    for kind, T in KINDS + [("tv", 0.01), ("pm_log", 0.005), ("pm_exp", 0.3)]:
        out[f"pen_c_{kind}_{T}"] = np.array([r.diffusivity(kind, T, v) for v in t])
        out[f"pen_r_{kind}_{T}"] = np.array([r.r_value(kind, T, v) for v in t])

    for backend in ("scalar", "avx2"):
        assert r.select_backend(backend == "scalar"), backend
        # --- operators
        x1 = rng.uniform(-1, 1, 50)
        out[f"{backend}_conv1d_x"] = x1
        out[f"{backend}_conv1d_y"] = r.apply(r.op_conv1d(50, 0.05), x1, 50)
        for nx, ny, s in [(40, 40, 0.05), (33, 21, 0.04)]:
            x = rng.uniform(-1, 1, nx * ny)
            out[f"{backend}_blur2d_{nx}x{ny}_x"] = x
            out[f"{backend}_blur2d_{nx}x{ny}_y"] = r.apply(r.op_blur2d(nx, ny, s), x, nx * ny)
        a = rng.uniform(-1, 1, (17, 23))
        xa = rng.uniform(-1, 1, 23)
        ya = rng.uniform(-1, 1, 17)
        out[f"{backend}_dense_a"] = a
        out[f"{backend}_dense_x"] = xa
        out[f"{backend}_dense_y"] = ya
        out[f"{backend}_dense_ax"] = r.apply(r.op_dense(a), xa, 17)
        out[f"{backend}_dense_aty"] = r.adjoint(r.op_dense(a), ya, 23)

        # --- assembled M (1D and 2D) + penalty functional
        for dims, shape, h in [(1, (33,), 1 / 33), (2, (9, 7), 0.1)]:
            nn = int(np.prod(shape))
            f = rng.standard_normal(nn)
            out[f"{backend}_M{dims}d_f"] = f
            for kind, T in KINDS:
                M, eps = r.assemble_dense(dims, shape, h, f, kind, T)
                out[f"{backend}_M{dims}d_{kind}_dense"] = M
                out[f"{backend}_M{dims}d_{kind}_eps"] = np.array(eps)
                out[f"{backend}_M{dims}d_{kind}_R"] = np.array(
                    r.penalty_functional(dims, shape, h, f, kind, T))

        # --- mlsqr / lsqr on a random dense instance with a dense SPD Cholesky map
        A = rng.uniform(-1, 1, (40, 30))
        g = rng.uniform(-1, 1, 40)
        B = rng.uniform(-1, 1, (30, 30))
        Mspd = B @ B.T + 2.0 * np.eye(30)
        out[f"{backend}_kry_A"], out[f"{backend}_kry_g"], out[f"{backend}_kry_M"] = A, g, Mspd
        for tau in (0.0, 1.0):
            res = r.mlsqr(r.op_dense(A), r.map_chol_dense(Mspd), g, tau, stop(15), 30, snapshots=True)
            out[f"{backend}_mlsqr_dense_tau{tau}_alphas"] = res.alphas
            out[f"{backend}_mlsqr_dense_tau{tau}_betas"] = res.betas
            out[f"{backend}_mlsqr_dense_tau{tau}_f"] = res.f
            out[f"{backend}_mlsqr_dense_tau{tau}_snap"] = res.snapshots
            out[f"{backend}_mlsqr_dense_tau{tau}_trace"] = np.array(
                [[t_["res_damped"], t_["res_data"], t_["s2_value"], t_["anorm_est"], t_["cond_est"],
                  t_["xnorm_est"], t_["alpha"], t_["beta"]] for t_ in res.trace])
            res = r.mlsqr(r.op_dense(A), None, g, tau, stop(25), 30, lsqr=True)
            out[f"{backend}_lsqr_dense_tau{tau}_alphas"] = res.alphas
            out[f"{backend}_lsqr_dense_tau{tau}_betas"] = res.betas
            out[f"{backend}_lsqr_dense_tau{tau}_f"] = res.f
            res = r.mlsqr(r.op_dense(A), r.map_identity(30), g, tau, stop(25), 30)
            out[f"{backend}_mlsqr_ident_tau{tau}_f"] = res.f

        # --- 1D deconvolution, ideal PM-log prior, S4 stop (test_krylov.cpp:350-360 setup)
        n = 128
        ft = phantom1d(n)
        gg = r.apply(r.op_conv1d(n, 0.03), ft, n) + r.gauss(99, n, 0.01)
        delta = 0.01 / np.sqrt(1.0 / n)
        out[f"{backend}_deconv_ftrue"], out[f"{backend}_deconv_g"] = ft, gg
        for tau in (0.0, 0.1):
            st = stop(20, s4=True, delta=delta, eta=1.1)
            res = r.mlsqr(r.op_conv1d(n, 0.03), r.map_assembled(1, (n,), 1 / n, ft, "pm_log", 0.005),
                          gg, tau, st, n)
            out[f"{backend}_deconv_tau{tau}_alphas"] = res.alphas
            out[f"{backend}_deconv_tau{tau}_betas"] = res.betas
            out[f"{backend}_deconv_tau{tau}_f"] = res.f
            out[f"{backend}_deconv_tau{tau}_iters"] = np.array(res.iterations)
            out[f"{backend}_deconv_tau{tau}_resdata"] = np.array([t_["res_data"] for t_ in res.trace])

        # --- 2D deblur 24x24, assembled TV prior at the truth, 30 iterations, tau=1e-2
        nx = 24
        f2 = np.zeros(nx * nx)
        yy, xx = np.meshgrid((np.arange(nx) + 0.5) / nx, (np.arange(nx) + 0.5) / nx, indexing="ij")
        f2[((xx > 0.2) & (xx < 0.6) & (yy > 0.3) & (yy < 0.7)).ravel()] = 1.0
        f2[(((xx - 0.7) ** 2 + (yy - 0.3) ** 2) < 0.02).ravel()] = 0.5
        g2 = r.apply(r.op_blur2d(nx, nx, 0.04), f2, nx * nx) + r.gauss(5, nx * nx, 0.01)
        out[f"{backend}_deblur_ftrue"], out[f"{backend}_deblur_g"] = f2, g2
        res = r.mlsqr(r.op_blur2d(nx, nx, 0.04), r.map_assembled(2, (nx, nx), 1 / nx, f2, "tv", 0.05),
                      g2, 1e-2, stop(30), nx * nx)
        out[f"{backend}_deblur_alphas"], out[f"{backend}_deblur_betas"] = res.alphas, res.betas
        out[f"{backend}_deblur_f"] = res.f
        # same with a fixed, well-conditioning shift (the auto shift makes the exact
        # inverse amplify the constant mode ~1e8: SURVEY.md §7 hard part 1)
        res = r.mlsqr(r.op_blur2d(nx, nx, 0.04),
                      r.map_assembled(2, (nx, nx), 1 / nx, f2, "tv", 0.05, eps=1.0),
                      g2, 1e-2, stop(30), nx * nx)
        out[f"{backend}_deblur_eps1_alphas"], out[f"{backend}_deblur_eps1_betas"] = res.alphas, res.betas
        out[f"{backend}_deblur_eps1_f"] = res.f

        # --- solve_projected (krylov.cpp:631-678) over this backend's stored bidiagonalizations
        for src in ("mlsqr_dense_tau0.0", "deblur_eps1"):
            al, be = out[f"{backend}_{src}_alphas"], out[f"{backend}_{src}_betas"]
            k = min(al.size, be.size - 1)
            for tau in (0.0, 1e-3, 0.1, 10.0):
                out[f"{backend}_proj_{src}_tau{tau}"] = r.solve_projected(al[:k], be[:k + 1], be[0], tau)

        # --- cg_normal (krylov.cpp:551-628), the unpriorconditioned baseline
        for tau in (0.0, 0.1):
            st = stop(20, s4=True, delta=delta, eta=1.1)
            res = r.cg_normal(r.op_conv1d(n, 0.03), 1, (n,), 1 / n, ft, "pm_log", 0.005, -1.0, tau, gg, st, n)
            pre = f"{backend}_cgn_deconv_tau{tau}"
            out[pre + "_f"] = res.f
            out[pre + "_iters"] = np.array([res.iterations, res.status])
            out[pre + "_trace"] = np.array([[t_["res_data"], t_["res_damped"], t_["s2_value"], t_["xnorm_est"]]
                                            for t_ in res.trace])
        res = r.cg_normal(r.op_blur2d(nx, nx, 0.04), 2, (nx, nx), 1 / nx, f2, "tv", 0.05, 1.0, 1e-2, g2,
                          stop(30), nx * nx)
        out[f"{backend}_cgn_deblur_f"] = res.f
        out[f"{backend}_cgn_deblur_trace"] = np.array([[t_["res_data"], t_["res_damped"], t_["s2_value"],
                                                         t_["xnorm_est"]] for t_ in res.trace])

        # --- nonlinear (lagged diffusivity) 1D runs, reference outer loop with Cholesky M^-1
        for pen, T in (("pm_log", 0.005), ("tikhonov", 1.0), ("tv", 0.01)):
            st = stop(1000, s4=True, delta=delta, eta=1.1)
            rep = r.solve_nonlinear(r.op_conv1d(n, 0.03), gg, 1, (n,), 1 / n, tau=0.0, pen=pen, T=T,
                                    inner_stop=st, inner_cap=20, threshold=0.15, max_outer=25,
                                    keep=True)
            pre = f"{backend}_outer_{pen}"
            out[pre + "_f"] = rep["f"]
            out[pre + "_iterates"] = rep["iterates"]
            out[pre + "_R"] = np.array([s_["penalty_value"] for s_ in rep["steps"]])
            out[pre + "_inner"] = np.array([s_["inner_iterations"] for s_ in rep["steps"]])
            out[pre + "_trigger"] = np.array(rep["triggered_at"])

    # --- SpdSolver maps over the assembled M (spdsolve.cpp:22-137): envelope Cholesky and
    #     inner CG, one solve each; own generator so the arrays above keep their inputs
    rng2 = np.random.default_rng(22137)
    for dims, shape, h in [(1, (33,), 1 / 33), (2, (9, 7), 0.1), (2, (24, 24), 1 / 24)]:
        nn = int(np.prod(shape))
        tag = "x".join(map(str, shape))
        f, p = rng2.standard_normal(nn), rng2.standard_normal(nn)
        out[f"maps_{tag}_f"], out[f"maps_{tag}_p"] = f, p
        for backend in ("scalar", "avx2"):
            assert r.select_backend(backend == "scalar"), backend
            for kind, T in KINDS[:3]:
                out[f"{backend}_maps_{tag}_{kind}_chol"] = r.map_solve(
                    r.map_assembled(dims, shape, h, f, kind, T), p)
                out[f"{backend}_maps_{tag}_{kind}_cg7"] = r.map_solve(
                    r.map_assembled(dims, shape, h, f, kind, T, inner_cg=7), p)

    # --- krylov_basis (krylov.cpp:700-754): the three spaces the runner dumps (runner.cpp:245-275)
    for backend in ("scalar", "avx2"):
        assert r.select_backend(backend == "scalar"), backend
        ft, gg = out["scalar_deconv_ftrue"], out["scalar_deconv_g"]
        od = r.op_conv1d(128, 0.03)
        out[f"{backend}_kb_plain"] = r.krylov_basis(od, 128, 6, gg)[0]
        out[f"{backend}_kb_tauM"] = r.krylov_basis(od, 128, 6, gg, tau=0.1,
                                                   m=(1, (128,), 1 / 128, ft, "pm_log", 0.005, -1.0))[0]
        out[f"{backend}_kb_pc"] = r.krylov_basis(
            od, 128, 4, gg, md=r.map_assembled(1, (128,), 1 / 128, ft, "pm_log", 0.005))[0]
        out[f"{backend}_kb_pc_cg"] = r.krylov_basis(
            od, 128, 4, gg, md=r.map_assembled(1, (128,), 1 / 128, ft, "pm_log", 0.005, inner_cg=8))[0]
        # rank exhaustion: 3x3 identity has a 1-D Krylov space
        kb, ex = r.krylov_basis(r.op_identity(3), 3, 3, np.array([1.0, 2.0, 3.0]))
        out[f"{backend}_kb_ident"] = kb
        out[f"{backend}_kb_ident_exhausted"] = np.array(int(ex))

    # --- SignFlipMap breakdown (test_krylov.cpp:131-145)
    @VEC_FN
    def flip(ctx, p, v):
        for i in range(8):
            v[i] = -p[i]
        return 0

    A = rng.uniform(-1, 1, (10, 8))
    g = rng.uniform(-1, 1, 10)
    res = r.mlsqr(r.op_dense(A), r.map_callback(8, C.cast(flip, C.c_void_p).value, None), g, 0.0,
                  stop(5), 8)
    out["signflip_A"], out["signflip_g"] = A, g
    out["signflip_status"] = np.array([res.status, res.breakdown_iteration])

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
