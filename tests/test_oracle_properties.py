"""Property tests for the oracle parts that have NO reference implementation
(3D blur, 3D edge grid, V-cycle SpdMap, device arithmetic order, generators).
These mirror the reference's own property tests (test_linops.cpp,
test_diffusion.cpp, test_spdsolve.cpp) -- "parity unpinned" against the
reference, pinned by properties instead.
"""
import numpy as np
import pytest

from pyoracle import stop

KINDS = [("tikhonov", 1.0), ("tv", 0.5), ("pm_log", 0.25), ("pm_exp", 0.75)]


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def conv_matrix(n, taps):
    R = (len(taps) - 1) // 2
    C = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - R), min(n, i + R + 1)):
            C[i, j] = taps[R + j - i]
    return C


def test_blur3d_is_kronecker_and_self_adjoint(orc):
    nx, ny, nz = 7, 6, 5
    taps = orc.taps(8, 0.12, radius=2)
    op = orc.blur(3, (nx, ny, nz), taps)
    K = np.kron(conv_matrix(nz, taps), np.kron(conv_matrix(ny, taps), conv_matrix(nx, taps)))
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, nx * ny * nz)
    y = rng.uniform(-1, 1, nx * ny * nz)
    assert rel(op.apply(x), K @ x) < 1e-12  # test_linops.cpp:185-206 (2D analogue)
    lhs, rhs = op.apply(x) @ y, x @ op.adjoint(y)
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(op.apply(x)) * np.linalg.norm(y)


@pytest.mark.parametrize("kind,T", KINDS)
def test_m3d_properties(orc, kind, T):
    shape = (6, 5, 4)
    grid = orc.grid(3, shape, 0.2)
    n = int(np.prod(shape))
    f = np.random.default_rng(3).standard_normal(n)
    cx, cy, cz = orc.edge_coeffs(grid, f, kind, T)
    M = np.stack([orc.m_apply(grid, cx, cy, cz, 0.0, e) for e in np.eye(n)], 1)
    assert np.array_equal(M, M.T)                                      # exact symmetry
    assert np.linalg.norm(M @ np.ones(n)) <= 1e-12 * np.linalg.norm(M)  # annihilates constants
    off = M - np.diag(np.diag(M))
    assert (off <= 0).all()                                             # M-matrix
    assert (np.diag(M) >= -off.sum(1) * (1 - 1e-14)).all()
    # R(f) gradient = M f (test_diffusion.cpp:179-206), finite differences
    g = M @ f
    for i in (0, 17, n - 1):
        step = 1e-6 * (1 + abs(f[i]))
        fp, fm = f.copy(), f.copy()
        fp[i] += step
        fm[i] -= step
        fd = (orc.penalty_functional(grid, fp, kind, T) - orc.penalty_functional(grid, fm, kind, T)) / (2 * step)
        assert fd == pytest.approx(g[i], rel=1e-5, abs=1e-8)


def aggregation_p(shape, dims):
    nx, ny, nz = shape
    cn = (nx // 2, ny // 2 if dims >= 2 else 1, nz // 2 if dims >= 3 else 1)
    P = np.zeros((nx * ny * nz, cn[0] * cn[1] * cn[2]))
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                Z = z // 2 if dims >= 3 else 0
                Y = y // 2 if dims >= 2 else 0
                P[(z * ny + y) * nx + x, (Z * cn[1] + Y) * cn[0] + x // 2] = 1.0
    return P


@pytest.mark.parametrize("dims,shape", [(1, (16, 1, 1)), (2, (8, 8, 1)), (3, (8, 4, 4))])
def test_vcycle_hierarchy_is_galerkin(orc, dims, shape):
    grid = orc.grid(dims, shape[:dims], 1.0 / shape[0])
    n = int(np.prod(shape))
    f = np.random.default_rng(dims).standard_normal(n)
    cx, cy, cz = orc.edge_coeffs(grid, f, "tv", 0.3)
    mg = orc.vcycle(grid, 2)
    mg.set(cx, cy, cz, 1e-3)
    (cnx, cny, cnz), ccx, ccy, ccz, ceps = mg.level(1)
    M = np.stack([orc.m_apply(grid, cx, cy, cz, 1e-3, e) for e in np.eye(n)], 1)
    P = aggregation_p(shape, dims)
    cg = orc.grid(dims, (cnx, cny, cnz)[:dims], 1.0)
    nc = cnx * cny * cnz
    Mc = np.stack([orc.m_apply(cg, ccx, ccy, ccz, ceps, e) for e in np.eye(nc)], 1)
    assert np.allclose(Mc, P.T @ M @ P, rtol=1e-14, atol=1e-12 * np.abs(M).max())
    assert ceps == 1e-3 * 2 ** dims


@pytest.mark.parametrize("dims,shape,levels", [(1, (64,), 4), (2, (16, 16), 3), (3, (8, 8, 8), 3)])
def test_vcycle_is_a_fixed_spd_linear_map(orc, dims, shape, levels):
    """SpdMap contract (spdsolve.hpp:11-14): fixed, symmetric, positive definite, linear."""
    grid = orc.grid(dims, shape, 1.0 / shape[0])
    n = int(np.prod(shape))
    rng = np.random.default_rng(11)
    f = rng.standard_normal(n)
    cx, cy, cz = orc.edge_coeffs(grid, f, "pm_log", 0.5)
    eps = 1e-8 * orc.max_diag(grid, cx, cy, cz)
    mg = orc.vcycle(grid, levels)
    mg.set(cx, cy, cz, eps)
    B = np.stack([mg.solve(e) for e in np.eye(n)], 1)
    assert np.abs(B - B.T).max() <= 1e-12 * np.abs(B).max()
    ev = np.linalg.eigvalsh(0.5 * (B + B.T))
    assert ev.min() > 0
    # bounded gain on the eps (constant) mode: no 1/eps amplification
    assert ev.max() < 1e3 / np.abs(np.diag(np.stack([orc.m_apply(grid, cx, cy, cz, eps, e) for e in np.eye(n)]))).min()
    p, q = rng.standard_normal(n), rng.standard_normal(n)
    assert rel(mg.solve(2.0 * p - 3.0 * q), 2.0 * mg.solve(p) - 3.0 * mg.solve(q)) < 1e-13
    assert np.array_equal(mg.solve(p), mg.solve(p))  # bitwise repeatable


def test_vcycle_priorconditioned_mlsqr_matches_cholesky_early_iterates(orc):
    """V-cycle-preconditioned mlsqr vs Cholesky-preconditioned mlsqr on the
    same M: the Krylov spaces differ (B != M^-1) but both are valid SpdMaps;
    the V-cycle run must satisfy the same monotone-residual property."""
    n = 32
    grid = orc.grid(2, (n, n), 1 / n)
    f = orc.rects2d(n, n, 8, 1)
    taps = orc.taps(n, 2 / n, radius=6)
    op = orc.blur(2, (n, n), taps)
    g = op.apply(f) + orc.gauss(5, n * n, 0.01 * np.abs(op.apply(f)).max())
    cx, cy, cz = orc.edge_coeffs(grid, f, "tv", 0.01)
    eps = 1e-8 * orc.max_diag(grid, cx, cy, cz)
    mg = orc.vcycle(grid, 3)
    mg.set(cx, cy, cz, eps)
    res = orc.mlsqr(op, mg, g, 1e-2, stop(30))
    r = [t["res_damped"] for t in res.trace]
    assert all(r[i + 1] <= r[i] * (1 + 1e-12) for i in range(len(r) - 1))


def test_canonical_dot_is_a_dot(orc):
    rng = np.random.default_rng(5)
    for n, L in [(1, 1), (31, 31), (64, 64), (1000, 1000), (24 * 24, 24), (128 * 128, 128), (40000, 200)]:
        x, y = rng.standard_normal(n), rng.standard_normal(n)
        assert orc.canon_dot(x, y, L) == pytest.approx(x @ y, rel=1e-12, abs=1e-12)
    assert orc.canon_dot(np.zeros(0), np.zeros(0), 1) == 0.0


def test_device_order_agrees_with_reference_order_to_rounding(orc, golden):
    A, g, M = golden["scalar_kry_A"], golden["scalar_kry_g"], golden["scalar_kry_M"]
    ref = orc.mlsqr(orc.dense(A), orc.chol_map(M), g, 1.0, stop(15))
    with orc.device_order():
        dev = orc.mlsqr(orc.dense(A), orc.chol_map(M), g, 1.0, stop(15))
    assert rel(dev.alphas, ref.alphas) < 1e-13 and rel(dev.f, ref.f) < 1e-10
    assert orc.lib.orc_dhypot(3.0, 4.0) == 5.0


def test_phantoms_and_generators(orc):
    f = orc.rects2d(128, 128, 8, 1)
    assert f.min() >= 0 and f.max() <= 1 and np.count_nonzero(f) > 100
    assert np.array_equal(f, orc.rects2d(128, 128, 8, 1))
    e = orc.ellipsoids3d(32, 32, 32, 10, 2, 10, 0.2, 1.0, 3)
    vals = np.unique(e)
    assert vals[0] == 0 and ((vals[1:] >= 0.2) & (vals[1:] <= 1.0)).all()
    gs, gd, a = orc.fdot(4, 3, 2, 1.0, 7)
    assert a.shape == (6, 64) and (a > 0).all()
    assert np.array_equal(a[1 * 2 + 1], gs[64:128] * gd[64:128])


def test_algorithm1_equals_algorithm2(orc):
    """test_krylov.cpp:75-97: explicit-factor preconditioned LSQR (Algorithm 1: plain LSQR on
    A R^-1 with M = R^T R, f = R^-1 x) and the factorization-free mlsqr (Algorithm 2) agree to
    1e-8 over 15 iterations -- here with the oracle's own lsqr and Cholesky map."""
    rng = np.random.default_rng(12)
    n, m = 40, 60
    A = rng.standard_normal((m, n)) / 8
    g = A @ rng.uniform(-1, 1, n) + 0.01 * rng.standard_normal(m)
    grid = orc.grid(1, (n,), 1.0 / n)
    cx, cy, cz = orc.edge_coeffs(grid, rng.uniform(0, 1, n), "tv", 0.1)
    eps = 0.1 * orc.max_diag(grid, cx, cy, cz)      # a well-conditioned M (the comparison is
    M = np.stack([orc.m_apply(grid, cx, cy, cz, eps, e) for e in np.eye(n)], 1)  # of two algorithms)
    R = np.linalg.cholesky(M).T                       # M = R^T R
    from scipy.linalg import solve_triangular
    Abar = solve_triangular(R, A.T, trans="T").T      # A R^-1
    st = stop(15)
    for tau in (0.0, 1e-2):
        r2 = orc.mlsqr(orc.dense(A), orc.chol_map(M), g, tau, st)
        r1 = orc.mlsqr(orc.dense(Abar), None, g, tau, st, lsqr=True)
        f1 = solve_triangular(R, r1.f)
        assert np.linalg.norm(f1 - r2.f) <= 1e-8 * np.linalg.norm(r2.f)
        assert np.max(np.abs(r1.alphas - r2.alphas) / r2.alphas) < 1e-8
