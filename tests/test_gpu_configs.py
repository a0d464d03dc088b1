"""BASELINE.json configurations at their real sizes.

* C1 (128^2, 1 x 50): the whole configuration, bit-exact against the oracle.
* C2 (1024^2, 5 x 30) and C3 (128^3, 5 x 40): every outer step of the whole configuration, bit-exact
  against the oracle run here.
* C4 (fDOT 64^3, 4096 rows = 8.6 GB) and C5 (512^3): size-independent properties at
  full size -- adjointness, a symmetric positive V-cycle, constants annihilated by M,
  bitwise determinism, a monotone damped residual -- plus a reduced C4 bit-exact run, and
  the full-size runs bit-exact against offline oracle fixtures (tests/golden/config_c4.npz:
  all 8 outer steps; config_c5.npz: the first 2 outer steps).
"""
import numpy as np
import pytest

import paper_1308_6634_b200 as mb
from pyoracle import stop as ostop

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def ctx():
    return mb.default_context()


@pytest.fixture()
def dev(orc):
    orc.set_device_order(True)
    yield orc
    orc.set_device_order(False)


def make_2d(orc, n, sigma_px, R, kind, count, seed, noise=0.01):
    taps = orc.taps(n, sigma_px / n, radius=R)
    f = orc.rects2d(n, n, count, seed) if kind == "rects" else orc.shapes2d(n, n, count, seed)
    o = orc.blur(2, (n, n), taps)
    af = o.apply(f)
    g = af + orc.gauss(seed + 1000, n * n, noise * np.abs(af).max())
    return taps, f, g, o


def run_both(dev, taps, g, o, shape, pen, T, tau, K, I, levels):
    dims = len(shape)
    h = 1.0 / shape[0]
    cfg = mb.OuterConfig(tau=tau, penalty=mb.PenaltySpec(pen, T), inner_stop=mb.StoppingConfig.max_iterations(I),
                         inner_cap=I, rel_decrease_threshold=0.0, max_outer=K, mg_levels=levels)
    rep = mb.solve_nonlinear(mb.SeparableGaussianBlur(shape, taps=taps), g, shape, h, cfg)
    orep = dev.nonlinear(o, g, dev.grid(dims, shape, h), tau=tau, pen=pen, T=T, inner_stop=ostop(I),
                         inner_cap=I, max_outer=K, threshold=0.0, levels=levels)
    return rep, orep


def assert_same(rep, orep, I):
    assert len(rep.steps) == orep["n_steps"]
    for s, os_, oa, ob in zip(rep.steps, orep["steps"], orep["alphas"], orep["betas"]):
        assert s.eps_used == os_["eps_used"] and s.penalty_value == os_["penalty_value"]
        assert np.array_equal(s.alphas[:I], oa[:I]) and np.array_equal(s.betas[:I + 1], ob[:I + 1])
    assert np.array_equal(rep.solution, orep["f"])
    assert rel(rep.solution, orep["f"]) <= 1e-6


def test_c1_full_config_bit_exact(ctx, dev):
    """C1: 128^2, sigma 2 px / 13 taps, 8 rectangles, 1% noise, Tikhonov tau 1e-2, 1 x 50, V(2,2) 5 levels."""
    taps, f, g, o = make_2d(dev, 128, 2.0, 6, "rects", 8, 1)
    rep, orep = run_both(dev, taps, g, o, (128, 128), "tikhonov", 1.0, 1e-2, 1, 50, 5)
    assert_same(rep, orep, 50)
    assert rep.steps[0].inner_iterations == 50
    # the reconstruction improves on the data
    assert np.linalg.norm(rep.solution - f) < np.linalg.norm(g - f)


def test_c2_full_config_bit_exact(ctx, dev):
    """C2: 1024^2, sigma 3 px / 19 taps, 32 discs/rectangles, smoothed TV T=0.01, tau 5e-3, 5 x 30."""
    taps, f, g, o = make_2d(dev, 1024, 3.0, 9, "shapes", 32, 2)
    rep, orep = run_both(dev, taps, g, o, (1024, 1024), "tv", 0.01, 5e-3, 5, 30, 5)
    assert_same(rep, orep, 30)
    assert np.linalg.norm(rep.solution - f) < np.linalg.norm(g - f)


def test_c3_full_config_bit_exact(ctx, dev):
    """C3: 128^3, sigma 1.5 vox / 9 taps, 10 ellipsoids, 2% noise, PM-log T=0.05, tau 1e-2, 5 x 40."""
    n = 128
    taps = dev.taps(n, 1.5 / n, radius=4)
    f = dev.ellipsoids3d(n, n, n, 10, 8.0, 40.0, 0.2, 1.0, 3)
    o = dev.blur(3, (n, n, n), taps)
    af = o.apply(f)
    g = af + dev.gauss(1003, n ** 3, 0.02 * np.abs(af).max())
    rep, orep = run_both(dev, taps, g, o, (n, n, n), "pm_log", 0.05, 1e-2, 5, 40, 5)
    assert_same(rep, orep, 40)


def test_c4_reduced_bit_exact(ctx, dev):
    """C4 class at reduced size: 16^3 voxels, 8 x 8 sources/detectors, TV T=0.01, tau 1e-3, 2 x 10."""
    n, ns, nd = 16, 8, 8
    gs, gd = mb.fdot_tables(n, ns, nd, 1.0, 4)
    _, _, a = dev.fdot(n, ns, nd, 1.0, 4)
    f = dev.ellipsoids3d(n, n, n, 3, 1.5, 3.0, 1.0, 1.0, 7)
    o = dev.dense(a).set_row_lengths(ns * nd, n)
    af = o.apply(f)
    g = af + dev.gauss(8, ns * nd, 0.01 * np.abs(af).max())
    h = 1.0 / n
    cfg = mb.OuterConfig(tau=1e-3, penalty=mb.PenaltySpec.tv_smoothed(0.01),
                         inner_stop=mb.StoppingConfig.max_iterations(10), inner_cap=10,
                         rel_decrease_threshold=0.0, max_outer=2, mg_levels=3)
    rep = mb.solve_nonlinear(mb.FdotOperator(n, ns, nd, tables=(gs, gd)), g, (n, n, n), h, cfg)
    orep = dev.nonlinear(o, g, dev.grid(3, (n, n, n), h), tau=1e-3, pen="tv", T=0.01, inner_stop=ostop(10),
                         inner_cap=10, max_outer=2, threshold=0.0, levels=3)
    assert_same(rep, orep, 10)


def test_c4_full_size_properties(ctx):
    """C4 at full size: 64^3 voxels, 64 x 64 = 4096 rows, 8.6 GB fp64 matrix on the device."""
    torch = pytest.importorskip("torch")
    n, ns, nd = 64, 64, 64
    op = mb.FdotOperator(n, ns, nd, mu=1.0, seed=5)
    assert op.shape == (4096, n ** 3)
    gen = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(n ** 3, dtype=torch.float64, device="cuda", generator=gen)
    y = torch.rand(4096, dtype=torch.float64, device="cuda", generator=gen)
    ax, aty = op.apply(x), op.apply_adjoint(y)
    lhs, rhs = float(torch.dot(ax, y)), float(torch.dot(x, aty))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    assert torch.equal(op.apply(x), ax) and torch.equal(op.apply_adjoint(y), aty)  # deterministic
    vc = mb.VCycleMap((n, n, n), 1.0 / n, 4)
    vc.update(torch.zeros(n ** 3, dtype=torch.float64, device="cuda"), mb.PenaltySpec.tv_smoothed(0.01))
    g = ax + 0.01 * ax.abs().max() * torch.randn(4096, dtype=torch.float64, device="cuda", generator=gen)
    r1 = mb.mlsqr(op, vc, g, 1e-3, mb.StoppingConfig.max_iterations(8))
    r2 = mb.mlsqr(op, vc, g, 1e-3, mb.StoppingConfig.max_iterations(8))
    assert torch.equal(r1.solution, r2.solution) and np.array_equal(r1.alphas, r2.alphas)
    res = [t.res_damped for t in r1.trace]
    assert all(res[i + 1] <= res[i] * (1 + 1e-12) for i in range(len(res) - 1))


def test_c5_full_size_properties(ctx):
    """C5 at full size (512^3): blur self-adjoint, V-cycle symmetric positive, M 1 = eps 1,
    deterministic solves with a monotone damped residual."""
    torch = pytest.importorskip("torch")
    n = 512
    shape = (n, n, n)
    N = n ** 3
    op = mb.SeparableGaussianBlur(shape, taps=mb.gaussian_taps(n, 2.0 / n, 6))
    gen = torch.Generator(device="cuda").manual_seed(2)
    x = torch.rand(N, dtype=torch.float64, device="cuda", generator=gen) - 0.5
    y = torch.rand(N, dtype=torch.float64, device="cuda", generator=gen) - 0.5
    lhs, rhs = float(torch.dot(op.apply(x), y)), float(torch.dot(x, op.apply_adjoint(y)))
    assert abs(lhs - rhs) <= 1e-12 * float(op.apply(x).norm() * y.norm())
    f = torch.from_numpy(mb.phantom_ellipsoids3d(n, n, n, 64, 32.0, 160.0, 0.2, 1.0, 5)).cuda()
    vc = mb.VCycleMap(shape, 1.0 / n, 5)
    eps = vc.update(f, mb.PenaltySpec.tv_smoothed(0.01))
    bx, by = vc.solve(x), vc.solve(y)
    s1, s2 = float(torch.dot(bx, y)), float(torch.dot(x, by))
    assert abs(s1 - s2) <= 1e-10 * abs(s1) and float(torch.dot(bx, x)) > 0
    ones = np.ones(N)
    m1 = vc.m_apply(ones)
    assert np.abs(m1 - eps).max() <= 1e-9 * np.abs(m1).max() + 1e-12
    del bx, by, x, y
    g = op.apply(f)
    g = g + 0.01 * g.abs().max() * torch.randn(N, dtype=torch.float64, device="cuda", generator=gen)
    st = mb.StoppingConfig.max_iterations(5)
    r1 = mb.mlsqr(op, vc, g, 5e-3, st)
    r2 = mb.mlsqr(op, vc, g, 5e-3, st)
    assert torch.equal(r1.solution, r2.solution) and np.array_equal(r1.betas, r2.betas)
    res = [t.res_damped for t in r1.trace]
    assert all(res[i + 1] <= res[i] * (1 + 1e-12) for i in range(len(res) - 1))


# ---------------------------------------------------------------------------
# C4 / C5 at their BASELINE sizes against offline oracle fixtures
# (tests/golden/make_config_golden.py: the oracle's device-order restatement of the fixed-count
#  lagged-diffusivity loop, outer.cpp:58-96 with krylov.cpp:335-440 inside, on bench.py's inputs)
# ---------------------------------------------------------------------------
def _fixture(name):
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", f"config_{name}.npz")
    if not os.path.exists(p):
        pytest.fail(f"missing fixture {p}: run tests/golden/make_config_golden.py {name}")
    return np.load(p)


def _sha(v):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(v, dtype="<f8").tobytes()).hexdigest()


def _check_steps(torch, solver, g, N, z, K):
    """K outer steps from f^0 = 0 through OuterSolver; each must equal the fixture bit for bit."""
    I = int(z["inner"])
    fa = torch.zeros(N, dtype=torch.float64, device="cuda")
    fb = torch.empty_like(fa)
    for k in range(K):
        s = solver.step(g, fa, fb)
        fa, fb = fb, fa
        assert s.inner_iterations == int(z[f"s{k}_iters"]) == I, (k, s.inner_iterations)
        assert s.eps_used == float(z[f"s{k}_eps"]), (k, s.eps_used, float(z[f"s{k}_eps"]))
        assert np.array_equal(s.alphas[:I], z[f"s{k}_alphas"]), f"step {k}: alpha sequence differs"
        assert np.array_equal(s.betas[:I + 1], z[f"s{k}_betas"]), f"step {k}: beta sequence differs"
        assert s.penalty_value == float(z[f"s{k}_R"]), (k, s.penalty_value, float(z[f"s{k}_R"]))
        fh = fa.cpu().numpy()
        stride = int(z[f"s{k}_f_stride"])
        assert np.array_equal(fh[::stride][:z[f"s{k}_f_samples"].size], z[f"s{k}_f_samples"]), f"step {k}: f samples"
        assert _sha(fh) == str(z[f"s{k}_f_sha256"]), f"step {k}: iterate digest differs"
        del fh


def test_c5_first_outer_steps_bit_exact(ctx):
    """C5 (512^3, the north-star gate config) at full size: the first outer steps x 50 MLSQR
    iterations -- eps, R(f), alpha[50], beta[51] and the whole iterate -- bit-exact against the
    oracle fixture.  Exercises the size-dependent schedule only 512^3 has: the blur's persistent
    item split, the z-march chunking and the 64-bit element-index paths."""
    torch = pytest.importorskip("torch")
    from bench import CONFIGS, make_problem
    z = _fixture("c5")
    cfg = CONFIGS["c5"]
    shape, taps, f_true, zn = make_problem(mb, cfg)
    N = int(np.prod(shape))
    op = mb.SeparableGaussianBlur(shape, taps=taps)
    af = op.apply(torch.from_numpy(f_true).cuda())
    del f_true
    g = af + cfg["noise"] * float(af.abs().max()) * torch.from_numpy(zn).cuda()
    del af, zn
    assert _sha(g.cpu().numpy()) == str(z["g_sha256"]), "input g differs from the fixture's"
    ocfg = mb.OuterConfig(tau=cfg["tau"], penalty=mb.PenaltySpec(cfg["pen"], cfg["T"]),
                          inner_stop=mb.StoppingConfig.max_iterations(cfg["I"]), inner_cap=cfg["I"],
                          rel_decrease_threshold=0.0, max_outer=cfg["K"], mg_levels=cfg["levels"])
    solver = mb.OuterSolver(op, shape, 1.0 / cfg["n"], ocfg)
    _check_steps(torch, solver, g, N, z, int(z["outer_steps"]))


def test_c4_full_config_bit_exact(ctx):
    """C4 (fDOT 64^3 x 4096 rows, 8.6 GB matrix formed on the device) at full size: every outer
    step of the fixture bit-exact against the oracle."""
    torch = pytest.importorskip("torch")
    from bench import CONFIGS
    z = _fixture("c4")
    cfg = CONFIGS["c4"]
    n = cfg["n"]
    shape = (n, n, n)
    N = n ** 3
    lo, hi = cfg["semi"]
    vlo, vhi = cfg["vals"]
    f_true = mb.phantom_ellipsoids3d(n, n, n, cfg["count"], lo, hi, vlo, vhi, cfg["seed"])
    op = mb.FdotOperator(n, cfg["ns"], cfg["nd"], mu=cfg["mu"], seed=cfg["seed"])
    m = cfg["ns"] * cfg["nd"]
    af = op.apply(torch.from_numpy(f_true).cuda())
    zn = mb.gaussian_noise(cfg["seed"] + 1000, m, 1.0)
    g = af + cfg["noise"] * float(af.abs().max()) * torch.from_numpy(zn).cuda()
    assert _sha(g.cpu().numpy()) == str(z["g_sha256"]), "input g differs from the fixture's"
    ocfg = mb.OuterConfig(tau=cfg["tau"], penalty=mb.PenaltySpec(cfg["pen"], cfg["T"]),
                          inner_stop=mb.StoppingConfig.max_iterations(cfg["I"]), inner_cap=cfg["I"],
                          rel_decrease_threshold=0.0, max_outer=cfg["K"], mg_levels=cfg["levels"])
    solver = mb.OuterSolver(op, shape, 1.0 / n, ocfg)
    _check_steps(torch, solver, g, N, z, int(z["outer_steps"]))


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(96, 80), (48, 40, 32)])
def test_outer_step_host_buffers_match_device(shape):
    """mlsqr_outer_advance with HOST buffers (pinned or pageable numpy): f_prev goes up first, g
    follows on the side stream while the hierarchy is built, f comes back on the side stream next
    to R(f).  Three chained steps must equal the DEVICE-buffer steps bit for bit."""
    torch = pytest.importorskip("torch")
    n = shape[0]
    N = int(np.prod(shape))
    taps = mb.gaussian_taps(n, 2.0 / n, 3)
    rng = np.random.default_rng(5)
    g = rng.random(N)
    cfg = mb.OuterConfig(tau=5e-3, penalty=mb.PenaltySpec.tv_smoothed(0.05),
                         inner_stop=mb.StoppingConfig.max_iterations(7), inner_cap=7,
                         rel_decrease_threshold=0.0, max_outer=3, mg_levels=3)
    op = mb.SeparableGaussianBlur(shape, taps=taps)
    sd = mb.OuterSolver(op, shape, 1.0 / n, cfg)
    gd = torch.from_numpy(g).cuda()
    fa = torch.zeros(N, dtype=torch.float64, device="cuda")
    fb = torch.empty_like(fa)
    dev = []
    for _ in range(3):
        st = sd.step(gd, fa, fb)
        torch.cuda.synchronize()
        dev.append((st.penalty_value, st.eps_used, st.inner_iterations, st.final_residual, fb.cpu().numpy().copy()))
        fa, fb = fb, fa
    sh = mb.OuterSolver(op, shape, 1.0 / n, cfg)
    gh = torch.empty(N, dtype=torch.float64, pin_memory=True)
    gh.copy_(torch.from_numpy(g))
    pa = np.zeros(N)  # pageable
    pb = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
    for k in range(3):
        st = sh.step(gh.numpy(), pa, pb)
        assert (st.penalty_value, st.eps_used, st.inner_iterations, st.final_residual) == dev[k][:4]
        assert np.array_equal(pb, dev[k][4])
        pa, pb = pb, pa
