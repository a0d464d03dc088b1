"""z-slab decomposition on one GPU: P virtual ranks (loopback communicator, one thread and
one Context per rank) must reproduce the unsharded results BIT FOR BIT -- blur with R-plane
ghosts, the V-cycle hierarchy with one-plane ghosts on every level and an allreduced max
diagonal, the canonical reductions (allgathered block partials / raw segments), mlsqr and
the outer loop.  The NCCL transport runs exactly the same code with ncclSend/Recv and
ncclAllGather instead of the loopback copies."""
import threading

import numpy as np
import pytest

import paper_1308_6634_b200 as mb

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]


def run_ranks(P, nz, fn):
    group = mb.LoopGroup(P)
    ctxs = []
    for r in range(P):
        c = mb.Context(0)
        c.set_comm_loopback(group, r)
        c.set_slab(nz, r * nz // P)
        ctxs.append(c)
    out, errs = [None] * P, []

    def work(r):
        try:
            out[r] = fn(r, ctxs[r], slice(r * nz // P, (r + 1) * nz // P))
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=500)
    assert not any(t.is_alive() for t in th), "a virtual rank hung"
    assert not errs, errs
    return out


def planes(v, shape):
    nx, ny, nz = shape
    return v.reshape(nz, ny * nx)


@pytest.fixture(scope="module")
def problem():
    shape = (64, 40, 64)
    nx, ny, nz = shape
    taps = mb.gaussian_taps(nx, 2.0 / nx, 6)
    rng = np.random.default_rng(3)
    f = mb.phantom_ellipsoids3d(nx, ny, nz, 6, 4.0, 16.0, 0.2, 1.0, 9)
    op = mb.SeparableGaussianBlur(shape, taps=taps)
    af = op.apply(f)
    g = af + 0.01 * np.abs(af).max() * rng.standard_normal(f.size)
    return shape, taps, f, g


@pytest.mark.parametrize("P", [2, 4])
def test_blur_and_vcycle_sharded_bit_exact(problem, P):
    shape, taps, f, g = problem
    nx, ny, nz = shape
    h = 1.0 / nx
    x = np.random.default_rng(P).uniform(-1, 1, f.size)
    ref_y = mb.SeparableGaussianBlur(shape, taps=taps).apply(x)
    vc = mb.VCycleMap(shape, h, 4)
    ref_eps = vc.update(f, mb.PenaltySpec.tv_smoothed(0.05))
    ref_v = vc.solve(x)

    def fn(r, ctx, sl):
        loc = (nx, ny, sl.stop - sl.start)
        op = mb.SeparableGaussianBlur(loc, taps=taps, ctx=ctx)
        y = op.apply(planes(x, shape)[sl].ravel())
        m = mb.VCycleMap(loc, h, 4, ctx=ctx)
        eps = m.update(planes(f, shape)[sl].ravel(), mb.PenaltySpec.tv_smoothed(0.05))
        v = m.solve(planes(x, shape)[sl].ravel())
        return y, eps, v

    res = run_ranks(P, nz, fn)
    assert np.array_equal(np.concatenate([r[0] for r in res]), ref_y)
    assert all(r[1] == ref_eps for r in res)
    assert np.array_equal(np.concatenate([r[2] for r in res]), ref_v)


@pytest.mark.parametrize("P", [2, 4])
def test_mlsqr_and_outer_sharded_bit_exact(problem, P):
    shape, taps, f, g = problem
    nx, ny, nz = shape
    h = 1.0 / nx
    op = mb.SeparableGaussianBlur(shape, taps=taps)
    vc = mb.VCycleMap(shape, h, 4)
    vc.update(f, mb.PenaltySpec.tv_smoothed(0.05))
    st = mb.StoppingConfig.max_iterations(15)
    ref = mb.mlsqr(op, vc, g, 5e-3, st)
    cfg = mb.OuterConfig(tau=5e-3, penalty=mb.PenaltySpec.tv_smoothed(0.05),
                         inner_stop=mb.StoppingConfig.max_iterations(8), inner_cap=8,
                         rel_decrease_threshold=0.0, max_outer=2, mg_levels=4)
    ref_nl = mb.solve_nonlinear(op, g, shape, h, cfg)

    def fn(r, ctx, sl):
        loc = (nx, ny, sl.stop - sl.start)
        o = mb.SeparableGaussianBlur(loc, taps=taps, ctx=ctx)
        m = mb.VCycleMap(loc, h, 4, ctx=ctx)
        m.update(planes(f, shape)[sl].ravel(), mb.PenaltySpec.tv_smoothed(0.05))
        gl = planes(g, shape)[sl].ravel()
        res = mb.mlsqr(o, m, gl, 5e-3, st)
        nl = mb.solve_nonlinear(o, gl, loc, h, cfg)
        return res, nl

    out = run_ranks(P, nz, fn)
    for res, nl in out:
        assert np.array_equal(res.alphas, ref.alphas) and np.array_equal(res.betas, ref.betas)
        assert [s.penalty_value for s in nl.steps] == [s.penalty_value for s in ref_nl.steps]
        assert [s.eps_used for s in nl.steps] == [s.eps_used for s in ref_nl.steps]
    assert np.array_equal(np.concatenate([o[0].solution for o in out]), ref.solution)
    assert np.array_equal(np.concatenate([o[1].solution for o in out]), ref_nl.solution)


def test_block_aligned_reduction_path_bit_exact():
    """1024 x 64 x 64 with P = 2: each rank owns 65536 reduction segments (two whole
    32768-blocks), so the ranks allgather level-3 tree partials instead of raw segments."""
    shape = (1024, 64, 64)
    nx, ny, nz = shape
    h = 1.0 / nx
    taps = mb.gaussian_taps(nx, 2.0 / nx, 4)
    rng = np.random.default_rng(7)
    g = rng.uniform(-1, 1, nx * ny * nz)
    op = mb.SeparableGaussianBlur(shape, taps=taps)
    vc = mb.VCycleMap(shape, h, 3)
    vc.update(np.zeros(g.size), mb.PenaltySpec.tikhonov())
    st = mb.StoppingConfig.max_iterations(6)
    ref = mb.mlsqr(op, vc, g, 1e-2, st)

    def fn(r, ctx, sl):
        loc = (nx, ny, sl.stop - sl.start)
        o = mb.SeparableGaussianBlur(loc, taps=taps, ctx=ctx)
        m = mb.VCycleMap(loc, h, 3, ctx=ctx)
        m.update(np.zeros(nx * ny * loc[2]), mb.PenaltySpec.tikhonov())
        return mb.mlsqr(o, m, planes(g, shape)[sl].ravel(), 1e-2, st)

    out = run_ranks(2, nz, fn)
    assert all(np.array_equal(o.alphas, ref.alphas) for o in out)
    assert np.array_equal(np.concatenate([o.solution for o in out]), ref.solution)


def test_nccl_world1_transport_runs_the_sharded_graph():
    """The NCCL transport on one GPU: dlopen + ncclGetUniqueId + ncclCommInitRank through the
    C-ABI, then the DECOMPOSED code path on a one-rank communicator (mlsqr_ctx_set_slab makes the
    context sharded even at P = 1): guarded vectors, ghost exchanges (NCCL group calls with no
    peers), reduce3 + ncclAllGather of the tree partials, ncclAllReduce(max) for eps, coarse-level
    agglomeration -- all inside the captured CUDA graph.  The result must equal the plain
    context's bit for bit.  N > 1 needs one GPU per rank (tools/nccl_parity.py)."""
    from paper_1308_6634_b200 import dist as pdist
    uid = mb.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128
    n = 32
    shape = (n, n, n)
    ctx = pdist.sharded_context(0, 0, 1, n, uid)
    taps = mb.gaussian_taps(n, 2.0 / n, 4)
    rng = np.random.default_rng(1)
    g = rng.uniform(-1, 1, n ** 3)
    cfg = mb.OuterConfig(tau=5e-3, penalty=mb.PenaltySpec("tv", 0.05), inner_stop=mb.StoppingConfig.max_iterations(8),
                         inner_cap=8, rel_decrease_threshold=0.0, max_outer=2, mg_levels=3)
    ctx.set_timing(True)
    a = mb.solve_nonlinear(mb.SeparableGaussianBlur(shape, taps=taps, ctx=ctx), g, shape, 1.0 / n, cfg)
    halo, coll = ctx.timing(mb.TCLASS["halo"]), ctx.timing(mb.TCLASS["coll"])
    ctx.set_timing(False)
    b = mb.solve_nonlinear(mb.SeparableGaussianBlur(shape, taps=taps), g, shape, 1.0 / n, cfg)
    assert halo[1] > 0 and coll[1] > 0, (halo, coll)  # the exchanges and collectives really ran
    assert np.array_equal(a.solution, b.solution)
    for sa, sb in zip(a.steps, b.steps):
        assert np.array_equal(sa.alphas, sb.alphas) and sa.eps_used == sb.eps_used
    # and with graph capture (timing off): the same bits
    c = mb.solve_nonlinear(mb.SeparableGaussianBlur(shape, taps=taps, ctx=ctx), g, shape, 1.0 / n, cfg)
    assert np.array_equal(c.solution, b.solution)


def test_nccl_world1_row_shard_dense():
    """C4's row-shard path on a one-rank NCCL communicator: A^T u allgathers the canonical chunk
    partials through ncclAllGather; bit-identical to the plain context."""
    uid = mb.nccl_unique_id()
    ctx = mb.Context(0)
    ctx.set_comm_nccl(uid, 0, 1)
    m, n = 256, 8 ** 3
    ctx.set_row_shard(m, 0)
    a = np.random.default_rng(4).standard_normal((m, n))
    g = a @ np.random.default_rng(5).standard_normal(n)
    vc_s = mb.VCycleMap((8, 8, 8), 1 / 8, 2, ctx=ctx)
    vc_s.update(np.zeros(n), mb.PenaltySpec.tikhonov())
    vc = mb.VCycleMap((8, 8, 8), 1 / 8, 2)
    vc.update(np.zeros(n), mb.PenaltySpec.tikhonov())
    st = mb.StoppingConfig.max_iterations(10)
    r1 = mb.mlsqr(mb.DenseOperator(a, sol_row_len=8, ctx=ctx), vc_s, g, 1e-3, st)
    r2 = mb.mlsqr(mb.DenseOperator(a, sol_row_len=8), vc, g, 1e-3, st)
    assert np.array_equal(r1.solution, r2.solution) and np.array_equal(r1.betas, r2.betas)


# ---------------------------------------------------------------------------
# row shards (C4: dense operator rows split over ranks, solution space replicated)
# ---------------------------------------------------------------------------
def run_row_ranks(P, m, fn):
    group = mb.LoopGroup(P)
    ctxs = []
    for r in range(P):
        c = mb.Context(0)
        c.set_comm_loopback(group, r)
        c.set_row_shard(m, r * m // P)
        ctxs.append(c)
    out, errs = [None] * P, []

    def work(r):
        try:
            out[r] = fn(r, ctxs[r], slice(r * m // P, (r + 1) * m // P))
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=500)
    assert not any(t.is_alive() for t in th), "a virtual rank hung"
    assert not errs, errs
    return out


@pytest.mark.parametrize("P", [2, 4, 8])
def test_dense_row_shards_bit_exact(P):
    """mlsqr with a replicated V-cycle and with the identity map on a row-sharded dense operator
    equals the single-rank solve bit for bit (A^T chunk partials allgathered, data norms
    allgathered, solution space replicated)."""
    n = 8
    m = 256
    rng = np.random.default_rng(11)
    A = rng.standard_normal((m, n ** 3)) / 16
    g = rng.standard_normal(m)
    shape = (n, n, n)
    f0 = rng.uniform(0, 1, n ** 3)
    st = mb.StoppingConfig.max_iterations(12)
    ref_i = mb.mlsqr(mb.DenseOperator(A, sol_row_len=n), mb.IdentityMap(n ** 3), g, 1e-2, st)
    vc = mb.VCycleMap(shape, 1.0 / n, 2)
    vc.update(f0, mb.PenaltySpec.tv_smoothed(0.05))
    ref_v = mb.mlsqr(mb.DenseOperator(A, sol_row_len=n), vc, g, 1e-2, st)

    def fn(r, ctx, sl):
        op = mb.DenseOperator(A[sl], sol_row_len=n, ctx=ctx)
        a = mb.mlsqr(op, mb.IdentityMap(n ** 3, ctx=ctx), g[sl], 1e-2, st)
        m_ = mb.VCycleMap(shape, 1.0 / n, 2, ctx=ctx)
        m_.update(f0, mb.PenaltySpec.tv_smoothed(0.05))
        b = mb.mlsqr(op, m_, g[sl], 1e-2, st)
        return a, b

    out = run_row_ranks(P, m, fn)
    for a, b in out:
        assert np.array_equal(a.alphas, ref_i.alphas) and np.array_equal(a.betas, ref_i.betas)
        assert np.array_equal(a.solution, ref_i.solution)
        assert np.array_equal(b.alphas, ref_v.alphas) and np.array_equal(b.solution, ref_v.solution)


@pytest.mark.parametrize("P", [2, 8])
def test_fdot_row_shards_nonlinear_bit_exact(P):
    """The C4 shape in miniature: fDOT rows (source, detector) split over ranks, the 3D TV
    outer loop with a replicated V-cycle; every outer step equals the single-rank run."""
    n, ns, nd = 8, 16, 16
    m = ns * nd
    shape = (n, n, n)
    op1 = mb.FdotOperator(n, ns, nd, seed=4)
    f_true = mb.phantom_ellipsoids3d(n, n, n, 3, 1.0, 3.0, 0.2, 1.0, 5)
    g = op1.apply(f_true)
    g = g + 0.01 * np.abs(g).max() * np.random.default_rng(2).standard_normal(m)
    cfg = mb.OuterConfig(tau=1e-3, penalty=mb.PenaltySpec.tv_smoothed(0.01),
                         inner_stop=mb.StoppingConfig.max_iterations(10), inner_cap=10,
                         rel_decrease_threshold=0.0, max_outer=3, mg_levels=2)
    ref = mb.solve_nonlinear(op1, g, shape, 1.0 / n, cfg)

    def fn(r, ctx, sl):
        op = mb.FdotOperator(n, ns, nd, seed=4, ctx=ctx)
        assert op.n_rows == m // P
        return mb.solve_nonlinear(op, g[sl], shape, 1.0 / n, cfg)

    out = run_row_ranks(P, m, fn)
    for nl in out:
        assert [s.penalty_value for s in nl.steps] == [s.penalty_value for s in ref.steps]
        assert np.array_equal(nl.solution, ref.solution)


def test_row_shard_validation():
    group = mb.LoopGroup(2)
    c = mb.Context(0)
    c.set_comm_loopback(group, 0)
    c.set_row_shard(96, 0)  # 48 local rows: not whole 32-row segments
    with pytest.raises((ValueError, mb.DimensionError)):
        mb.DenseOperator(np.zeros((48, 64)), ctx=c)
    with pytest.raises(ValueError):
        mb.SeparableGaussianBlur((16, 16, 16), taps=mb.gaussian_taps(16, 0.1, 2), ctx=c)


@pytest.mark.parametrize("P", [2, 4])
def test_outer_solver_steps_sharded_bit_exact(problem, P):
    """The bench's path: OuterSolver.step (mlsqr_outer_advance, resident hierarchy and
    workspace) on device tensors, three steps -- every rank's slab of f after each step and
    every step's R(f) / eps equal the single-rank run."""
    torch = pytest.importorskip("torch")
    shape, taps, f, g = problem
    nx, ny, nz = shape
    h = 1.0 / nx
    cfg = mb.OuterConfig(tau=5e-3, penalty=mb.PenaltySpec.tv_smoothed(0.05),
                         inner_stop=mb.StoppingConfig.max_iterations(6), inner_cap=6,
                         rel_decrease_threshold=0.0, max_outer=3, mg_levels=4)

    def run(op, shp, gl, ctx_dev=None):
        s = mb.OuterSolver(op, shp, h, cfg)
        gd = torch.from_numpy(gl).cuda()
        fa = torch.zeros(gl.size, dtype=torch.float64, device="cuda")
        fb = torch.empty_like(fa)
        out = []
        for _ in range(3):
            st = s.step(gd, fa, fb)
            torch.cuda.synchronize()
            out.append((st.penalty_value, st.eps_used, st.inner_iterations, fb.cpu().numpy().copy()))
            fa, fb = fb, fa
        return out

    ref = run(mb.SeparableGaussianBlur(shape, taps=taps), shape, g)

    def fn(r, ctx, sl):
        loc = (nx, ny, sl.stop - sl.start)
        return run(mb.SeparableGaussianBlur(loc, taps=taps, ctx=ctx), loc, planes(g, shape)[sl].ravel())

    out = run_ranks(P, nz, fn)
    for k in range(3):
        assert all(o[k][:3] == ref[k][:3] for o in out)
        assert np.array_equal(np.concatenate([o[k][3] for o in out]), ref[k][3])


@pytest.mark.parametrize("agg_planes", ["0", "4", "8", "16", "32"])
def test_coarse_agglomeration_bit_exact(problem, monkeypatch, agg_planes):
    """Coarse-level agglomeration: from the first level whose slab holds at most
    MLSQR_AGG_PLANES planes, every rank solves the remaining levels on the whole coarse grid
    (one allgather of the restricted rhs per V-cycle instead of ghost exchanges on every coarse
    sweep).  Every threshold -- none, late, early, from level 1 -- is bit-identical to one GPU."""
    monkeypatch.setenv("MLSQR_AGG_PLANES", agg_planes)
    shape, taps, f, g = problem
    nx, ny, nz = shape
    h = 1.0 / nx
    pen = mb.PenaltySpec.tv_smoothed(0.01)
    st = mb.StoppingConfig.max_iterations(8)
    vc = mb.VCycleMap(shape, h, 4)
    vc.update(f, pen)
    ref = mb.mlsqr(mb.SeparableGaussianBlur(shape, taps=taps), vc, g, 5e-3, st)

    for P in (2, 4):
        def fn(r, ctx, sl):
            loc = (nx, ny, sl.stop - sl.start)
            m = mb.VCycleMap(loc, h, 4, ctx=ctx)
            m.update(planes(f, shape)[sl].ravel(), pen)
            o = mb.SeparableGaussianBlur(loc, taps=taps, ctx=ctx)
            return mb.mlsqr(o, m, planes(g, shape)[sl].ravel(), 5e-3, st)

        out = run_ranks(P, nz, fn)
        assert all(np.array_equal(o.alphas, ref.alphas) for o in out), (P, agg_planes)
        assert np.array_equal(np.concatenate([o.solution for o in out]), ref.solution), (P, agg_planes)
