"""N > 1 host logic on CPU with a world-size-2 gloo group (no GPU): the slab plan is
consistent across ranks and covers the grid, the NCCL-unique-id broadcast mechanism
works, the ghost-plane exchange pattern delivers the neighbour planes, and the
distributed canonical reduction (block-aligned partials or raw segments, allgathered)
equals the oracle's single-process canonical dot bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1308_6634_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        # 1. slab plans agree and cover [0, nz)
        plan = pdist.slab_plan(512, world, levels=5, radius=6)
        plans = [None] * world
        dist.all_gather_object(plans, plan)
        res["plans_equal"] = all(p == plan for p in plans)
        res["covered"] = sorted(z for z0, n in plan for z in range(z0, z0 + n)) == list(range(512))
        # 2. unique-id broadcast (a stand-in token: NCCL needs a GPU box)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        res["uid_ok"] = obj[0] == bytes(range(128))
        # 3. ghost exchange pattern: send bottom/top planes, receive neighbour planes
        nx, ny, nz_loc = 8, 4, 6
        z0 = rank * nz_loc
        gen = np.random.default_rng(0)
        glob = gen.standard_normal((world * nz_loc, ny, nx))
        local = glob[z0:z0 + nz_loc]
        import torch
        lo = torch.zeros(ny * nx, dtype=torch.float64)
        hi = torch.zeros(ny * nx, dtype=torch.float64)
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(local[0].ravel().copy()), rank - 1))
            reqs.append(dist.irecv(lo, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(torch.from_numpy(local[-1].ravel().copy()), rank + 1))
            reqs.append(dist.irecv(hi, rank + 1))
        for r in reqs:
            r.wait()
        ok = True
        if rank > 0:
            ok &= np.array_equal(lo.numpy(), glob[z0 - 1].ravel())
        if rank + 1 < world:
            ok &= np.array_equal(hi.numpy(), glob[z0 + nz_loc].ravel())
        res["halo_ok"] = bool(ok)

        # 4. distributed canonical reduction, unaligned (raw segments) and aligned (blocks)
        def allgather(arr):
            t = torch.from_numpy(np.ascontiguousarray(arr))
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return [o.numpy() for o in out]

        for name, (L, rows_loc) in {"unaligned": (40, 30), "aligned": (1024, 1024)}.items():
            xg = np.random.default_rng(5).standard_normal(L * rows_loc * world)
            yg = np.random.default_rng(6).standard_normal(L * rows_loc * world)
            sl = slice(rank * L * rows_loc, (rank + 1) * L * rows_loc)
            segs = pdist.segments(xg[sl], yg[sl], L)
            res[name] = (pdist.dist_reduce(segs, allgather), xg.tobytes(), yg.tobytes(), L)
        # 5. the bench's cross-N fingerprint: slabs gathered in rank order hash like the whole
        #    vector, and alpha / beta hash identically on every rank
        import torch
        whole = np.random.default_rng(5).standard_normal(world * 1000)
        ab = np.random.default_rng(6).standard_normal(51)
        dg = pdist.step_digest(dist, torch.from_numpy(whole[rank * 1000:(rank + 1) * 1000].copy()), ab[:50], ab,
                               rank, world)
        res["digest"] = dg
        res["digest_whole"] = pdist.step_digest(None, torch.from_numpy(whole), ab[:50], ab, 0, 1)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_world2_gloo(orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        res = out[r]
        assert res["plans_equal"] and res["covered"] and res["uid_ok"] and res["halo_ok"]
        if r == 0:
            assert res["digest"] == res["digest_whole"]
        else:
            assert res["digest"] is None
        for name in ("unaligned", "aligned"):
            val, xb, yb, L = res[name]
            x = np.frombuffer(xb)
            y = np.frombuffer(yb)
            assert val == orc.canon_dot(x, y, L), name  # bit-exact vs single-process order
    assert out[0]["aligned"][0] == out[1]["aligned"][0]


def test_slab_plan_validation():
    assert pdist.slab_plan(512, 8, levels=5, radius=6) == [(64 * k, 64) for k in range(8)]
    with pytest.raises(ValueError):
        pdist.slab_plan(512, 3)
    with pytest.raises(ValueError):
        pdist.slab_plan(64, 8, levels=5)      # 8-plane slabs cannot halve 4 times
    with pytest.raises(ValueError):
        pdist.slab_plan(32, 8, levels=1, radius=6)  # 4-plane slab < 6-plane blur halo
