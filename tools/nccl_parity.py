#!/usr/bin/env python
"""Multi-GPU parity over NCCL: a BASELINE config solved on N ranks (one GPU each) must equal the
one-GPU solve bit for bit (canonical reductions are decomposition-invariant).

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port 29511 tools/nccl_parity.py --config c3 --outer 2

c3 / c5: z slabs (ghost planes + allgathered tree partials); c4: row shards of the dense
operator.  Every rank runs its share through the library's NCCL transport (the same code path
`bench.py --gpus N` times); rank 0 then solves the whole problem on a plain one-GPU context and
compares alpha / beta of every outer step and the gathered iterate bitwise.  Per-iteration
halo / collective time (CUDA events) is reported from an instrumented second solve.
MLSQR_NO_GRAPH=1 runs the same launches without graph capture (to bisect a capture failure).
At N = 1 the slab context still runs the decomposed path on a one-rank communicator.
Prints one JSON line on rank 0; exit code 0 iff bit-exact.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS, make_problem  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=["c3", "c4", "c5"])
    ap.add_argument("--outer", type=int, default=2)
    ap.add_argument("--inner", type=int, default=0, help="LSQR iterations per outer step (0: the config's)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    import torch
    import torch.distributed as dist

    import paper_1308_6634_b200 as mb
    from paper_1308_6634_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    n = cfg["n"]
    h = 1.0 / n
    I = args.inner or cfg["I"]
    ocfg = mb.OuterConfig(tau=cfg["tau"], penalty=mb.PenaltySpec(cfg["pen"], cfg["T"]),
                          inner_stop=mb.StoppingConfig.max_iterations(I), inner_cap=I,
                          rel_decrease_threshold=0.0, max_outer=args.outer, mg_levels=cfg["levels"])
    uid = pdist.broadcast_unique_id(dist, rank)
    dense = cfg.get("kind") == "fdot"

    def build(ctx, sharded):
        if dense:
            m_g = cfg["ns"] * cfg["nd"]
            op = mb.FdotOperator(n, cfg["ns"], cfg["nd"], mu=cfg["mu"], seed=cfg["seed"], ctx=ctx)
            f_true = mb.phantom_ellipsoids3d(n, n, n, cfg["count"], *cfg["semi"], *cfg["vals"], cfg["seed"])
            af = mb.FdotOperator(n, cfg["ns"], cfg["nd"], mu=cfg["mu"], seed=cfg["seed"]).apply(f_true)
            g = af + cfg["noise"] * np.abs(af).max() * mb.gaussian_noise(cfg["seed"] + 1000, m_g, 1.0)
            if sharded:
                g = np.ascontiguousarray(g[rank * m_g // world:(rank + 1) * m_g // world])
            return op, g, (n, n, n)
        shape, taps, f_true, z = make_problem(mb, cfg)
        af = mb.SeparableGaussianBlur(shape, taps=taps).apply(f_true)
        g = af + cfg["noise"] * np.abs(af).max() * z
        if sharded:
            z0, nzl = pdist.slab_plan(n, world, levels=cfg["levels"], radius=cfg["R"])[rank]
            plane = n * n
            g = np.ascontiguousarray(g[z0 * plane:(z0 + nzl) * plane])
            shape = (n, n, nzl)
        return mb.SeparableGaussianBlur(shape, taps=taps, ctx=ctx), g, shape

    ctx = mb.Context(local)
    ctx.set_comm_nccl(uid, rank, world)
    if dense:
        m_g = cfg["ns"] * cfg["nd"]
        ctx.set_row_shard(m_g, rank * m_g // world)
    else:
        z0, _ = pdist.slab_plan(n, world, levels=cfg["levels"], radius=cfg["R"])[rank]
        ctx.set_slab(n, z0)
    op, g, shape = build(ctx, True)
    rep = mb.solve_nonlinear(op, g, shape if not dense else (n, n, n), h, ocfg)
    ctx.set_timing(True)
    mb.solve_nonlinear(op, g, shape if not dense else (n, n, n), h, ocfg)
    t = {k: ctx.timing(mb.TCLASS[k]) for k in ("iter", "halo", "coll")}
    ctx.set_timing(False)
    f_local = torch.from_numpy(np.ascontiguousarray(rep.solution)).cuda()
    if dense or world == 1:
        f_all = f_local
    else:
        parts = [torch.empty_like(f_local) for _ in range(world)]
        dist.all_gather(parts, f_local)
        f_all = torch.cat(parts)
    ok = True
    line = None
    if rank == 0:
        op1, g1, shape1 = build(mb.Context(local), False)
        ref = mb.solve_nonlinear(op1, g1, shape1, h, ocfg)
        same_f = bool(np.array_equal(f_all.cpu().numpy(), ref.solution))
        same_ab = [bool(np.array_equal(a.alphas, b.alphas) and np.array_equal(a.betas, b.betas))
                   for a, b in zip(rep.steps, ref.steps)]
        ok = same_f and all(same_ab) and len(rep.steps) == len(ref.steps)
        it = max(1, t["iter"][1])
        line = {"config": args.config, "world": world, "decomposition": "row shards" if dense else "z slabs",
                "outer": args.outer, "inner": I, "bit_exact": ok, "f_equal": same_f, "alpha_beta_equal": same_ab,
                "graph": os.environ.get("MLSQR_NO_GRAPH", "0") in ("", "0"),
                "ms_per_iter_instrumented": t["iter"][0] / it,
                "halo_ms_per_iter": t["halo"][0] / it, "coll_ms_per_iter": t["coll"][0] / it}
        print(json.dumps(line), flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if int(flag.item()) == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
