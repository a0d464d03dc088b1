"""Host-side logic of the z-slab decomposition.

One process per GPU.  Rank k owns planes [k nz/P, (k+1) nz/P) of the global 3D grid.
Ghost planes (blur radius R for A / A^T, one plane for every V-cycle level) travel over
NCCL send/recv.  The canonical reductions allgather block-aligned tree partials, so every
rank holds the same scalars and the result is bit-identical for any P
(tests/test_gpu_sharded.py checks this on one GPU with the loopback communicator).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def slab_plan(nz: int, world: int, levels: int = 1, radius: int = 0) -> List[Tuple[int, int]]:
    """(z_offset, nz_local) per rank.  Every level's local extent must stay integral and
    even-aligned (restriction pairs fine planes); a slab must be at least as thick as
    the ghost width it provides to its neighbours."""
    if world < 1 or nz % world:
        raise ValueError(f"nz={nz} must split evenly over {world} ranks")
    loc = nz // world
    f = 1 << max(levels - 1, 0)
    if loc % f:
        raise ValueError(f"slab of {loc} planes does not halve {levels - 1} times")
    if world > 1 and loc < max(radius, 1):
        raise ValueError(f"slab of {loc} planes is thinner than the {radius}-plane halo")
    if world > 1 and loc // f < 1:
        raise ValueError("coarsest level has no plane on some rank")
    return [(k * loc, loc) for k in range(world)]


def broadcast_unique_id(dist, rank: int) -> bytes:
    """rank 0 creates the NCCL unique id; torch.distributed broadcasts it."""
    obj = [None]
    if rank == 0:
        import paper_1308_6634_b200 as mb
        obj[0] = mb.nccl_unique_id()
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def sharded_context(device: int, rank: int, world: int, nz_global: int, unique_id: bytes,
                    stream=None):
    """Context of rank `rank` owning its slab of a global grid with nz_global planes, over NCCL.
    At world 1 the slab is the whole grid, and the decomposed code path still runs (ghost
    exchanges without neighbours, one-rank NCCL collectives inside the captured graph)."""
    import paper_1308_6634_b200 as mb
    ctx = mb.Context(device, stream=stream)
    z0, _ = slab_plan(nz_global, world)[rank]
    ctx.set_comm_nccl(unique_id, rank, world)
    ctx.set_slab(nz_global, z0)
    return ctx


def step_digest(dist, f_local, alphas, betas, rank: int, world: int, row_shards: bool = False) -> dict | None:
    """Bitwise fingerprint of one outer step, comparable across GPU counts (bench.py prints it
    at every N, so N = 1 vs N = 8 equality can be read from the driver's records).

    f_local: this rank's slab of the iterate (a torch tensor; z slabs are equal-sized and
    concatenate in rank order) or, with row shards, the replicated solution (rank 0's copy
    is hashed).  alphas / betas are replicated on every rank.  Returns the digest on rank 0,
    None elsewhere."""
    import hashlib

    import torch

    if dist is not None and world > 1 and not row_shards:
        if f_local.is_cuda:  # NCCL: all_gather into rank-ordered slabs
            parts = [torch.empty_like(f_local) for _ in range(world)]
            dist.all_gather(parts, f_local)
        else:  # gloo
            parts = [torch.empty_like(f_local) for _ in range(world)] if rank == 0 else None
            dist.gather(f_local, parts, dst=0)
        if rank != 0:
            return None
        f = torch.cat(parts)
    else:
        if rank != 0:
            return None
        f = f_local
    fh = np.ascontiguousarray(f.detach().cpu().numpy(), dtype="<f8")
    a = np.ascontiguousarray(alphas, dtype="<f8")
    b = np.ascontiguousarray(betas, dtype="<f8")
    return {"f_sha256": hashlib.sha256(fh.tobytes()).hexdigest(), "f_l2": float(np.sqrt(np.dot(fh, fh))),
            "alphas_sha256": hashlib.sha256(a.tobytes()).hexdigest(),
            "betas_sha256": hashlib.sha256(b.tobytes()).hexdigest(), "n_alphas": int(a.size)}


# ---------------------------------------------------------------------------
# CPU model of the distributed canonical reduction (documentation + gloo tests)
# ---------------------------------------------------------------------------
def tree32(v: np.ndarray) -> float:
    v = list(v) + [0.0] * (32 - len(v))
    off = 16
    while off >= 1:
        for l in range(off):
            v[l] = v[l] + v[l + off]
        off //= 2
    return v[0]


def segments(x: np.ndarray, y: np.ndarray, row_len: int) -> np.ndarray:
    """per-32-element row segment partials of x*y (the kernels' level 0)."""
    rows = x.size // row_len
    chunks = (row_len + 31) // 32
    prod = (x * y).reshape(rows, row_len)
    out = np.empty(rows * chunks)
    for r in range(rows):
        for c in range(chunks):
            out[r * chunks + c] = tree32(prod[r, 32 * c:32 * c + 32])
    return out


def levels(vals: np.ndarray, nlev: int | None = None) -> np.ndarray:
    """tree-32 levels over consecutive partials (zero padded), until one value remains
    or `nlev` levels were applied."""
    v = np.asarray(vals, dtype=np.float64)
    k = 0
    while (nlev is None and v.size > 1) or (nlev is not None and k < nlev):
        G = (v.size + 31) // 32
        v = np.array([tree32(v[32 * g:32 * g + 32]) for g in range(G)])
        k += 1
        if nlev is None and v.size == 1:
            break
    return v


def dist_reduce(local_segments: np.ndarray, allgather) -> float:
    """What reduce_segments_dist does: block-aligned ranks reduce their 32768-blocks
    (3 levels) and allgather the partials; otherwise the raw segments are gathered."""
    J = local_segments.size
    if J % 32768 == 0:
        part = np.concatenate([levels(local_segments[b * 32768:(b + 1) * 32768], 3) for b in range(J // 32768)])
        gathered = np.concatenate(allgather(part))
    else:
        gathered = np.concatenate(allgather(local_segments))
    return float(levels(gathered)[0]) if gathered.size > 1 else float(levels(gathered, 1)[0])
