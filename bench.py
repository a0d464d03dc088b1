#!/usr/bin/env python
"""bench.py -- priorconditioned LSQR iterations/sec (incl. MG V-cycle) on B200.

Workload (default --config c5): BASELINE.json configs[4], the north-star gate --
3D smoothed-TV deblurring of a 512^3 fp64 volume (64 seeded ellipsoids, Gaussian
blur sigma = 2 voxels / 13 taps, 1% noise, T = 0.01, tau = 5e-3, 5-level V-cycle).
One STEP = one lagged-diffusivity outer step of that config on the device:
D update + hierarchy + auto shift, 50 MLSQR iterations from zero (each with one
V(2,2) cycle), R(f).  value = LSQR iterations / s over the timed steps
(warm-up steps continue the same fixed-point iteration first).  Inputs are
resident in HBM before the timed region; every vector is 1.07 GB >> the 126 MB
L2, so no L2 flush is needed.

Extra keys: roofline (dominant kernel class, algorithmic bytes / CUDA-event
duration measured in an instrumented step right after the timed region),
iteration_roofline (SURVEY.md §8d canonical B_iter), cpu_baseline (the
reference's own mlsqr core from oracle/_ref driving the oracle's restated 3D
blur and V-cycle, 1 thread, bounded sample), e2e (host g / f_prev in pinned
memory -> device -> host f per step through the public OuterSolver API),
clocks (nvidia-smi sampled during the timed region), gpu_launches.

--impl reference: the reference's own CPU implementation of the path (same
config / metric), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

METRIC = "priorconditioned LSQR iterations/sec (incl. MG V-cycle)"
UNIT = "it/s"

CONFIGS = {
    "c1": dict(workload="C1 2D Tikhonov deblurring 128x128 fp64", dims=2, n=128, sigma_px=2.0, R=6,
               phantom="rects", count=8, noise=0.01, pen="tikhonov", T=1.0, tau=1e-2, K=1, I=50,
               levels=5, seed=1),
    "c2": dict(workload="C2 2D smoothed-TV deblurring 1024x1024 fp64", dims=2, n=1024, sigma_px=3.0,
               R=9, phantom="shapes", count=32, noise=0.01, pen="tv", T=0.01, tau=5e-3, K=5, I=30,
               levels=5, seed=2),
    "c3": dict(workload="C3 3D Perona-Malik deconvolution 128^3 fp64", dims=3, n=128, sigma_px=1.5,
               R=4, phantom="ellipsoids", count=10, semi=(8.0, 40.0), vals=(0.2, 1.0), noise=0.02,
               pen="pm_log", T=0.05, tau=1e-2, K=5, I=40, levels=5, seed=3),
    "c4": dict(workload="C4 3D fDOT-like dense reconstruction 64^3 x 4096 rows fp64", dims=3, n=64,
               kind="fdot", ns=64, nd=64, mu=1.0, phantom="ellipsoids", count=3, semi=(6.0, 6.0),
               vals=(1.0, 1.0), noise=0.01, pen="tv", T=0.01, tau=1e-3, K=8, I=50, levels=4, seed=4, R=0),
    "c5": dict(workload="C5 3D smoothed-TV deblurring 512^3 fp64 (north-star gate)", dims=3, n=512,
               sigma_px=2.0, R=6, phantom="ellipsoids", count=64, semi=(32.0, 160.0),
               vals=(0.2, 1.0), noise=0.01, pen="tv", T=0.01, tau=5e-3, K=10, I=50, levels=5, seed=5),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def canonical_bytes_per_iter(cfg) -> float:
    """B_iter = 8 (W_A + W_B + W_MG + W_U), kc = 4 coarse sweeps."""
    d = cfg["dims"]
    n = float(cfg["n"] ** d)
    dense = cfg.get("kind") == "fdot"
    m = float(cfg["ns"] * cfg["nd"]) if dense else n
    r = 2.0 ** -d
    L = cfg["levels"]
    kc = 4
    nl = [n * r ** l for l in range(L)]
    W_A = n + 2 * m + (m * n if dense else 0.0)
    W_B = m + 2 * n + (m * n if dense else 0.0)
    W_MG = (15 + 5 * d + 2 * r) * sum(nl[:-1]) + kc * (3 + d) * nl[-1]
    W_U = 8 * n
    return 8.0 * (W_A + W_B + W_MG + W_U)


def class_bytes(cfg, world=1):
    """Algorithmic bytes per launch of each timed kernel class (level-0 vectors, 8 B words).
    Single kernels: blur (K_A / K_B), dense (A x / A^T y), sweep_fn (pre-sweeps 1+2 fused),
    sweep_prolong (prolongation + post-sweep 1), sweep_last (post-sweep 2 + <v, p> partials),
    restrict (residual + restriction), update (K_U).  "smooth" is the class aggregate of the
    three level-0 smoothing kernels (their mean bytes per launch)."""
    d = cfg["dims"]
    n = float(cfg["n"] ** d)
    r = 2.0 ** -d
    m = float(cfg["ns"] * cfg["nd"]) if cfg.get("kind") == "fdot" else n
    fn = (1 + d) + 1          # b + d coefficient arrays -> x
    pro = 3 + d + r           # x, x_c, b, coefficients -> x
    last = 3 + d              # x, b, coefficients -> x
    return {
        "dense": 8.0 * (m * n + n + 2 * m),        # A x (or A^T y): the matrix once + the vectors
        "blur": 8.0 * 3 * n,                       # read x, read old, write out (m = n)
        "sweep_fn": 8.0 * n * fn,
        "sweep_prolong": 8.0 * n * pro,
        "sweep_last": 8.0 * n * last,
        "restrict": 8.0 * n * (2 + d + r),         # x, b, coefficients -> b_c
        "smooth": 8.0 * n * (fn + pro + last) / 3,
        "update": 8.0 * 8 * n,                     # read f w q v p, write f w q
    }


SINGLE_KERNELS = ("dense", "blur", "sweep_fn", "sweep_prolong", "sweep_last", "restrict", "update")


def measured_dram_per_iter():
    """DRAM bytes per LSQR iteration (dram__bytes_read.sum + dram__bytes_write.sum summed over a
    bench launch list, divided by its iterations) from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "dram_per_iter.json")) as fh:
            t = json.load(fh)
        return t["bytes_per_iter"], t["source"]
    except Exception:
        return None, None


def measured_traffic(kernel_class):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the class's
    level-0 kernels from the committed `ncu --set full` captures (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)
        return t["classes"][kernel_class]["bytes_per_launch"], t["source"]
    except Exception:
        return None, None


def make_problem(mb, cfg):
    """Seeded synthetic input of BASELINE's shapes (host generators of the library)."""
    n, d = cfg["n"], cfg["dims"]
    shape = (n,) * d
    N = n ** d
    if cfg["phantom"] == "rects":
        f = mb.phantom_rects2d(n, n, cfg["count"], cfg["seed"])
    elif cfg["phantom"] == "shapes":
        f = mb.phantom_shapes2d(n, n, cfg["count"], cfg["seed"])
    else:
        lo, hi = cfg["semi"]
        vlo, vhi = cfg["vals"]
        f = mb.phantom_ellipsoids3d(n, n, n, cfg["count"], lo, hi, vlo, vhi, cfg["seed"])
    taps = mb.gaussian_taps(n, cfg["sigma_px"] / n, cfg["R"])
    z = mb.gaussian_noise(cfg["seed"] + 1000, N, 1.0)
    return shape, taps, f, z


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region (the sampler
    is live before the region starts: rows from before it are dropped)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw,enforced.power.limit")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        def num(k):
            v = [float(r[k]) for r in self.rows if r[k].replace(".", "").isdigit()]
            return statistics.median(v) if v else None
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w": num(6), "power_limit_w": num(7)}


def cpu_reference_rate(cfg, iters: int, warm: int, threads_note: str):
    """The reference's own mlsqr (oracle/_ref, compiled from the reference sources) driving
    the oracle's restated blur / V-cycle through C callbacks, on this host's cores (1 thread:
    the reference has no threading).  Times iterations warm+1..warm+iters of the first outer
    step at the full config size; the init and warm-up iterations are excluded."""
    import pyoracle
    orc = pyoracle.Oracle()
    ref = pyoracle.Reference()
    n, d = cfg["n"], cfg["dims"]
    shape = (n,) * d
    N = n ** d
    dense = cfg.get("kind") == "fdot"
    if dense:
        # C4: the reference's own DenseOperator (linop.cpp:64-84) over the fDOT-like matrix
        _, _, a = orc.fdot(n, cfg["ns"], cfg["nd"], cfg["mu"], cfg["seed"])
        lo, hi = cfg["semi"]
        vlo, vhi = cfg["vals"]
        f = orc.ellipsoids3d(n, n, n, cfg["count"], lo, hi, vlo, vhi, cfg["seed"])
        od = ref.op_dense(a)
        M = a.shape[0]
        af = ref.apply(od, f, M)
        del f
        g = af + orc.gauss(cfg["seed"] + 1000, M, cfg["noise"] * float(np.abs(af).max()))
        del af
        grid = orc.grid(d, shape, 1.0 / n)
        cx, cy, cz = orc.edge_coeffs(grid, np.zeros(N), cfg["pen"], cfg["T"])
        eps = 1e-8 * orc.max_diag(grid, cx, cy, cz)
        mg = orc.vcycle(grid, cfg["levels"])
        mg.set(cx, cy, cz, eps)
        md = ref.map_callback(N, orc.solve_cb, mg.h)
        with pinned_core() as core:
            secs, done, _ = ref.mlsqr_timed(od, md, g, cfg["tau"], iters, warm, N)
        timed = done - warm
        return {"value": timed / secs if secs > 0 else None, "seconds": secs, "iterations": timed,
                "sample": f"first outer step of {cfg['workload']}: reference mlsqr + reference DenseOperator "
                          f"(oracle/_ref) iterations {warm + 1}..{done} at full size, V-cycle = oracle restatement; "
                          f"{threads_note}; {core}"}
    if cfg["phantom"] == "rects":
        f = orc.rects2d(n, n, cfg["count"], cfg["seed"])
    elif cfg["phantom"] == "shapes":
        f = orc.shapes2d(n, n, cfg["count"], cfg["seed"])
    else:
        lo, hi = cfg["semi"]
        vlo, vhi = cfg["vals"]
        f = orc.ellipsoids3d(n, n, n, cfg["count"], lo, hi, vlo, vhi, cfg["seed"])
    taps = orc.taps(n, cfg["sigma_px"] / n, radius=cfg["R"])
    op = orc.blur(d, shape, taps)
    af = op.apply(f)
    del f
    g = af + orc.gauss(cfg["seed"] + 1000, N, cfg["noise"] * float(np.abs(af).max()))
    del af
    grid = orc.grid(d, shape, 1.0 / n)
    cx, cy, cz = orc.edge_coeffs(grid, np.zeros(N), cfg["pen"], cfg["T"])  # outer step 1: f^0 = 0
    eps = 1e-8 * orc.max_diag(grid, cx, cy, cz)
    mg = orc.vcycle(grid, cfg["levels"])
    mg.set(cx, cy, cz, eps)
    del cx, cy, cz
    od = ref.op_callback(N, N, orc.apply_cb, orc.adjoint_cb, op.h)
    md = ref.map_callback(N, orc.solve_cb, mg.h)
    with pinned_core() as core:
        secs, done, _ = ref.mlsqr_timed(od, md, g, cfg["tau"], iters, warm, N)
    timed = done - warm
    return {"value": timed / secs if secs > 0 else None, "seconds": secs, "iterations": timed,
            "sample": f"first outer step of {cfg['workload']}: reference mlsqr (oracle/_ref) iterations "
                      f"{warm + 1}..{done} at full size, init + {warm} warm-up iteration(s) excluded; "
                      f"operators = oracle's restated {d}D blur + V-cycle (the reference has none); {threads_note}; "
                      f"{core}"}


class pinned_core:
    """Pin this process to one host core for the CPU reference timing (the reference
    has no threading, so one core is the reference); reports the core, nproc and the CPU model."""

    def __enter__(self):
        self.old = None
        core = 0
        try:
            self.old = os.sched_getaffinity(0)
            core = min(self.old)
            os.sched_setaffinity(0, {core})
        except Exception:
            pass
        model = "unknown CPU"
        try:
            with open("/proc/cpuinfo") as fh:
                model = next(l.split(":", 1)[1].strip() for l in fh if l.startswith("model name"))
        except Exception:
            pass
        return f"pinned to core {core} of nproc={os.cpu_count()} ({model})"

    def __exit__(self, *a):
        if self.old:
            try:
                os.sched_setaffinity(0, self.old)
            except Exception:
                pass


def reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # bounded: at most 4 timed iterations after 1 warm-up (~2-3 min single-core at 512^3)
    iters = max(1, min(args.steps, 4 if cfg["n"] >= 512 else 20))
    warm = max(0, min(args.warmup, 1 if cfg["n"] >= 512 else 3))
    r = cpu_reference_rate(cfg, iters, warm, "1 thread")
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": r["iterations"], "warmup": warm, "ms_per_step": 1000.0 * r["seconds"] / max(1, r["iterations"]),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; BASELINE.json shapes)",
        "config": {"workload": cfg["workload"], "step": "one reference LSQR iteration (A, A^T, one V-cycle)"},
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "reference", "sample": r["sample"]},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg)

    import torch
    import paper_1308_6634_b200 as mb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    # one dedicated stream for torch's input set-up, the library and the timing events
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx = mb.Context(local, stream=stream.cuda_stream)
    n = cfg["n"]
    h = 1.0 / n
    dense = cfg.get("kind") == "fdot"
    if world > 1:
        from paper_1308_6634_b200 import dist as pdist
        ctx.set_comm_nccl(pdist.broadcast_unique_id(dist, rank), rank, world)
        if dense:
            # row shards: rank k owns data rows [k m/P, (k+1) m/P); solution space replicated
            m_g = cfg["ns"] * cfg["nd"]
            ctx.set_row_shard(m_g, rank * m_g // world)
        else:
            # one global grid in z slabs: rank k owns planes [k n/P, (k+1) n/P)
            if cfg["dims"] != 3:
                raise SystemExit("multi-GPU slabs need a 3D config (c3 / c5)")
            z0, nzl = pdist.slab_plan(n, world, levels=cfg["levels"], radius=cfg["R"])[rank]
            ctx.set_slab(n, z0)

    # ---- inputs resident in HBM
    if dense:
        shape = (n, n, n)
        lo, hi = cfg["semi"]
        vlo, vhi = cfg["vals"]
        f_true = mb.phantom_ellipsoids3d(n, n, n, cfg["count"], lo, hi, vlo, vhi, cfg["seed"])
        op = mb.FdotOperator(n, cfg["ns"], cfg["nd"], mu=cfg["mu"], seed=cfg["seed"], ctx=ctx)
        m_g = cfg["ns"] * cfg["nd"]
        z = mb.gaussian_noise(cfg["seed"] + 1000, m_g, 1.0)
        if world > 1:
            z = np.ascontiguousarray(z[rank * m_g // world:(rank + 1) * m_g // world])
        taps = []
    else:
        shape, taps, f_true, z = make_problem(mb, cfg)
        if world > 1:
            plane = n * n
            f_true = np.ascontiguousarray(f_true[z0 * plane:(z0 + nzl) * plane])
            z = np.ascontiguousarray(z[z0 * plane:(z0 + nzl) * plane])
            shape = (n, n, nzl)
        op = mb.SeparableGaussianBlur(shape, taps=taps, ctx=ctx)
    N = int(np.prod(shape))
    f_d = torch.from_numpy(f_true).cuda()
    af = op.apply(f_d)
    amax = af.abs().max().reshape(1)
    if dist:
        dist.all_reduce(amax, op=dist.ReduceOp.MAX)
    sigma = cfg["noise"] * float(amax)
    g_d = af + sigma * torch.from_numpy(z).cuda()
    del af, f_d, z
    ocfg = mb.OuterConfig(tau=cfg["tau"], penalty=mb.PenaltySpec(cfg["pen"], cfg["T"]),
                          inner_stop=mb.StoppingConfig.max_iterations(cfg["I"]), inner_cap=cfg["I"],
                          rel_decrease_threshold=0.0, max_outer=cfg["K"], mg_levels=cfg["levels"])
    solver = mb.OuterSolver(op, shape, h, ocfg)
    fa = torch.zeros(N, dtype=torch.float64, device="cuda")
    fb = torch.empty_like(fa)
    torch.cuda.synchronize()

    def one_step():
        nonlocal fa, fb
        s = solver.step(g_d, fa, fb)
        fa, fb = fb, fa
        return s

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ctx.launch_count(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            iters += one_step().inner_iterations
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launch_count()
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # strong scaling: all ranks iterate the same global problem, count it once
    value = iters / (ms / 1000.0)

    # ---- instrumented step: per-kernel CUDA-event durations (eager launches, same stream)
    ctx.set_timing(True)
    one_step()
    torch.cuda.synchronize()
    cls_ms = {k: ctx.timing(c) for k, c in mb.TCLASS.items()}
    ctx.set_timing(False)
    # this rank's share: z slabs split everything; row shards split only the dense operator
    cb = {k: v / world if (not dense or k == "dense") else v for k, v in class_bytes(cfg, world).items()}
    peak, peak_src = peaks()
    # roofline: the single kernel with the largest summed time in the step (not a class average)
    cands = {k: cls_ms[k] for k in SINGLE_KERNELS if cls_ms[k][1] > 0}
    dom = max(cands, key=lambda k: cands[k][0])
    dms, dn = cands[dom]
    achieved = cb[dom] * dn / (dms / 1000.0) / 1e9 if dms > 0 else None
    n_iter = max(1, cls_ms["iter"][1])
    it_ms = cls_ms["iter"][0] / n_iter
    traffic, traffic_src = measured_traffic(dom) if world == 1 and args.config == "c5" else (None, None)
    per_class = {k: {"ms_per_launch": v[0] / v[1], "launches": v[1], "share_of_iter": v[0] / max(cls_ms["iter"][0], 1e-9),
                     "algorithmic_bytes": cb[k], "achieved_gbs": cb[k] / (v[0] / v[1] / 1e3) / 1e9,
                     "frac": cb[k] / (v[0] / v[1] / 1e3) / 1e9 / peak}
                 for k, v in cls_ms.items() if k in cb and v[1] > 0}
    comm = {k: {"ms_per_iter": cls_ms[k][0] / n_iter, "calls_per_iter": cls_ms[k][1] / n_iter}
            for k in ("halo", "coll")} if world > 1 else None
    b_iter = canonical_bytes_per_iter(cfg)
    dram_iter, dram_src = measured_dram_per_iter() if world == 1 and args.config == "c5" else (None, None)

    # ---- cross-N fingerprint: outer step 1 from f^0 = 0 (the step tests/golden/config_<cfg>.npz pins
    #      against the oracle), bitwise digest of alpha / beta and the whole f (slabs gathered)
    from paper_1308_6634_b200 import dist as pdist
    f0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    f1 = torch.empty_like(f0)
    s1 = solver.step(g_d, f0, f1)
    torch.cuda.synchronize()
    digest = pdist.step_digest(dist, f1, s1.alphas, s1.betas, rank, world, row_shards=dense)
    del f0, f1
    if digest is not None:
        fx = os.path.join(ROOT, "tests", "golden", f"config_{args.config}.npz")
        if os.path.exists(fx):
            import hashlib
            z = np.load(fx)
            digest["oracle_fixture"] = os.path.relpath(fx, ROOT)
            digest["matches_oracle_fixture"] = bool(
                str(z["s0_f_sha256"]) == digest["f_sha256"]
                and hashlib.sha256(np.ascontiguousarray(z["s0_alphas"], "<f8").tobytes()).hexdigest()
                == digest["alphas_sha256"]
                and hashlib.sha256(np.ascontiguousarray(z["s0_betas"], "<f8").tobytes()).hexdigest()
                == digest["betas_sha256"])

    # ---- e2e through the public API with host (pinned) buffers
    e2e = None
    if not args.no_e2e:
        gh = torch.empty(op.n_rows, dtype=torch.float64, pin_memory=True)
        gh.copy_(g_d)
        fph = torch.zeros(N, dtype=torch.float64, pin_memory=True)
        foh = torch.empty(N, dtype=torch.float64, pin_memory=True)
        solver_e = solver
        # untimed e2e warm-up: grows the C-ABI's host staging buffers once
        for _ in range(max(2, args.warmup)):
            solver_e.step(gh.numpy(), fph.numpy(), foh.numpy())
            fph, foh = foh, fph
        fph.zero_()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e_steps = max(1, args.steps)
        t0 = time.perf_counter()
        e_iters = 0
        for _ in range(e_steps):
            s = solver_e.step(gh.numpy(), fph.numpy(), foh.numpy())  # H2D g, f_prev; D2H f (sync)
            e_iters += s.inner_iterations
            fph, foh = foh, fph
        t1 = time.perf_counter()
        secs = t1 - t0
        if dist:
            t = torch.tensor([secs], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            secs = float(t.item())
        e2e = {"value": e_iters / secs, "unit": UNIT, "h2d_bytes_per_step": 8 * (op.n_rows + N) * world,
               "d2h_bytes_per_step": 8 * N * world, "steps": e_steps,
               "path": "mlsqr_outer_advance(ptr_kind=HOST): pinned g, f_prev -> HBM, f -> host, per step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            # N >= 3 timed iterations after one warm-up iteration
            r = cpu_reference_rate(cfg, 3, 1, "1 thread (the reference is single-threaded)")
            cpu = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "reference", "sample": r["sample"]}
        except Exception as e:  # never fail the bench line on the baseline leg
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded phantoms + Gaussian noise with BASELINE.json shapes)",
            "config": {"workload": cfg["workload"], "grid": [n] * cfg["dims"], "slab": list(shape),
                       "data_rows_local": op.n_rows, "taps": len(taps),
                       "step": f"one lagged-diffusivity outer step = {cfg['I']} MLSQR iterations "
                               f"(A, A^T, one V(2,2) {cfg['levels']}-level cycle each) + D update + R(f)",
                       "parallelism": "single GPU" if world == 1 else (
                           f"row shards x{world}: local A rows, allgathered A^T chunk partials, replicated V-cycle"
                           if dense else f"z-slabs x{world}: NCCL ghost planes + allgathered canonical tree partials"),
                       "l2": ("no flush needed: the %.2f GB matrix streamed by every A / A^T exceeds the 126 MB L2"
                              % (8.0 * op.n_rows * N / 1e9)) if dense else
                             "no flush needed: every vector (8 B x %d) exceeds the 126 MB L2" % N},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "algorithmic_bytes_per_launch": cb[dom], "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "note": "the single kernel with the largest summed time in an instrumented step: "
                                 "algorithmic bytes per launch / mean CUDA-event launch time"},
            "iteration_roofline": {"bytes_per_iter": b_iter, "model": "SURVEY.md 8d canonical B_iter",
                                   "achieved_gbs": b_iter * value / world / 1e9,
                                   "frac": b_iter * value / world / 1e9 / peak,
                                   "measured_dram_bytes_per_iter": dram_iter,
                                   "measured_dram_frac": (dram_iter * value / world / 1e9 / peak) if dram_iter else None,
                                   "measured_dram_source": dram_src},
            "kernel_classes_ms": {k: {"ms": v[0], "launches": v[1]} for k, v in cls_ms.items()},
            "class_rooflines": per_class,
            "comm": comm,
            "digest_outer_step1": digest,
            "instrumented_ms_per_iter": it_ms,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
