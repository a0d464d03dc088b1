"""Small, fast driver for ncu: runs the C5-size (512^3) hot kernels a few times.

    python profiles/kernel_driver.py [--n 512] [--reps 3]

Phases (in launch order): 3D blur apply, V-cycle solve, 4 MLSQR iterations.
Used as the <cmd> of the ncu recipes in /opt/skills/guides/B200_PROFILING.md.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--time", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_1308_6634_b200 as mb
    n = a.n
    shape = (n, n, n)
    ctx = mb.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    taps = mb.gaussian_taps(n, 2.0 / n, 6)
    op = mb.SeparableGaussianBlur(shape, taps=taps, ctx=ctx)
    x = torch.rand(n ** 3, dtype=torch.float64, device="cuda")
    for _ in range(a.reps):
        y = op.apply(x)
    vc = mb.VCycleMap(shape, 1.0 / n, 5, ctx=ctx)
    vc.update(x * 0.01, mb.PenaltySpec.tv_smoothed(0.01))
    for _ in range(a.reps):
        v = vc.solve(y)
    g = op.apply(x)
    mb.mlsqr(op, vc, g, 5e-3, mb.StoppingConfig.max_iterations(a.iters))
    torch.cuda.synchronize()
    if a.time:
        def timed(fn, reps=10):
            fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps
        nb = 8.0 * n ** 3
        t_blur = timed(lambda: op.apply(x, y))
        t_vc = timed(lambda: vc.solve(y, v))
        print(f"blur apply: {t_blur:.3f} ms  ({2 * nb / t_blur / 1e6:.0f} GB/s on 2 vectors)")
        print(f"V-cycle   : {t_vc:.3f} ms")
        it_ms = timed(lambda: mb.mlsqr(op, vc, g, 5e-3, mb.StoppingConfig.max_iterations(20)), reps=2) / 20
        print(f"mlsqr iteration (20-it solve incl. init): {it_ms:.3f} ms")
    print("driver done", float(v[0]))


if __name__ == "__main__":
    main()
