"""Per-step timing of OuterSolver.step with pinned host buffers vs device buffers (C2 size)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_6634_b200 as mb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
shape = (n, n)
ctx = mb.Context(0, stream=torch.cuda.current_stream().cuda_stream)
op = mb.SeparableGaussianBlur(shape, taps=mb.gaussian_taps(n, 3.0 / n, 9), ctx=ctx)
g = torch.rand(n * n, dtype=torch.float64, device="cuda")
cfg = mb.OuterConfig(tau=5e-3, penalty=mb.PenaltySpec.tv_smoothed(0.01),
                     inner_stop=mb.StoppingConfig.max_iterations(30), inner_cap=30,
                     rel_decrease_threshold=0.0, max_outer=5, mg_levels=5)
s = mb.OuterSolver(op, shape, 1.0 / n, cfg)
fa = torch.zeros_like(g)
fb = torch.empty_like(g)
for _ in range(3):
    s.step(g, fa, fb)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    s.step(g, fa, fb)
    torch.cuda.synchronize()
    print("device step ms", round(1e3 * (time.perf_counter() - t0), 2))
gh = torch.empty(n * n, dtype=torch.float64, pin_memory=True)
gh.copy_(g)
fph = torch.zeros(n * n, dtype=torch.float64, pin_memory=True)
foh = torch.empty(n * n, dtype=torch.float64, pin_memory=True)
for _ in range(4):
    t0 = time.perf_counter()
    s.step(gh.numpy(), fph.numpy(), foh.numpy())
    print("host step ms", round(1e3 * (time.perf_counter() - t0), 2))
    fph, foh = foh, fph
