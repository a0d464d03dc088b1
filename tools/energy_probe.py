"""Power / clock / energy per launch of the C5 building blocks (512^3), each looped ~4 s while
nvidia-smi samples power.draw and clocks.sm:  python tools/energy_probe.py"""
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1308_6634_b200 as mb  # noqa: E402


def sample(fn, secs=4.0):
    rows = []
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=subprocess.PIPE, text=True)
    th = threading.Thread(target=lambda: [rows.append(l) for l in p.stdout], daemon=True)
    th.start()
    fn()  # warm
    torch.cuda.synchronize()
    n = 0
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.perf_counter() - t0 < secs:
        fn()
        n += 1
        if n % 8 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    p.terminate()
    ms = e0.elapsed_time(e1) / n
    vals = [tuple(float(x) for x in r.split(",")) for r in rows[len(rows) // 4:] if r.count(",") == 1]
    pw = sum(v[0] for v in vals) / max(1, len(vals))
    clk = sum(v[1] for v in vals) / max(1, len(vals))
    return ms, pw, clk


def main():
    n = 512
    shape = (n, n, n)
    ctx = mb.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    op = mb.SeparableGaussianBlur(shape, taps=mb.gaussian_taps(n, 2.0 / n, 6), ctx=ctx)
    x = torch.rand(n ** 3, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    vc = mb.VCycleMap(shape, 1.0 / n, 5, ctx=ctx)
    vc.update(x * 0.01, mb.PenaltySpec.tv_smoothed(0.01))
    v = torch.empty_like(x)
    g = op.apply(x)
    big = torch.empty(2 * n ** 3, dtype=torch.float64, device="cuda")
    cases = {
        "copy 2 GB (torch, DRAM reference)": lambda: big[: n ** 3].copy_(big[n ** 3:]),
        "blur apply": lambda: op.apply(x, y),
        "V-cycle": lambda: vc.solve(y, v),
        "mlsqr 10 it (per it)": lambda: mb.mlsqr(op, vc, g, 5e-3, mb.StoppingConfig.max_iterations(10)),
    }
    for name, fn in cases.items():
        ms, pw, clk = sample(fn)
        per = ms / 10 if "10 it" in name else ms
        print(f"{name:36s} {per:8.3f} ms  {pw:7.1f} W  {clk:6.0f} MHz  {pw * per / 1e3:7.3f} J/launch")


if __name__ == "__main__":
    main()
