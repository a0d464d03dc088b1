"""A/B of the fused 3D blur at C5 size (512^3, 13 taps) with its LSQR epilogue.

    python tools/blur_ab.py LIB [LIB ...]        # each LIB: a libmlsqr_b200.so build ('-' = in-tree)

For every build (own subprocess, MLSQR_LIB_PATH): 12 MLSQR iterations with per-class CUDA-event
timing on; prints the mean K_A / K_B blur launch (xpby + |u|^2 epilogue, the bench's shape), the
plain apply (no epilogue) and a sha256 of the iterate, so builds can be checked bit for bit."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import paper_1308_6634_b200 as mb
    n = int(os.environ.get("AB_N", "512"))
    shape = (n, n, n)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = mb.Context(0, stream=stream.cuda_stream)
    op = mb.SeparableGaussianBlur(shape, taps=mb.gaussian_taps(n, 2.0 / n, 6), ctx=ctx)
    gen = torch.Generator(device="cuda").manual_seed(7)
    x = torch.rand(n ** 3, dtype=torch.float64, device="cuda", generator=gen)
    y = torch.empty_like(x)
    for _ in range(3):
        op.apply(x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(20):
        op.apply(x, y)
    e1.record(stream)
    torch.cuda.synchronize()
    plain = e0.elapsed_time(e1) / 20
    hy = hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:16]
    vc = mb.VCycleMap(shape, 1.0 / n, 5, ctx=ctx)
    vc.update(x * 0.01, mb.PenaltySpec.tv_smoothed(0.01))
    g = op.apply(x)
    mb.mlsqr(op, vc, g, 5e-3, mb.StoppingConfig.max_iterations(2))
    ctx.set_timing(True)
    r = mb.mlsqr(op, vc, g, 5e-3, mb.StoppingConfig.max_iterations(12))
    torch.cuda.synchronize()
    ms, cnt = ctx.timing(mb.TCLASS["blur"])
    it_ms, it_n = ctx.timing(mb.TCLASS["iter"])
    ctx.set_timing(False)
    hf = hashlib.sha256(r.solution.cpu().numpy().tobytes()).hexdigest()[:16]
    nb = 3 * 8.0 * n ** 3
    print(json.dumps({"plain_ms": plain, "plain_gbs": 2 * 8.0 * n ** 3 / plain / 1e6, "epi_ms": ms / cnt,
                      "epi_gbs": nb / (ms / cnt) / 1e6, "launches": cnt, "iter_ms": it_ms / max(1, it_n),
                      "y_sha": hy, "f_sha": hf}))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        return child()
    for lib in sys.argv[1:] or ["-"]:
        env = dict(os.environ)
        name = lib
        if lib != "-":
            env["MLSQR_LIB_PATH"] = os.path.abspath(lib)
        else:
            name = "in-tree"
        out = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
        print(f"{name}: {line}", flush=True)


if __name__ == "__main__":
    main()
