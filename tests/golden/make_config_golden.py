"""Offline fixtures for the BASELINE configs that are too large for the oracle at test time.

    python tests/golden/make_config_golden.py c5      # 512^3, first 2 outer steps x 50 (~1 h, 1 core)
    python tests/golden/make_config_golden.py c4      # fDOT 64^3 x 4096, all 8 outer steps x 50

TEST INFRASTRUCTURE ONLY.  Runs the oracle's DEVICE-order restatement (oracle/liborc.so,
`orc_set_device_order(1)`) of the fixed-count lagged-diffusivity loop (outer.cpp:58-96 minus the
stagnation break; mlsqr krylov.cpp:335-440 inside) on exactly the inputs bench.py builds for
the config (BASELINE.json configs[3] / configs[4]), and stores, per outer step, what a GPU run
must reproduce bit for bit:
  eps_used, penalty_value (R(f^k)), alphas[I], betas[I+1], and a digest of the iterate f^k
  (sha256 of the little-endian fp64 bytes, its l2 norm, and 4096 strided samples).
The input g is digested too, so a test can tell an input mismatch from a solver mismatch.
tests/test_gpu_configs.py::test_c5_first_outer_steps_bit_exact / test_c4_full_config_bit_exact
compare the device against these files.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

import pyoracle  # noqa: E402
from bench import CONFIGS  # noqa: E402  (the single source of the bench workloads)

NSAMPLES = 4096


def digest(v: np.ndarray) -> dict:
    v = np.ascontiguousarray(v, dtype="<f8")
    stride = max(1, v.size // NSAMPLES)
    return {"sha256": hashlib.sha256(v.tobytes()).hexdigest(), "l2": float(np.sqrt(np.dot(v, v))),
            "stride": stride, "samples": v[::stride][:NSAMPLES].copy()}


def path(name: str) -> str:
    return os.path.join(ROOT, "tests", "golden", f"config_{name}.npz")


def save(name: str, cfg: dict, K: int, g: np.ndarray, rep: dict, secs: float) -> None:
    out = {"config": np.array(name), "outer_steps": np.array(K), "inner": np.array(cfg["I"]),
           "seconds": np.array(secs)}
    dg = digest(g)
    out["g_sha256"], out["g_l2"] = np.array(dg["sha256"]), np.array(dg["l2"])
    I = cfg["I"]
    for k in range(rep["n_steps"]):
        s = rep["steps"][k]
        out[f"s{k}_eps"] = np.array(s["eps_used"])
        out[f"s{k}_R"] = np.array(s["penalty_value"])
        out[f"s{k}_iters"] = np.array(s["inner_iterations"])
        out[f"s{k}_alphas"] = rep["alphas"][k][:I].copy()
        out[f"s{k}_betas"] = rep["betas"][k][:I + 1].copy()
        d = digest(rep["iterates"][k])
        out[f"s{k}_f_sha256"], out[f"s{k}_f_l2"] = np.array(d["sha256"]), np.array(d["l2"])
        out[f"s{k}_f_stride"], out[f"s{k}_f_samples"] = np.array(d["stride"]), d["samples"]
    np.savez_compressed(path(name), **out)
    print(f"wrote {path(name)} ({secs:.0f} s)", flush=True)


def make_c5(orc, K: int) -> None:
    cfg = CONFIGS["c5"]
    n, d = cfg["n"], cfg["dims"]
    N = n ** d
    shape = (n,) * d
    lo, hi = cfg["semi"]
    vlo, vhi = cfg["vals"]
    t0 = time.time()
    f = orc.ellipsoids3d(n, n, n, cfg["count"], lo, hi, vlo, vhi, cfg["seed"])
    taps = orc.taps(n, cfg["sigma_px"] / n, radius=cfg["R"])
    op = orc.blur(3, shape, taps)
    af = op.apply(f)
    del f
    # bench.py: g = A f + (noise * max|A f|) * z,  z = N(0, 1) from seed + 1000
    g = af + (cfg["noise"] * float(np.abs(af).max())) * orc.gauss(cfg["seed"] + 1000, N, 1.0)
    del af
    print(f"c5 inputs ready ({time.time() - t0:.0f} s)", flush=True)
    rep = orc.nonlinear(op, g, orc.grid(d, shape, 1.0 / n), tau=cfg["tau"], pen=cfg["pen"], T=cfg["T"],
                        inner_stop=pyoracle.stop(cfg["I"]), inner_cap=cfg["I"], max_outer=K, threshold=0.0,
                        levels=cfg["levels"], keep=True)
    assert rep["status"] == 0 and rep["n_steps"] == K, rep["status"]
    save("c5", cfg, K, g, rep, time.time() - t0)


def make_c4(orc, K: int) -> None:
    cfg = CONFIGS["c4"]
    n = cfg["n"]
    N = n ** 3
    ns, nd = cfg["ns"], cfg["nd"]
    t0 = time.time()
    _, _, a = orc.fdot(n, ns, nd, cfg["mu"], cfg["seed"])
    lo, hi = cfg["semi"]
    vlo, vhi = cfg["vals"]
    f = orc.ellipsoids3d(n, n, n, cfg["count"], lo, hi, vlo, vhi, cfg["seed"])
    op = orc.dense(a).set_row_lengths(ns * nd, n)
    af = op.apply(f)
    g = af + (cfg["noise"] * float(np.abs(af).max())) * orc.gauss(cfg["seed"] + 1000, ns * nd, 1.0)
    print(f"c4 inputs ready ({time.time() - t0:.0f} s)", flush=True)
    rep = orc.nonlinear(op, g, orc.grid(3, (n, n, n), 1.0 / n), tau=cfg["tau"], pen=cfg["pen"], T=cfg["T"],
                        inner_stop=pyoracle.stop(cfg["I"]), inner_cap=cfg["I"], max_outer=K, threshold=0.0,
                        levels=cfg["levels"], keep=True)
    assert rep["status"] == 0 and rep["n_steps"] == K, rep["status"]
    save("c4", cfg, K, g, rep, time.time() - t0)


def main() -> None:
    which = sys.argv[1] if len(sys.argv) > 1 else "c5"
    orc = pyoracle.Oracle()
    orc.set_device_order(True)
    if which == "c5":
        make_c5(orc, int(sys.argv[2]) if len(sys.argv) > 2 else 2)
    elif which == "c4":
        make_c4(orc, int(sys.argv[2]) if len(sys.argv) > 2 else CONFIGS["c4"]["K"])
    else:
        raise SystemExit(f"unknown config {which}")


if __name__ == "__main__":
    main()
