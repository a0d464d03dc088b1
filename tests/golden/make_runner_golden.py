"""Record the REFERENCE's own `mlsqr run` artifacts as golden fixtures (tests/golden/runner_golden.npz).

Runs the unmodified reference harness (config.cpp + runner.cpp + the core, built by
`make -C oracle ref-runner` into oracle/_ref/mlsqr_ref_run) on
  * the five configurations the reference ships (proj/configs/*.json), and
  * variants written here that reach the remaining schema paths (cg_normal, laplacian
    regularizer, inner CG, explicit phantoms, a non-square grid, tau > 0 bases, S1/S2),
with both kernel backends (MLSQR_KERNELS=scalar and the default avx2: their spread is the
reference's own rounding floor), plus the reference's exit code and message for malformed
configurations.  Every artifact is parsed into arrays; the config texts are stored too, so the
GPU tests never read /root/reference.

Usage (in the build container):  make -C oracle ref-runner && python tests/golden/make_runner_golden.py
"""
from __future__ import annotations

import glob
import json
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_RUN = os.path.join(ROOT, "oracle", "_ref", "mlsqr_ref_run")
REF_CONFIGS = "/root/reference/proj/configs"

VARIANTS = {
    "deblur2d_cg_normal": {
        "problem": {"type": "deblur2d", "nx": 32, "ny": 32, "sigma_f": 0.04, "sigma_n": 0.01, "seed": 11},
        "solver": {"method": "cg_normal", "tau": 1e-2, "penalty": {"kind": "tv_smoothed", "T": 0.05},
                   "regularizer": "ideal", "stopping": {"criteria": ["S4"], "delta": 0.01, "eta": 1.1,
                                                        "max_iters": 60}},
        "output": {"directory": "out/x", "traces": True, "solutions": True, "basis_vectors": 3},
    },
    "deblur2d_nonsquare_lsqr": {
        "problem": {"type": "deblur2d", "nx": 40, "ny": 24, "sigma_f": 0.04, "sigma_n": 0.02, "seed": 5,
                    "phantom": [{"shape": "rect", "x0": 0.1, "y0": 0.2, "x1": 0.5, "y1": 0.7, "value": 1.0},
                                {"shape": "disk", "cx": 0.7, "cy": 0.5, "r": 0.15, "value": 0.5}]},
        "solver": {"method": "lsqr", "tau": 1e-3,
                   "stopping": {"criteria": ["S1", "S2"], "atol": 1e-6, "btol": 1e-6, "max_iters": 40}},
        "output": {"directory": "out/x", "traces": True, "solutions": True, "basis_vectors": 3},
    },
    "deconv1d_laplacian_innercg": {
        "problem": {"type": "deconv1d", "n": 256, "sigma_f": 0.02, "sigma_n": 0.01, "seed": 3,
                    "phantom": [[0.0, 0.0], [0.2, 1.0], [0.45, 0.3], [0.7, 0.0]]},
        "solver": {"method": "mlsqr", "tau": 0.05, "penalty": {"kind": "tikhonov"}, "regularizer": "laplacian",
                   "stopping": {"criteria": ["S4"], "delta": 0.01, "eta": 1.1, "max_iters": 60},
                   "spd": {"mode": "inner_cg", "k_inner": 12}, "epsilon": 1e-6},
        "output": {"directory": "out/x", "traces": True, "solutions": True, "basis_vectors": 2},
    },
    "deconv1d_nonlinear_innercg": {
        "problem": {"type": "deconv1d", "n": 256, "sigma_f": 0.02, "sigma_n": 0.01, "seed": 9},
        "solver": {"method": "lagged_diffusivity", "tau": 0.0, "penalty": {"kind": "tv_smoothed", "T": 0.01},
                   "stopping": {"criteria": ["S4"], "delta": 0.01, "eta": 1.1, "max_iters": 300},
                   "spd": {"mode": "inner_cg", "k_inner": 16}, "epsilon": "auto", "inner_cap": 15,
                   "rel_decrease_threshold": 0.1, "max_outer": 4},
        "output": {"directory": "out/x", "traces": True, "solutions": True, "outer_snapshots": True,
                   "basis_vectors": 2},
    },
    "deblur2d_traces_off": {
        "problem": {"type": "deblur2d", "nx": 32, "ny": 32, "sigma_f": 0.05, "sigma_n": 0.01, "seed": 2},
        "solver": {"method": "mlsqr", "tau": 0.0, "penalty": {"kind": "pm_log", "T": 0.05},
                   "stopping": {"criteria": ["S4"], "delta": 0.01, "eta": 1.1, "max_iters": 100},
                   "spd": {"mode": "cholesky"}},
        "output": {"directory": "out/x", "traces": False, "solutions": True},
    },
}

# malformed configurations: the reference's exit code and message are the contract
BAD = {
    "unknown_root_key": {"problem": {}, "solver": {}, "output": {}, "extra": 1},
    "bad_type": {"problem": {"type": "deblur3d", "n": 4, "sigma_f": 0.1, "sigma_n": 0.0, "seed": 0},
                 "solver": {}, "output": {}},
    "missing_key": {"problem": {"type": "deconv1d", "sigma_f": 0.1, "sigma_n": 0.0, "seed": 0},
                    "solver": {}, "output": {}},
    "bad_method": {"problem": {"type": "deconv1d", "n": 64, "sigma_f": 0.1, "sigma_n": 0.0, "seed": 0},
                   "solver": {"method": "gmres", "stopping": {"criteria": [], "max_iters": 5}},
                   "output": {"directory": "x"}},
    "penalty_required": {"problem": {"type": "deconv1d", "n": 64, "sigma_f": 0.1, "sigma_n": 0.0, "seed": 0},
                         "solver": {"method": "mlsqr", "stopping": {"criteria": ["S4"], "max_iters": 5}},
                         "output": {"directory": "x"}},
    "bad_eta": {"problem": {"type": "deconv1d", "n": 64, "sigma_f": 0.1, "sigma_n": 0.0, "seed": 0},
                "solver": {"method": "lsqr", "stopping": {"criteria": ["S4"], "eta": 1.0, "max_iters": 5}},
                "output": {"directory": "x"}},
    "bad_phantom": {"problem": {"type": "deconv1d", "n": 64, "sigma_f": 0.1, "sigma_n": 0.0, "seed": 0,
                                "phantom": [[0.5, 1.0]]},
                    "solver": {"method": "lsqr", "stopping": {"criteria": [], "max_iters": 5}},
                    "output": {"directory": "x"}},
    "bad_threshold": {"problem": {"type": "deconv1d", "n": 64, "sigma_f": 0.1, "sigma_n": 0.0, "seed": 0},
                      "solver": {"method": "lagged_diffusivity", "penalty": {"kind": "tikhonov"},
                                 "rel_decrease_threshold": 1.5,
                                 "stopping": {"criteria": [], "max_iters": 5}},
                      "output": {"directory": "x"}},
    "negative_n": {"problem": {"type": "deconv1d", "n": -3, "sigma_f": 0.1, "sigma_n": 0.0, "seed": 0},
                   "solver": {}, "output": {}},
    "not_json": "{ this is not json",
}


def read_csv(path):
    with open(path) as fh:
        header = fh.readline().strip()
    data = np.genfromtxt(path, delimiter=",", skip_header=1, dtype=np.float64)
    return header, np.atleast_2d(data)


def run_reference(cfg_path, out_dir, backend):
    env = dict(os.environ)
    if backend == "scalar":
        env["MLSQR_KERNELS"] = "scalar"
    else:
        env.pop("MLSQR_KERNELS", None)
    r = subprocess.run([REF_RUN, "--quiet", "--out", out_dir, "run", cfg_path], capture_output=True, text=True,
                       env=env)
    return r.returncode, r.stderr


def main():
    out = {}
    configs = {}
    for path in sorted(glob.glob(os.path.join(REF_CONFIGS, "*.json"))):
        with open(path) as fh:
            configs[os.path.splitext(os.path.basename(path))[0]] = fh.read()
    for name, doc in VARIANTS.items():
        configs[name] = json.dumps(doc, indent=1)
    out["names"] = np.array(sorted(configs))
    with tempfile.TemporaryDirectory() as tmp:
        for name, text in sorted(configs.items()):
            cfg_path = os.path.join(tmp, name + ".json")
            with open(cfg_path, "w") as fh:
                fh.write(text)
            out[f"{name}__config"] = np.array(text)
            for backend in ("scalar", "avx2"):
                od = os.path.join(tmp, f"{name}_{backend}")
                rc, err = run_reference(cfg_path, od, backend)
                assert rc == 0, (name, backend, err)
                files = sorted(os.listdir(od))
                pre = f"{name}__{backend}"
                out[pre + "__files"] = np.array(files)
                for f in files:
                    if f.endswith(".csv"):
                        header, data = read_csv(os.path.join(od, f))
                        out[f"{pre}__{f}__header"] = np.array(header)
                        out[f"{pre}__{f}"] = data
                with open(os.path.join(od, "meta.json")) as fh:
                    out[pre + "__meta"] = np.array(fh.read())
        bad_names = sorted(BAD)
        out["bad_names"] = np.array(bad_names)
        for name in bad_names:
            doc = BAD[name]
            cfg_path = os.path.join(tmp, "bad_" + name + ".json")
            with open(cfg_path, "w") as fh:
                fh.write(doc if isinstance(doc, str) else json.dumps(doc))
            rc, err = run_reference(cfg_path, os.path.join(tmp, "bad_out"), "scalar")
            out[f"bad__{name}__config"] = np.array(doc if isinstance(doc, str) else json.dumps(doc))
            out[f"bad__{name}__rc"] = np.array(rc)
            out[f"bad__{name}__stderr"] = np.array(err)
    path = os.path.join(HERE, "runner_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
