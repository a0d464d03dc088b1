"""The B200 harness `mlsqr-b200 run | compare` (paper_1308_6634_b200/runner/mlsqr_b200_run.cpp)
against the reference's own harness on the paths that need no GPU: the configuration schema
(config.cpp:1-309) -- same exit code (tools/main.cpp:13-16) and the same message for every
malformed configuration the reference was run on (tests/golden/make_runner_golden.py) -- usage
errors, and no CPU fallback for a valid configuration."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNNER = os.path.join(ROOT, "paper_1308_6634_b200", "mlsqr-b200")
GOLDEN = os.path.join(ROOT, "tests", "golden", "runner_golden.npz")


@pytest.fixture(scope="module")
def runner():
    if not os.path.exists(RUNNER):
        from paper_1308_6634_b200.build import build
        build(verbose=False)
    return RUNNER


@pytest.fixture(scope="module")
def rg():
    return np.load(GOLDEN)


def run(runner, *args, cwd=None):
    return subprocess.run([runner, *args], capture_output=True, text=True, cwd=cwd, timeout=120)


def test_config_errors_match_reference(runner, rg, tmp_path):
    names = list(rg["bad_names"])
    assert len(names) >= 10
    for name in names:
        p = tmp_path / f"{name}.json"
        p.write_text(str(rg[f"bad__{name}__config"]))
        r = run(runner, "--quiet", "--out", str(tmp_path / "o"), "run", str(p))
        assert r.returncode == int(rg[f"bad__{name}__rc"]) == 3, (name, r.stderr)
        assert r.stderr == str(rg[f"bad__{name}__stderr"]), name


def test_usage_and_missing_file(runner, tmp_path):
    assert run(runner).returncode == 2
    assert run(runner, "run").returncode == 2
    assert run(runner, "frobnicate", "x").returncode == 2
    r = run(runner, "run", str(tmp_path / "nope.json"))
    assert r.returncode == 2 and "config file not found" in r.stderr
    assert run(runner, "--help").returncode == 0


def test_compare_requires_identical_problems(runner, rg, tmp_path):
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    a.write_text(str(rg["deconv1d_ideal__config"]))
    b.write_text(str(rg["deblur2d_ideal__config"]))
    r = run(runner, "--quiet", "--out", str(tmp_path / "c"), "compare", str(a), str(b))
    assert r.returncode == 3 and r.stderr == "config error: compare requires identical problem sections\n"


def test_valid_config_has_no_cpu_fallback(runner, rg, tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    p = tmp_path / "c.json"
    p.write_text(str(rg["deconv1d_lsqr__config"]))
    r = run(runner, "--quiet", "--out", str(tmp_path / "o"), "run", str(p))
    assert r.returncode == 1 and "no CUDA device" in r.stderr
