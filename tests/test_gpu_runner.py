"""`mlsqr-b200 run` on the B200 against the reference's own `mlsqr run` artifacts
(tests/golden/runner_golden.npz: the five shipped configurations + variants, both reference
backends).  Checked per configuration: the artifact set (runner.cpp:55-121, 245-299), CSV headers
and grid columns (bit-exact), the meta.json schema and its config / derived sections, the stop
reason and iteration counts (equal to one of the reference's backends), and every numeric column
within north_star's reconstruction tolerance (1e-6 relative l2) or, where the reference's own two
backends already disagree by more, 25 x that scalar-vs-AVX2 spread."""
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNNER = os.path.join(ROOT, "paper_1308_6634_b200", "mlsqr-b200")
RG = np.load(os.path.join(ROOT, "tests", "golden", "runner_golden.npz"))
NAMES = [str(n) for n in RG["names"]]


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    m = np.isfinite(b)
    assert np.array_equal(m, np.isfinite(a))
    return np.linalg.norm(a[m] - b[m]) / max(np.linalg.norm(b[m]), 1e-300)


def read_csv(path):
    with open(path) as fh:
        header = fh.readline().strip()
    return header, np.atleast_2d(np.genfromtxt(path, delimiter=",", skip_header=1, dtype=np.float64))


def close(ours, sc, av, what):
    floor = rel(av, sc) if sc.shape == av.shape else 1.0
    tol = max(1e-6, 25 * floor)
    err = rel(ours, sc) if ours.shape == sc.shape else np.inf
    if ours.shape == av.shape:
        err = min(err, rel(ours, av))
    assert err <= tol, f"{what}: rel {err:.3e} > {tol:.3e} (reference floor {floor:.3e})"


@pytest.mark.parametrize("name", NAMES)
def test_runner_artifacts_match_reference(name, tmp_path):
    cfg = tmp_path / "cfg.json"
    cfg.write_text(str(RG[f"{name}__config"]))
    out = tmp_path / "out"
    r = subprocess.run([RUNNER, "--quiet", "--out", str(out), "run", str(cfg)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    files = sorted(os.listdir(out))
    sc_files, av_files = list(RG[f"{name}__scalar__files"]), list(RG[f"{name}__avx2__files"])
    assert files in (sc_files, av_files), (files, sc_files)
    ref = "scalar" if files == sc_files else "avx2"
    meta = json.load(open(out / "meta.json"))
    metas = {b: json.loads(str(RG[f"{name}__{b}__meta"])) for b in ("scalar", "avx2")}
    m0 = metas[ref]
    assert set(meta) == set(m0)
    for sec in ("config", "derived", "result"):
        assert set(meta[sec]) == set(m0[sec]), sec
    assert meta["config"] == m0["config"]
    assert meta["derived"]["data_cell_measure"] == m0["derived"]["data_cell_measure"]
    assert meta["derived"]["delta_euclid"] == m0["derived"]["delta_euclid"]
    assert len(meta["derived"]["epsilon_used"]) == len(m0["derived"]["epsilon_used"])
    assert rel(meta["derived"]["epsilon_used"], m0["derived"]["epsilon_used"]) <= 1e-14
    res = meta["result"]
    counts = [(m["result"]["stop_reason"], m["result"]["inner_iterations"], m["result"]["outer_iterations"])
              for m in metas.values()]
    # the reference's two backends agree on the iteration path for every configuration but the
    # shipped lagged-diffusivity one (exact Cholesky M^-1, 25 outer steps: 57 vs 38 inner
    # iterations); there the first outer step must agree and the counts lie in their span
    stable = counts[0] == counts[1]
    if stable:
        assert (res["stop_reason"], res["inner_iterations"], res["outer_iterations"]) == counts[0]
        assert res["inner_stop_reasons"] == metas["scalar"]["result"]["inner_stop_reasons"]
    else:
        assert res["stop_reason"] in {c[0] for c in counts}
        assert min(c[2] for c in counts) <= res["outer_iterations"] <= max(c[2] for c in counts)
        assert min(c[1] for c in counts) - 2 <= res["inner_iterations"] <= max(c[1] for c in counts) + 2
    for key in ("final_residual", "final_error", "final_penalty"):
        close(np.array([res[key]]), np.array([metas["scalar"]["result"][key]]),
              np.array([metas["avx2"]["result"][key]]), key)
    for f in files:
        if not f.endswith(".csv"):
            continue
        header, data = read_csv(out / f)
        assert header == str(RG[f"{name}__{ref}__{f}__header"]), f
        sc = RG[f"{name}__scalar__{f}"] if f in sc_files else None
        av = RG[f"{name}__avx2__{f}"] if f in av_files else None
        base = sc if sc is not None else av
        if f == "trace.csv":
            assert data.shape[1] == 9
            if stable:
                assert data.shape[0] in [x.shape[0] for x in (sc, av) if x is not None]
                k = min(x.shape[0] for x in (sc, av) if x is not None)
            else:  # the first outer step (rows with outer_k <= 1)
                k = int(np.sum(sc[:, 0] <= 1))
                assert k == int(np.sum(av[:, 0] <= 1)) == int(np.sum(data[:, 0] <= 1))
            other = av if av is not None else sc
            assert np.array_equal(data[:k, :2], base[:k, :2])  # outer_k, inner_i
            for c in range(2, 9):
                close(data[:k, c], base[:k, c], other[:k, c], f"{f} column {c}")
        else:
            assert data.shape == base.shape, f
            ncoord = data.shape[1] - (2 if f.startswith("solution") else 1)
            assert np.array_equal(data[:, :ncoord], base[:, :ncoord]), f  # grid coordinates
            if f.startswith("solution"):
                assert np.array_equal(data[:, -1], base[:, -1]), f  # f_true
                col = data.shape[1] - 2
            else:
                col = data.shape[1] - 1
            other = av if av is not None and av.shape == base.shape else base
            if not stable and f.startswith("solution_outer_") and f != "solution_outer_001.csv":
                continue  # past the first outer step the reference's own backends diverge
            close(data[:, col], base[:, col], other[:, col], f)


def test_compare_subcommand(tmp_path):
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    a.write_text(str(RG["deblur2d_ideal__config"]))
    b.write_text(str(RG["deblur2d_innercg__config"]))
    r = subprocess.run([RUNNER, "--out", str(tmp_path / "c"), "compare", str(a), str(b)], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0].split() == ["metric", "mlsqr", "mlsqr"] and len(lines) == 7
    assert sorted(os.listdir(tmp_path / "c")) == ["a", "b"]


def test_seed_override_changes_noise(tmp_path):
    cfg = tmp_path / "cfg.json"
    cfg.write_text(str(RG["deconv1d_lsqr__config"]))
    for seed in ("1", "2"):
        r = subprocess.run([RUNNER, "--quiet", "--seed", seed, "--out", str(tmp_path / seed), "run", str(cfg)],
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        assert json.load(open(tmp_path / seed / "meta.json"))["config"]["seed_used"] == int(seed)
    assert read_csv(tmp_path / "1" / "solution.csv")[1][:, 1].tolist() != \
        read_csv(tmp_path / "2" / "solution.csv")[1][:, 1].tolist()


def test_vcycle_extension_runs(tmp_path):
    doc = json.loads(str(RG["deblur2d_ideal__config"]))
    doc["solver"]["spd"] = {"mode": "vcycle", "levels": 4, "nu_pre": 2, "nu_post": 2}
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps(doc))
    r = subprocess.run([RUNNER, "--quiet", "--out", str(tmp_path / "o"), "run", str(cfg)], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    meta = json.load(open(tmp_path / "o" / "meta.json"))
    assert meta["result"]["stop_reason"] == "S4"
    assert meta["result"]["final_residual_weighted"] <= 1.1 * 0.01 * 1.0001
