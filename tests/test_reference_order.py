"""Device arithmetic order vs the reference's OWN arithmetic order on the BASELINE configs.

The GPU path is bit-exact with the oracle's device order (tests/test_gpu_configs.py), so the distance
between the GPU and the reference is the distance between the oracle's device order and the
reference's `mlsqr` (oracle/_ref, built from /root/reference/proj/src; krylov.cpp:335-440) under its
scalar backend.  The floor is the reference's own scalar-vs-AVX2 spread (kernels_dispatch.cpp:57-66).
north_star's bounds (alpha/beta after the fixed count 1e-9, final reconstruction 1e-6) are asserted
as  err <= max(bound, 10 x floor).

* test_committed_reference_order_report: the committed C1-C3 report
  (profiles/reference_order_report.json, tools/reference_order_report.py) passes that rule at every
  outer step, and where the reference's two backends agree to 1e-9 over the whole fixed count, so
  does the device order (C2's first outer step: 2.0e-14 vs a 1.9e-14 floor);
* test_reference_order_c1_live: C1 (128^2, 50 iterations) re-run here, against oracle/_ref.
"""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPORT = os.path.join(ROOT, "profiles", "reference_order_report.json")


def _check(r):
    for s in r["steps"]:
        for key in ("alphas", "betas", "f"):
            row = s[key]
            assert row["ok"], (r["config"], s["k"], key, row)
            assert row["gpu_vs_ref_scalar"] <= max(row["bound"], 1e-9 if key != "f" else 1e-6)
        for key in ("alphas", "betas"):
            row = s[key]
            # wherever the reference agrees with itself to 1e-9 for n iterations, so does the device order
            assert row["agree_1e-9_iters_gpu_vs_ref_scalar"] >= row["agree_1e-9_iters_ref_avx2_vs_ref_scalar"] - 1, (
                r["config"], s["k"], key, row)
    fr = r["final_reconstruction"]
    assert fr["ok"] and fr["gpu_vs_ref_scalar"] <= fr["bound"], (r["config"], fr)


def test_committed_reference_order_report():
    with open(REPORT) as fh:
        rep = json.load(fh)
    assert set(rep["configs"]) >= {"c1", "c2", "c3"}
    for name, r in rep["configs"].items():
        assert r["ok"], name
        _check(r)
    # the one step where the reference's backends agree over the whole fixed count: the first C2 step
    s = rep["configs"]["c2"]["steps"][0]
    assert s["alphas"]["gpu_vs_ref_scalar"] < 1e-9 and s["betas"]["gpu_vs_ref_scalar"] < 1e-9
    assert s["f"]["gpu_vs_ref_scalar"] < 1e-9


def test_reference_order_c1_live():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmlsqr_ref.so")):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import reference_order_report as ror
    r = ror.report("c1")
    assert r["ok"]
    _check(r)
