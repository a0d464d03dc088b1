"""CPU-side checks of the drop-in boundary (no GPU needed):
the C-ABI library builds for sm_100a, loads, exports every symbol that
include/mlsqr_b200.h declares, refuses to run without a B200 (no CPU
fallback), and its host-side input generators are bit-identical to the
oracle's independent restatement."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1308_6634_b200 as mb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mlsqr_b200.h")


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(mb.LIB_PATH):
        from paper_1308_6634_b200 import build
        build.build(verbose=False)
    return mb.lib()


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?\w+\s*\**\s*(mlsqr_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_every_declared_symbol_is_exported(built):
    out = subprocess.run(["nm", "-D", "--defined-only", mb.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mlsqr_\w+)", out))
    declared = header_functions()
    assert len(declared) >= 35
    missing = [n for n in declared if n not in exported]
    assert not missing, missing
    # and the Python mirror binds exactly the declared surface
    assert set(mb.SIGNATURES) == set(declared)


def test_library_is_sm100a_only(built):
    out = subprocess.run(["cuobjdump", "--list-elf", mb.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if line.strip())


def test_no_cpu_fallback_without_gpu(built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mb.CudaError):
        mb.Context(0)


def test_version_string(built):
    assert b"sm_100a" in mb.lib().mlsqr_version()


def test_host_generators_match_oracle(built, orc):
    assert np.array_equal(mb.gaussian_taps(128, 2 / 128, 6), orc.taps(128, 2 / 128, radius=6))
    assert np.array_equal(mb.gaussian_taps(1024, 3 / 1024), orc.taps(1024, 3 / 1024))
    assert np.array_equal(mb.gaussian_noise(11, 4097, 0.2), orc.gauss(11, 4097, 0.2))
    assert np.array_equal(mb.phantom_rects2d(64, 48, 8, 3), orc.rects2d(64, 48, 8, 3))
    assert np.array_equal(mb.phantom_shapes2d(64, 64, 32, 4), orc.shapes2d(64, 64, 32, 4))
    assert np.array_equal(mb.phantom_ellipsoids3d(32, 24, 16, 10, 2, 10, 0.2, 1.0, 5),
                          orc.ellipsoids3d(32, 24, 16, 10, 2, 10, 0.2, 1.0, 5))
    gs, gd = mb.fdot_tables(6, 3, 4, 1.0, 9)
    ogs, ogd, _ = orc.fdot(6, 3, 4, 1.0, 9)
    assert np.array_equal(gs, ogs) and np.array_equal(gd, ogd)


def test_python_mirror_validation_matches_reference_contract():
    # StoppingConfig::validate (krylov.cpp:219-226) and PenaltySpec::validate (penalty.cpp:27-32)
    with pytest.raises(ValueError):
        mb.StoppingConfig.max_iterations(0)
    with pytest.raises(ValueError):
        mb.StoppingConfig(use_s4=True, eta=1.0).validate()
    with pytest.raises(ValueError):
        mb.StoppingConfig(use_s4=True, delta=-1.0).validate()
    with pytest.raises(ValueError):
        mb.PenaltySpec.tv_smoothed(0.0).validate()
    assert issubclass(mb.DimensionError, ValueError)
    assert mb.BreakdownError("x", 3).iteration == 3


@pytest.mark.timeout(60)
def test_nccl_unique_id_without_gpu():
    """ncclGetUniqueId only opens the bootstrap socket: it works here and must not hang
    (regression: the dlopen'ed symbol table was once resolved re-entrantly under call_once)."""
    uid = mb.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128
