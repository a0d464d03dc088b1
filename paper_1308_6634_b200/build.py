"""In-tree build of libmlsqr_b200.so (sm_100a only, no JIT, no fallback).

    python -m paper_1308_6634_b200.build          # or __graft_entry__.build()

Every .cu is compiled with
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
-fmad=false keeps every mul+add pair separately rounded (the canonical
arithmetic order); the host generator is compiled without FMA too.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libmlsqr_b200.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr", "-Xptxas", "-v"]
CXXFLAGS = ["-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-Wall"]


def _sources():
    cu = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    cpp = sorted(f for f in os.listdir(CSRC) if f.endswith(".cpp"))
    return cu, cpp


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, src + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "mlsqr_b200.h"))
    if not _newer(obj, deps):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(BUILD, src + ".log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"  built {src}")
    return obj


def build(verbose: bool = True) -> str:
    os.makedirs(BUILD, exist_ok=True)
    cu, cpp = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), cu + cpp))
    lib_changed = _newer(LIB, objs)
    if lib_changed:
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt", "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"  linked {LIB}")
    build_runner(verbose)
    return LIB


# the reference's `mlsqr run | compare` harness on the device path (runner/mlsqr_b200_run.cpp);
# JSON via nlohmann/json 3.11.3 -- the library the reference's config.cpp uses, header-only
RUNNER_SRC = os.path.join(HERE, "runner", "mlsqr_b200_run.cpp")
RUNNER = os.path.join(HERE, "mlsqr-b200")
JSON_DIRS = [os.environ.get("MLSQR_JSON_INCLUDE", ""),
             "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann",
             "/usr/include/nlohmann"]


def build_runner(verbose: bool = True) -> str:
    inc = next((d for d in JSON_DIRS if d and os.path.exists(os.path.join(d, "json.hpp"))), None)
    if inc is None:
        raise RuntimeError("nlohmann/json.hpp not found (set MLSQR_JSON_INCLUDE)")
    deps = [RUNNER_SRC, LIB, os.path.join(HERE, "..", "include", "mlsqr_b200.h")]
    if not _newer(RUNNER, deps):
        return RUNNER
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-ffp-contract=off", "-I", inc, RUNNER_SRC, "-o", RUNNER,
           "-L", HERE, "-lmlsqr_b200", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"runner build failed\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"  built {RUNNER}")
    return RUNNER


if __name__ == "__main__":
    build(verbose="-q" not in sys.argv)
