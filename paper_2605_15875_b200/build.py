"""Builds the in-tree CUDA library libdabd_gpu.so for sm_100a with nvcc.

Every translation unit is compiled for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo (so ncu source pages map back) and host code with
-ffp-contract=off (scene moments round like the reference build). The
library is linked with the static CUDA runtime and hidden visibility except
for the `dabd_gpu_*` C ABI of include/dabd_gpu.h.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(HERE, "build", "obj")
LIB = os.path.join(HERE, "libdabd_gpu.so")

SOURCES = ["scene.cpp", "balance.cpp", "body3d.cpp", "geometry.cu", "solver.cu", "solver_scalar.cu", "pcg.cu", "admm.cu", "engine.cu",
           "audit.cu", "contact3d.cu", "broad3d.cu", "sim3d.cu", "capi.cpp"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _flags(src: str):
    common = ["-O3", "-std=c++20", "-lineinfo", "-I", INCLUDE, "-I", CSRC,
              "-Xcompiler", "-fPIC,-fvisibility=hidden,-ffp-contract=off",
              "--expt-relaxed-constexpr", "-diag-suppress", "20012"]
    if src.endswith(".cu"):
        return ARCH + common + ["-Xptxas", "-O3"]
    return common + ["-x", "cu"] + ARCH


def _deps_mtime() -> float:
    m = 0.0
    for d in (CSRC, INCLUDE):
        for f in os.listdir(d):
            if f.endswith((".hpp", ".cuh", ".h")):
                m = max(m, os.path.getmtime(os.path.join(d, f)))
    return m


def _compile(src: str, hdr_mtime: float, verbose: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), hdr_mtime):
        return obj
    cmd = [nvcc(), "-c", path, "-o", obj] + _flags(src)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr.strip():
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    hdr = _deps_mtime()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr, verbose), SOURCES))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [nvcc(), "-shared", "-o", LIB] + objs + ARCH + ["-cudart", "static",
                                                             "-Xcompiler", "-fvisibility=hidden"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


ADAPTER_SRC = os.path.join(ROOT, "tests", "cpp", "adapter_main.cpp")
ADAPTER_BIN = os.path.join(ROOT, "tests", "cpp", "adapter_main")


def build_adapter() -> str:
    """g++ build of the C++ adapter test driver (include/dabd_gpu.hpp over
    libdabd_gpu.so), rpath'd to the in-tree library."""
    lib = build()
    hdr = os.path.join(INCLUDE, "dabd_gpu.hpp")
    if (os.path.exists(ADAPTER_BIN) and os.path.getmtime(ADAPTER_BIN) >=
            max(os.path.getmtime(ADAPTER_SRC), os.path.getmtime(hdr), os.path.getmtime(lib))):
        return ADAPTER_BIN
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", INCLUDE, ADAPTER_SRC, "-L", HERE,
           "-ldabd_gpu", "-Wl,-rpath,$ORIGIN/../../paper_2605_15875_b200", "-o", ADAPTER_BIN]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"adapter build failed:\n{r.stdout}\n{r.stderr}")
    return ADAPTER_BIN


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
