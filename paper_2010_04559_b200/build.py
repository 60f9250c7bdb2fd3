"""Build libstamg_b200.so in-tree: hand-written sm_100a CUDA + host C++.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 for every .cu,
host setup compiled by the same driver, linked with the static CUDA runtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libstamg_b200.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CCBIN = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-ccbin", CCBIN, "-I" + os.path.join(HERE, "..", "include")] + os.environ.get("STAMG_NVCC_EXTRA", "").split()
SOURCES = ["setup.cpp", "generic_setup.cpp", "generic.cu", "sweep.cu", "transport.cu", "scatter.cu", "multigrid.cu", "blas.cu", "couplings.cu", "context.cu"]


def _obj(src):
    return os.path.join(BUILD, os.path.splitext(src)[0] + ".o")


def _needs(src, obj):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".hpp", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "stamg_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose):
    obj = _obj(src)
    cmd = [NVCC] + ARCH + FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
    if src.endswith(".cu") and verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return src, r.stderr


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    todo = [s for s in SOURCES if force or _needs(s, _obj(s))]
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(todo)))) as ex:
        for src, err in ex.map(lambda s: _compile(s, verbose), todo):
            if verbose and err:
                print(f"--- {src}\n{err}", file=sys.stderr)
    if todo or not os.path.exists(OUT):
        cmd = [NVCC] + ARCH + ["-shared", "-ccbin", CCBIN, "-o", OUT] + [_obj(s) for s in SOURCES] + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
