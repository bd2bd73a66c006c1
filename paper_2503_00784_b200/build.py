"""Build libduodec_b200.so in-tree: nvcc for the sm_100a kernels, g++ for host C++.

The library is the product: a C-ABI shared object (include/duodec_b200.h).
Only -gencode arch=compute_100a,code=sm_100a is emitted (no PTX fallback for
other archs, no CPU fallback).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libduodec_b200.so"

CU_SOURCES = ["gemm.cu", "gemm_wide.cu", "model.cu", "attention.cu", "attention_f32.cu", "pass.cu", "accept.cu", "tp.cu",
              "target.cu"]
CPP_SOURCES = ["plant.cpp", "draft.cpp", "engine.cpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
]
# host C++ runs on the GPU box's Xeon: x86-64-v3 (AVX2/FMA) baseline
CXX_FLAGS = ["-O3", "-std=c++20", "-fPIC", "-march=x86-64-v3", "-mtune=generic",
             "-ffp-contract=off", "-pthread", "-Wall", "-Wno-unused-function"]


def _nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _run(cmd, log):
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.write(" ".join(cmd) + "\n" + r.stdout + r.stderr + "\n")
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def _stale(out: Path, deps) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(p.stat().st_mtime > t for p in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "duodec_b200.h"]
    objs = []
    with open(BUILD / "build.log", "w") as log:
        for src in CU_SOURCES:
            if not (CSRC / src).exists():
                continue
            obj = BUILD / (src + ".o")
            if force or _stale(obj, [CSRC / src, *headers]):
                _run([_nvcc(), *NVCC_FLAGS, "-c", str(CSRC / src), "-o", str(obj)], log)
            objs.append(obj)
        for src in CPP_SOURCES:
            if not (CSRC / src).exists():
                continue
            obj = BUILD / (src + ".o")
            if force or _stale(obj, [CSRC / src, *headers]):
                _run(["g++", *CXX_FLAGS, "-I", str(Path(_nvcc()).parent.parent / "include"),
                      "-c", str(CSRC / src), "-o", str(obj)], log)
            objs.append(obj)
        if force or _stale(LIB, objs):
            _run([_nvcc(), "-shared", "-o", str(LIB), *map(str, objs),
                  "-Xcompiler", "-pthread", "-lcuda" if False else "-lcudart_static"], log)
    if verbose:
        print((BUILD / "build.log").read_text())
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
