"""INTEGRATION.md's C++ adapter (integration/gpu_target.hpp) compiles against the
reference's own headers (/root/reference/proj/include) and links against the
product library and the compiled reference.  Without a GPU the adapter must
surface the missing device as the reference's ConfigError (no CPU fallback).
Needs the reference sources, so it runs in the build container only."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_INC = Path("/root/reference/proj/include")
LIB = ROOT / "paper_2503_00784_b200" / "libduodec_b200.so"
REF_LIB = ROOT / "oracle" / "_ref" / "libduodec_ref.so"


@pytest.mark.skipif(not REF_INC.exists() or shutil.which("g++") is None, reason="reference headers absent")
def test_adapter_compiles_against_reference(tmp_path):
    if not LIB.exists() or not REF_LIB.exists():
        pytest.skip("build() not run")
    exe = tmp_path / "adapter_check"
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Werror", f"-I{ROOT / 'integration'}", f"-I{ROOT / 'include'}",
           f"-I{REF_INC}", str(ROOT / "integration" / "adapter_check.cpp"), "-o", str(exe),
           f"-L{LIB.parent}", "-lduodec_b200", f"-L{REF_LIB.parent}", "-lduodec_ref",
           f"-Wl,-rpath,{LIB.parent}:{REF_LIB.parent}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True, timeout=120).stdout
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        assert out.startswith("GPU ok"), out
    else:
        assert out.startswith("ConfigError: no CUDA device"), out
