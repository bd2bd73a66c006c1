"""The drop-in C ABI (include/duodec_b200.h): the shared library loads, exports
every declared entry point, and fails loudly (no CPU fallback) without a GPU."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "duodec_b200.h"


def declared():
    src = HEADER.read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dd_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(native):
    names = declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(native, n), f"missing export {n}"


def test_binding_covers_header():
    from paper_2503_00784_b200 import _lib
    assert set(declared()) == set(_lib.SIGNATURES)


def test_struct_layouts_match_header(native):
    from paper_2503_00784_b200 import _lib
    # sizes must agree with the C compiler's view of the header
    import subprocess, tempfile, os
    code = '#include "duodec_b200.h"\n#include <stdio.h>\nint main(){printf("%zu %zu %zu %zu %zu %zu %zu\\n",' \
           'sizeof(dd_model_desc),sizeof(dd_plant_desc),sizeof(dd_verify_args),sizeof(dd_verify_out),' \
           'sizeof(dd_engine_config),sizeof(dd_iteration_record),sizeof(dd_generation_result));}'
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "t.c"), "w").write(code)
        subprocess.run(["gcc", "-I", str(ROOT / "include"), os.path.join(d, "t.c"), "-o",
                        os.path.join(d, "t")], check=True)
        sizes = [int(x) for x in subprocess.check_output([os.path.join(d, "t")]).split()]
    ours = [C.sizeof(t) for t in (_lib.ModelDesc, _lib.PlantDesc, _lib.VerifyArgs, _lib.VerifyOut,
                                  _lib.EngineConfigC, _lib.IterationRecordC, _lib.GenerationResultC)]
    assert sizes == ours


def test_no_gpu_fails_loudly(native):
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("GPU present")
    from paper_2503_00784_b200 import SHAPES, DeviceError, Target
    with pytest.raises(DeviceError, match="no CUDA device"):
        Target(SHAPES["tiny"], max_seq=64)


def test_bad_shape_rejected(native):
    from paper_2503_00784_b200 import ConfigError, Target
    bad = dict(n_layers=1, d_model=100, n_heads=2, n_kv_heads=2, head_dim=50, ffn_dim=128,
               vocab=1000)
    with pytest.raises(ConfigError):
        Target(bad, max_seq=16)
