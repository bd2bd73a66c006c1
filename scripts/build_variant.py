"""Build an A/B variant of the library with one source file replaced:
python scripts/build_variant.py NAME target.cu path/to/replacement.cu [extra nvcc -D flags...]
-> alt/lib_NAME.so (the other objects come from the in-tree build)."""
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2503_00784_b200 import build as B  # noqa: E402

name, target, repl = sys.argv[1], sys.argv[2], Path(sys.argv[3]).resolve()
defs = sys.argv[4:]
B.build()
tmp = Path("/tmp/ddvar_" + name)
shutil.rmtree(tmp, ignore_errors=True)
shutil.copytree(B.CSRC, tmp / "pkg" / "csrc")
shutil.copytree(ROOT / "include", tmp / "include")
dst = tmp / "pkg" / "csrc" / target
shutil.copy(repl, dst)
obj = tmp / (target + ".o")
subprocess.run([B._nvcc(), *B.NVCC_FLAGS, *defs, "-c", str(dst), "-o", str(obj)], check=True,
               capture_output=True)
objs = []
for src in B.CU_SOURCES + B.CPP_SOURCES:
    objs.append(obj if src == target else B.BUILD / (src + ".o"))
out = ROOT / "alt" / f"lib_{name}.so"
out.parent.mkdir(exist_ok=True)
subprocess.run([B._nvcc(), "-shared", "-o", str(out), *map(str, objs), "-Xcompiler", "-pthread",
                "-lcudart_static"], check=True)
print(out)
