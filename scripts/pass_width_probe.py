"""Pass time by width: persistent pass kernel (DD_PASS_MAXW raised) vs one
launch per GEMM (DD_PASS_KERNEL=0).  Usage: pass_width_probe.py SHAPE MODE
where MODE is 'kernel' or 'launch' (set the env before the library loads)."""
import json
import os
import sys
from pathlib import Path

shape, mode = sys.argv[1], sys.argv[2]
if mode == "kernel":
    os.environ["DD_PASS_MAXW"] = "128"
else:
    os.environ["DD_PASS_KERNEL"] = "0"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Target  # noqa: E402

t = Target(SHAPES[shape], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
t.prefill([(7 * i) % 32000 for i in range(128)])
out = {}
for w in (8, 16, 17, 24, 32, 43, 48, 64):
    out[w] = round(t.time_pass(w, 10), 4)
print(json.dumps({"shape": shape, "mode": mode, "pass_ms": out}))
