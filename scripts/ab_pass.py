"""A/B pass time of two builds of the library on the same box (alternating
processes): python scripts/ab_pass.py alt/lib_r01.so [W] [ctx,...] [rounds]"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
alt = sys.argv[1]
w = sys.argv[2] if len(sys.argv) > 2 else "9"
ctxs = sys.argv[3] if len(sys.argv) > 3 else "128,2048"
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 2
CHILD = r'''
import sys
sys.path.insert(0, "%s")
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target
t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
out = []
for n in [int(x) for x in "%s".split(",")]:
    t.truncate(0)
    t.prefill([(7 * i) %% 32000 for i in range(n)])
    out.append(min(t.time_pass(%s, trials=10) for _ in range(3)))
print("RESULT", " ".join("%%.4f" %% x for x in out))
''' % (ROOT, ctxs, w)
for r in range(rounds):
    for name, lib in (("new", None), ("alt", alt)):
        env = dict(os.environ)
        env.pop("DD_LIB_AB", None)
        if lib:
            env["DD_LIB_AB"] = str(Path(lib).resolve())
        p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
        print(name, f"W={w} ctx={ctxs}:", line[0][7:] if line else ("FAILED " + p.stderr[-300:]), flush=True)
