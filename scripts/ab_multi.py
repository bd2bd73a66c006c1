"""Pass time of several library builds / env settings on one box, interleaved:
python scripts/ab_multi.py W ctx1,ctx2 rounds "name=lib_or_-[:VAR=VAL ...]" ...
(lib "-" = the in-tree build)."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
w, ctxs, rounds = sys.argv[1], sys.argv[2], int(sys.argv[3])
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
    for spec in sys.argv[4:]:
        name, rest = spec.split("=", 1)
        parts = rest.split(":")
        env = dict(os.environ)
        env.pop("DD_LIB_AB", None)
        if parts[0] != "-":
            env["DD_LIB_AB"] = str((ROOT / parts[0]).resolve())
        for kv in parts[1:]:
            k, v = kv.split("=", 1)
            env[k] = v
        try:
            p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=150)
            line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
            print(f"{name:12s} W={w} ctx={ctxs}:", line[0][7:] if line else "FAILED " + p.stderr[-200:], flush=True)
        except subprocess.TimeoutExpired:
            print(f"{name:12s} TIMEOUT", flush=True)
