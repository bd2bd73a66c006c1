"""A/B pass time of one build under several environment settings on the same box
(alternating processes):
python scripts/env_ab.py W ctx1,ctx2 rounds "A=1 B=2" "A=0" ...
Each setting is a space-separated list of VAR=VALUE ("-" = no overrides)."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
w, ctxs, rounds = sys.argv[1], sys.argv[2], int(sys.argv[3])
settings = sys.argv[4:]
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
    for st in settings:
        env = dict(os.environ)
        if st != "-":
            for kv in st.split():
                k, v = kv.split("=", 1)
                env[k] = v
        try:
            p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                               timeout=float(os.environ.get("AB_TIMEOUT", "150")))
        except subprocess.TimeoutExpired:
            print(f"[{st}] W={w} ctx={ctxs}: TIMEOUT", flush=True)
            continue
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
        print(f"[{st}] W={w} ctx={ctxs}:", line[0][7:] if line else ("FAILED " + p.stderr[-300:]),
              flush=True)
