"""CPU draft single-token time (calibration probe and a 16-token greedy
draft_dynamic at a 200-token context) for two library builds, alternating
processes: python scripts/draft_token_ab.py alt/lib_other.so [rounds] [threads]"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
th = int(sys.argv[3]) if len(sys.argv) > 3 else 12
CHILD = r'''
import sys, time
sys.path.insert(0, "%s")
import numpy as np
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Draft
d = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=%d, cpus=list(range(2, 2 + %d)))
t0 = time.time()
while time.time() - t0 < 1.0: d.time_token(4)
tt = min(d.time_token(12) for _ in range(3))
ctx = np.random.default_rng(1).integers(0, 32000, 200).tolist()
ts = []
for r in range(20):
    t = time.perf_counter(); d.draft_dynamic(ctx, 16, 4, seed=r, greedy=True); ts.append((time.perf_counter() - t) * 1e3)
print("RESULT time_token %%.4f draft16 %%.3f" %% (tt, float(np.median(ts))))
''' % (ROOT, th, th)
alt = sys.argv[1]
for r in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    for name, lib in (("new", None), ("alt", alt)):
        env = dict(os.environ)
        env.pop("DD_LIB_AB", None)
        if lib:
            env["DD_LIB_AB"] = str((ROOT / lib).resolve())
        p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
        print(name, line[0][7:] if line else "FAILED " + p.stderr[-300:], flush=True)
