"""Draft-side time per duo iteration for two library builds on the same box
(alternating processes): greedy duo at budget 16 on the 7B target, mean
IterationRecord.draft_ms / comm_ms / target_ms and tokens/s.
python scripts/draft_ab.py alt/lib_other.so [rounds]"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r'''
import sys
sys.path.insert(0, "%s")
import numpy as np
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Draft, EngineConfig, Target, run_generation
tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
drf = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=12, cpus=list(range(2, 14)))
prompt = np.random.default_rng(1).integers(0, 32000, 128).tolist()
cfg = EngineConfig(mode="duo", budget=16, max_sequences=4, max_new_tokens=128, greedy=True)
rs = [run_generation(tgt, drf, prompt, cfg) for _ in range(4)][1:]
its = [it for r in rs for it in r.iterations[1:]]
print("RESULT draft_ms %%.3f comm_ms %%.3f target_ms %%.3f tps %%.1f" %% (
    np.mean([i.draft_ms for i in its]), np.mean([i.comm_ms for i in its]),
    np.mean([i.target_ms for i in its]), np.mean([r.tps for r in rs])))
''' % ROOT
alt = sys.argv[1]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for r in range(rounds):
    for name, lib in (("new", None), ("alt", alt)):
        env = dict(os.environ)
        env.pop("DD_LIB_AB", None)
        if lib:
            env["DD_LIB_AB"] = str((ROOT / lib).resolve())
        p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
        print(name, line[0][7:] if line else "FAILED " + p.stderr[-300:], flush=True)
