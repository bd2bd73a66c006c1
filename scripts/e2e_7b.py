"""End-to-end 7B-shape target on one B200 + 68M-shape draft on host cores."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import (SHAPES, DEFAULT_PLANT, Draft, EngineConfig, Target,  # noqa
                                   calibrate, run_generation)

alpha = float(sys.argv[1]) if len(sys.argv) > 1 else DEFAULT_PLANT["alpha"]
plant = dict(DEFAULT_PLANT, alpha=alpha)
t0 = time.time()
tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=plant, max_seq=4096)
drf = Draft(SHAPES["llama_68m"], weight_seed=99, plant=plant, threads=12, cpus=list(range(2, 14)))
print("init", round(time.time() - t0, 1), "s; draft ms/token", round(drf.time_token(12), 3), flush=True)
print("pass ms W=1,8:", round(tgt.time_pass(1), 3), round(tgt.time_pass(8), 3))
c, b = calibrate(tgt, drf)
print("calibrate c=%.2f budget=%d" % (c, b), flush=True)
prompt = np.random.default_rng(1).integers(0, 32000, 128).tolist()
for mode, bud in [("vanilla", 2), ("sps", max(2, b // 2)), ("duo", b), ("duo", 2 * b)]:
    cfg = EngineConfig(mode=mode, budget=bud, max_sequences=4, max_new_tokens=128, greedy=True)
    for rep in range(2):
        r = run_generation(tgt, drf if mode != "vanilla" else None, prompt, cfg)
    acc = [it.tokens_processed for it in r.iterations]
    dms = np.mean([it.draft_ms for it in r.iterations])
    tms = np.mean([it.target_ms for it in r.iterations])
    cms = np.mean([it.comm_ms for it in r.iterations])
    print(f"{mode:8s} gamma={bud:3d} tps={r.tps:8.1f} ttft={r.ttft_ms:7.2f}ms iters={len(r.iterations)} "
          f"tok/iter={np.mean(acc):.2f} draft={dms:.2f} target={tms:.2f} comm={cms:.2f} first16={r.tokens[:16]}",
          flush=True)
