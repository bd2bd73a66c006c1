"""First-iteration breakdown of duo vs SpS vs vanilla (TTFT anatomy)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_00784_b200 import (DEFAULT_PLANT, SHAPES, Draft, EngineConfig, Target,  # noqa: E402
                                   calibrate, run_generation)

tcore, dcores = bench.core_slice(0, 1)
os.sched_setaffinity(0, {tcore})
tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
drf = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=len(dcores), cpus=dcores)
coef, budget = calibrate(tgt, drf, probe_len=8, trials=12)
print("budget", budget, "draft token ms", drf.time_token(12))
for mode, bud in (("duo", budget), ("sps", max(2, budget // 2)), ("vanilla", 2)):
    cfg = EngineConfig(mode=mode, budget=bud, max_new_tokens=16, greedy=True)
    for rep in range(3):
        r = run_generation(tgt, drf if mode != "vanilla" else None, bench.make_prompt(rep + 1), cfg)
        it = r.iterations[0]
        print(f"{mode:7s} ttft dev {r.device_ttft_ms:6.2f} wall {r.ttft_ms:6.2f} | it0 draft {it.draft_ms:6.2f} "
              f"target {it.target_ms:6.2f} verify {it.verify_ms:5.2f} comm {it.comm_ms:5.2f}")
