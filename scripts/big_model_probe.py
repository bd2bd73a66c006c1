"""Llama-2-70B-shape target on ONE B200 (TP=1: 138 GB of bf16 weights fit in
180 GB HBM): pass times by width and a short greedy generation per mode.
Config 5 runs this shape at TP=8; this is its single-GPU reference point."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2503_00784_b200 import (DEFAULT_PLANT, SHAPES, Draft, EngineConfig,  # noqa: E402
                                   Target, run_generation)

t0 = time.time()
tgt = Target(SHAPES["llama2_70b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
print("init s", round(time.time() - t0, 1), flush=True)
wb = tgt.pass_weight_bytes() if hasattr(tgt, "pass_weight_bytes") else None
res = {"weight_bytes": wb}
for w in (1, 8, 16):
    ms = tgt.time_pass(w, 10)
    res[f"pass_ms_w{w}"] = round(ms, 3)
    if wb:
        res[f"GBs_w{w}"] = round(wb / ms / 1e6, 1)
    print(w, ms, flush=True)
drf = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=12,
            cpus=list(range(2, 14)))
prompt = np.random.default_rng(1).integers(0, 32000, 128).tolist()
for mode, budget in (("vanilla", 2), ("duo", 24), ("sps", 8)):
    cfg = EngineConfig(mode=mode, budget=budget, max_sequences=4, max_new_tokens=64, greedy=True,
                       budget_hard_cap=32)
    r = run_generation(tgt, drf if mode != "vanilla" else None, prompt, cfg)
    dec = (len(r.tokens) - 1) / ((r.total_ms - r.ttft_ms) / 1000.0)
    res[mode] = dict(tps=round(r.tps, 1), decode_tps=round(dec, 1), ttft_ms=round(r.ttft_ms, 2),
                     iters=len(r.iterations), tokens=len(r.tokens))
    print(mode, res[mode], flush=True)
print(json.dumps(res))
