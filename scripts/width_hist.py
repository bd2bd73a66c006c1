"""Pass-width histogram of config-2 duo generations (bench's models and prompts):
python scripts/width_hist.py [budget]"""
import collections
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Draft, EngineConfig, Target, run_generation  # noqa: E402

budget = int(sys.argv[1]) if len(sys.argv) > 1 else 16
tgt = Target(SHAPES["llama2_7b"], weight_seed=bench.SEED_W_TARGET, plant=DEFAULT_PLANT, max_seq=1024)
drf = Draft(SHAPES["llama_68m"], weight_seed=bench.SEED_W_DRAFT, plant=DEFAULT_PLANT, threads=12)
cfg = EngineConfig(mode="duo", budget=budget, max_sequences=4, max_new_tokens=128, greedy=True,
                   budget_hard_cap=256)
h = collections.Counter()
tok = iters = 0
for s in range(1, 6):
    r = run_generation(tgt, drf, bench.make_prompt(s), cfg)
    for it in r.iterations[1:]:
        h[it.width] += 1
    tok += len(r.tokens)
    iters += len(r.iterations)
print(f"budget {budget}: tokens/iteration {tok / iters:.3f}; widths", dict(sorted(h.items())))
