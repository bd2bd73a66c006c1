"""Pass time (ms, min of 3 x 10 trials) of the 7B target by width and context:
python scripts/width_sweep.py 1,8,16,17,32 128,2048"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target  # noqa: E402

ws = [int(x) for x in sys.argv[1].split(",")]
ctxs = [int(x) for x in sys.argv[2].split(",")]
t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
for n in ctxs:
    t.truncate(0)
    t.prefill([(7 * i) % 32000 for i in range(n)])
    print(f"ctx {n}: " + "  ".join(f"W={w}: {min(t.time_pass(w, trials=10) for _ in range(3)):.4f}" for w in ws),
          flush=True)
