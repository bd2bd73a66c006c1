"""128-token scored pass (the first-iteration / TTFT pass) and 127-token prefill times."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Target  # noqa: E402

t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
t.prefill([1, 2])
print("W=128 pass ms", round(t.time_pass(128, 10), 3), " W=64", round(t.time_pass(64, 10), 3), flush=True)
