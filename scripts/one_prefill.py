"""One 128-token scored pass of the 7B target (the TTFT pass), for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Target  # noqa: E402

t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
for _ in range(2):
    t.truncate(0)
    t.score([(7 * i) % 32000 for i in range(128)])
    t.logits(0, 1)
