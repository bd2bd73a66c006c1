"""One prefill + a few scored passes of the 7B target (for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 1
tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
tgt.prefill(list(range(128)))
for _ in range(3):
    tgt.score(list(range(w)))
    tgt.logits(0, 1)
    tgt.truncate(128)
