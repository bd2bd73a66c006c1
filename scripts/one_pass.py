"""One prefill + a few scored passes of the 7B target (for ncu launch lists).
usage: one_pass.py [W] [context]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=max(1024, n + 512))
tgt.prefill([(7 * i) % 32000 for i in range(n)])
for _ in range(3):
    tgt.score(list(range(w)))
    tgt.logits(0, 1)
    tgt.truncate(n)
