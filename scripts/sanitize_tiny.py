"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
tiny target, prefill + scored passes on the persistent pass kernel (W=1, 8),
the tokens-on-M path (W=40) and the acceptance kernel, plus a CPU draft."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, Target  # noqa: E402
from paper_2503_00784_b200 import _lib as L  # noqa: E402

os.environ.setdefault("DD_PASS_KERNEL", "1")
t = Target(SHAPES["tiny"], weight_seed=3, max_seq=256)
t.prefill(list(range(20)))
for w in (1, 8, 40):
    t.score(list(range(w)))
    t.logits(0, 1)
    t.verify(L.DD_MODE_DUO, tail_len=w - 1, firsts=[1], greedy=True, q_onehot=True)
    t.truncate(20)
t.close()
print("sanitize workload done")
