"""compute-sanitizer workload for the tensor-parallel path: a TP=2 group of the
tiny target on one GPU (in-process connect), prefill + scored passes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, Target  # noqa: E402

shape = dict(SHAPES["tiny"], n_kv_heads=4)
ranks = [Target(shape, weight_seed=3, max_seq=256, tp_rank=r, tp_size=2) for r in range(2)]
Target.tp_connect_local(ranks)
for t in ranks:
    t.prefill(list(range(20)))
for w in (1, 8, 40):
    for t in ranks:
        t.score(list(range(w)))
    for t in ranks:
        t.logits(0, 1)
        t.truncate(20)
for t in ranks:
    t.close()
print("sanitize tp workload done")
