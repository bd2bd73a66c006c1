"""Wall time of a 2K-token prompt prefill (16 chunks of 128) + one scored token."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Target  # noqa: E402

t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
toks = [(7 * i) % 32000 for i in range(2048)]
res = []
for r in range(4):
    t.truncate(0)
    t0 = time.perf_counter()
    t.prefill(toks[:-1])
    t.score(toks[-1:])
    t.logits(0, 1)
    res.append((time.perf_counter() - t0) * 1e3)
print("2K prefill+score ms", [round(x, 1) for x in res], flush=True)
