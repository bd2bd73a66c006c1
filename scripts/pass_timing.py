"""Time scored passes of the 7B-shape target on one B200 (device CUDA events)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target  # noqa: E402

shape = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "llama2_7b"]
t0 = time.time()
tgt = Target(shape, weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
print("init_s", round(time.time() - t0, 2), flush=True)
tgt.prefill(list(range(128)))
wb = tgt.pass_weight_bytes()
res = {}
for w in (1, 2, 4, 8, 16, 25, 32, 64):
    ms = tgt.time_pass(w, trials=12)
    prof = tgt.profile_pass(w)
    res[w] = dict(ms=round(ms, 4), gbs=round(wb / ms / 1e6, 1), **{k: round(v, 4) for k, v in prof.items()})
    print(w, res[w], flush=True)
print(json.dumps(res))
