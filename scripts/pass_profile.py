"""Per-width pass timing + class breakdown (gemm / attention / norms) of the 7B
target, plus CPU draft prefill and per-token timings (device CUDA events / wall)."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target, Draft  # noqa: E402

widths = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,8,16,32,64,127,256").split(",")]
ctx_len = int(sys.argv[2]) if len(sys.argv) > 2 else 128
tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
tgt.prefill(list(range(ctx_len)))
wb = tgt.pass_weight_bytes()
res = {}
for w in widths:
    ms = tgt.time_pass(w, trials=8)
    prof = tgt.profile_pass(w)
    res[w] = dict(ms=round(ms, 4), frac=round(wb / ms / 1e6 / 6554.9, 3),
                  **{k: round(v, 4) for k, v in prof.items()})
    print(w, res[w], flush=True)
tgt.close()
cpus = sorted(os.sched_getaffinity(0))[1:13]
drf = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=len(cpus), cpus=cpus)
for n in (128, 2048):
    ctx = [(7 * i) % 32000 for i in range(n)]
    t = []
    for _ in range(3):
        drf.logits([1])
        t0 = time.perf_counter(); drf.logits(ctx); t.append(time.perf_counter() - t0)
    print("draft prefill", n, "ms", round(min(t) * 1e3, 2), flush=True)
print("draft token ms", round(drf.time_token(12), 4))
