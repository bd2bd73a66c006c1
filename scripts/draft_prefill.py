"""CPU draft prefill time (128 and 2048-token prompts), AMX vs VNNI (DD_DRAFT_AMX=0)."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Draft  # noqa: E402

n_thr = int(sys.argv[1]) if len(sys.argv) > 1 else 12
cpus = sorted(os.sched_getaffinity(0))
d = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=n_thr,
          cpus=cpus[1:1 + n_thr] if len(cpus) > n_thr else cpus)
rng = np.random.default_rng(0)
for n in (128, 2048):
    ts = []
    for r in range(4):
        p = rng.integers(0, 32000, n).tolist()
        t0 = time.perf_counter()
        d.logits(p)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"AMX={os.environ.get('DD_DRAFT_AMX', '1')} prefill {n}: {np.median(ts[1:]):.2f} ms", flush=True)
