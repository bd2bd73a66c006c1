"""Calibration repeatability: c over repeated calibrate() calls, as bench.py
sets it up (target-role core, draft core slice) for a given KV capacity."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Draft, Target, calibrate  # noqa: E402

max_seq = int(sys.argv[1]) if len(sys.argv) > 1 else 768
tcore, dcores = bench.core_slice(0, 1)
os.sched_setaffinity(0, {tcore})
tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=max_seq)
drf = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=len(dcores), cpus=dcores)
print(max_seq, [round(calibrate(tgt, drf, probe_len=8, trials=12)[0], 2) for _ in range(5)],
      "tok", round(drf.time_token(12), 4), "pass", round(tgt.time_pass(8, 10), 4), flush=True)
