"""A/B the persistent pass kernel against per-kernel launches (device time)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target  # noqa: E402

widths = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,8,16,32").split(",")]
ctx_len = int(sys.argv[2]) if len(sys.argv) > 2 else 128
tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
tgt.prefill([(7 * i) % 32000 for i in range(ctx_len)])
wb = tgt.pass_weight_bytes()
mode = os.environ.get("DD_PASS_KERNEL", "1")
for w in widths:
    ms = tgt.time_pass(w, trials=10)
    print(f"mode={mode} n={ctx_len} W={w}: {ms:.4f} ms  {wb / ms / 1e6:.0f} GB/s  frac {wb / ms / 1e6 / 6554.9:.3f}", flush=True)
