"""Skinny stream-K GEMM vs tokens-on-M GEMM by pass width (DD_WIDE_MIN)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Target  # noqa: E402

t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
t.prefill(list(range(128)))
print({w: round(t.time_pass(w, 10), 3) for w in (17, 24, 32, 40, 48)}, flush=True)
