"""Per-launch GEMM time by CTA count (DD_PASS_KERNEL=0 path)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target
import os
t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
t.prefill(list(range(128)))
ms, n = t.time_gemms(8, trials=5)
wb = t.pass_weight_bytes()
print(os.environ.get("DD_GEMM_CTAS", "default"), os.environ.get("DD_GEMM_STAGES", "default"), f"gemm seq {ms:.3f} ms {wb/ms/1e6:.0f} GB/s")
