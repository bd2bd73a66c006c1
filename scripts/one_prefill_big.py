"""One long-prompt prefill of the 7B target (for ncu launch lists): [n_tokens]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
t.prefill([(7 * i) % 32000 for i in range(n)])
t.kv_len()
