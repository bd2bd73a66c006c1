"""Prefill time of a long prompt on the 7B shape (CUDA events around dd_prefill):
python scripts/prefill_2k.py [n_tokens ...]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target  # noqa: E402

ns = [int(x) for x in sys.argv[1:]] or [1920, 2048]
t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
shp = SHAPES["llama2_7b"]
flop_tok = 2 * t.pass_weight_bytes() / 2  # 2 flops per weight per token (GEMMs)
for n in ns:
    toks = [(7 * i) % 32000 for i in range(n)]
    best = 1e9
    for r in range(3):
        t.truncate(0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t.prefill(toks)
        t.kv_len()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    # causal attention flops: 4 * hd * heads * layers * n^2 / 2
    attn = 4 * shp["head_dim"] * shp["n_heads"] * shp["n_layers"] * n * n / 2
    print(f"prefill {n} tokens: {best:.2f} ms  GEMM {flop_tok * n / best / 1e9:.0f} TFLOP/s-equiv "
          f"(+attention {attn / 1e12:.2f} TFLOP)", flush=True)
