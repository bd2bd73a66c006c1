"""Parity diagnostic: logit error vs the oracle across shapes / paths / modes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.llama import OracleLlama
from paper_2503_00784_b200 import SHAPES, Target

PLANT = dict(plant_seed=7, alpha=0.5, gain=1.0, emb_std=1.0)
V = dict(vocab=32000, rms_eps=1e-5, rope_theta=1e4)
shapes = {
    "tiny": SHAPES["tiny"],
    "mid128": SHAPES["mid128"],
    "mid128_L1": dict(SHAPES["mid128"], n_layers=1),
    "mid64": dict(n_layers=2, d_model=1024, n_heads=16, n_kv_heads=16, head_dim=64, ffn_dim=2816, **V),
    "d512_hd128": dict(n_layers=4, d_model=512, n_heads=4, n_kv_heads=4, head_dim=128, ffn_dim=1408, **V),
    "gqa128": SHAPES["gqa128"],
}
for name, sh in shapes.items():
    tgt = Target(sh, weight_seed=17, plant=PLANT, max_seq=512)
    orc = OracleLlama(sh, weight_seed=17, plant=PLANT, max_seq=512)
    rng = np.random.default_rng(1)
    ctx = rng.integers(0, 32000, 33).tolist()
    for w in (1, 8, 17, 200):
        new = rng.integers(0, 32000, w).tolist()
        res = []
        for pb in (0, 1):
            orc.set_p_bf16(pb)
            tgt.truncate(0); orc.truncate(0)
            tgt.prefill(ctx); orc.forward(ctx, last_only=True)
            tgt.score(new)
            g = tgt.logits(0, w); o = orc.forward(new)
            res.append(np.abs(g - o).max() / np.abs(o).max())
        print(f"{name:12s} W={w:3d} rel={res[0]:.2e} rel(p_bf16 oracle)={res[1]:.2e} "
              f"maxlogit={np.abs(o).max():.2f}", flush=True)
    tgt.close(); orc.close()
