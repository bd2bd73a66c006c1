"""Persistent pass kernel above 16 tokens (DD_PASS_MAXW) vs the per-launch path: logits agreement by width."""
import os, sys
os.environ["DD_PASS_MAXW"] = "128"
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2503_00784_b200 import SHAPES, Target
TINY = SHAPES["tiny"]; PLANT = dict(plant_seed=7, alpha=0.5, gain=1.0, emb_std=1.0)
a = Target(TINY, weight_seed=11, plant=PLANT, max_seq=512)
os.environ["DD_PASS_KERNEL"] = "0"
b = Target(TINY, weight_seed=11, plant=PLANT, max_seq=512)
rng = np.random.default_rng(3)
for w in (17, 24, 40, 64, 100):
    ctx = rng.integers(0, 32000, 50).tolist(); new = rng.integers(0, 32000, w).tolist()
    out = []
    for t in (a, b):
        t.truncate(0); t.prefill(ctx); t.score(new); out.append(t.logits(0, w))
    rel = np.abs(out[0] - out[1]).max() / np.abs(out[1]).max()
    print(w, rel, (out[0].argmax(-1) == out[1].argmax(-1)).mean(), flush=True)
