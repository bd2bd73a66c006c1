"""Soak test of the persistent pass kernel's synchronisation (-m gpu): many
scored passes of random widths (1..32, both register-chunk instantiations) and
contexts, each re-run after a KV rollback; every re-run must give bit-identical
logits.  The dataflow protocol (tile flags through the publisher warp, tile
groups / k-groups, stream-K partial counters, attention group merges, 4 TMEM
accumulators, 9-stage ring) has a fixed reduction order, so any race or
missed acquire shows up as a run-to-run difference.  Shapes: the tiny
head_dim-64 target, the head_dim-128 GQA shape and the 7B shape (whose gate/up
and down run as tile groups / k-groups)."""
import numpy as np
import pytest

from paper_2503_00784_b200 import SHAPES, Target

pytestmark = pytest.mark.gpu

PLANT = dict(plant_seed=7, alpha=0.5, gain=1.0, emb_std=1.0)


@pytest.mark.parametrize("shape_name,iters", [("tiny", 200), ("gqa128", 200), ("llama2_7b", 80)])
def test_rerun_bit_identical(shape_name, iters):
    shape = SHAPES[shape_name]
    t = Target(shape, weight_seed=77, plant=PLANT, max_seq=1024)
    rng = np.random.default_rng(2024)
    ctx = rng.integers(0, shape["vocab"], 600).tolist()
    n = 0
    t.prefill(ctx[:40])
    n = 40
    for it in range(iters):
        w = int(rng.integers(1, 33))
        toks = rng.integers(0, shape["vocab"], w).tolist()
        t.score(toks)
        a = t.logits(0, w)
        t.truncate(n)
        t.score(toks)
        b = t.logits(0, w)
        assert np.array_equal(a, b), f"iteration {it}: W={w} after {n} keys differs on re-run"
        # keep a random prefix of the pass (rollback), grow the context
        keep = int(rng.integers(0, w + 1))
        t.truncate(n + keep)
        n += keep
        if n > 900:
            t.truncate(40)
            n = 40
    t.close()
