"""Tensor-parallel machinery at 7B scale on ONE GPU: a TP=2 group (both ranks
on this device, connected in-process) against the unsharded target on the
same per-launch GEMM path.  The two ranks share one GPU's bandwidth, so the
pair streams the same weight bytes as TP=1; the difference is the cost of the
64 rank-ordered reductions + logits gather per pass (local memory here, NVLink
peers on a multi-GPU box).  Wall time per scored pass (8 tokens after a
128-token context), median of repeated blocks."""
import json
import os
import statistics
import sys
import time
from pathlib import Path

os.environ["DD_PASS_KERNEL"] = "0"  # TP contexts run the per-launch path; compare like with like
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Target  # noqa: E402

shape = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "llama2_7b"]
ctx = [(7 * i) % 32000 for i in range(128)]
new = list(range(8))


def bench(group, reps=5, n=20):
    for t in group:
        t.truncate(0)
    for t in group:
        t.prefill(ctx)
    res = []
    for r in range(reps + 1):
        t0 = time.perf_counter()
        for _ in range(n):
            for t in group:
                t.truncate(len(ctx))
            for t in group:
                t.score(new)
            group[0].logits(0, 1)  # syncs rank 0 (the others finish with it)
        for t in group[1:]:
            t.logits(0, 1)
        if r:
            res.append((time.perf_counter() - t0) / n * 1e3)
    return statistics.median(res)


full = Target(shape, weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
t1 = bench([full])
full.close()
ranks = [Target(shape, weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024, tp_rank=r, tp_size=2)
         for r in range(2)]
Target.tp_connect_local(ranks)
t2 = bench(ranks)
print(json.dumps({"shape": sys.argv[1] if len(sys.argv) > 1 else "llama2_7b", "width": 8,
                  "context": 128, "tp1_ms_per_pass": round(t1, 3), "tp2_same_gpu_ms_per_pass": round(t2, 3),
                  "reductions_per_pass": 2 * shape["n_layers"] + 1,
                  "overhead_us_per_reduction": round((t2 - t1) * 1e3 / (2 * shape["n_layers"] + 1), 2)}))
