"""TP=2 group on ONE GPU (both ranks in this process): the persistent pass
kernel with the in-epilogue tile exchange (DD_TP_PASS=1, default) against the
per-launch path with separate reduction kernels (DD_TP_PASS=0): logits of a
W-token scored pass after a 128-token context must match the unsharded target
within bf16 tolerance and agree across ranks; wall time per pass (both ranks
share the GPU, 74 SMs each for the pass kernel).
python scripts/tp_pass_check.py [shape] [W]"""
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if len(sys.argv) > 3:  # child: one mode
    sys.path.insert(0, str(ROOT))
    import numpy as np
    from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Target
    shape, w = SHAPES[sys.argv[1]], int(sys.argv[2])
    ctx = [(7 * i) % shape["vocab"] for i in range(128)]
    new = [(13 * i + 5) % shape["vocab"] for i in range(w)]
    ranks = [Target(shape, weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024, tp_rank=r, tp_size=2)
             for r in range(2)]
    Target.tp_connect_local(ranks)
    for t in ranks:
        t.prefill(ctx)
    res = []
    for rep in range(6):
        t0 = time.perf_counter()
        for _ in range(10):
            for t in ranks:
                t.truncate(len(ctx))
            for t in ranks:
                t.score(new)
            g0 = ranks[0].logits(0, w)  # synchronises rank 0 (rank 1 finishes with it)
        g1 = ranks[1].logits(0, w)
        if rep:
            res.append((time.perf_counter() - t0) / 10 * 1e3)
    np.save(sys.argv[3], np.stack([g0, g1]))
    print("MS", statistics.median(res))
    sys.exit(0)

shape = sys.argv[1] if len(sys.argv) > 1 else "llama2_7b"
w = sys.argv[2] if len(sys.argv) > 2 else "8"
out = {}
for mode in ("1", "0"):
    env = dict(os.environ, DD_TP_PASS=mode)
    p = subprocess.run([sys.executable, __file__, shape, w, f"/tmp/tp_{mode}.npy"], env=env,
                       capture_output=True, text=True, timeout=600)
    ms = [l for l in p.stdout.splitlines() if l.startswith("MS")]
    out[mode] = float(ms[0].split()[1]) if ms else p.stderr[-400:]
import numpy as np  # noqa: E402
a, b = np.load("/tmp/tp_1.npy"), np.load("/tmp/tp_0.npy")
print(json.dumps({"shape": shape, "width": int(w), "context": 128,
                  "pass_kernel_ms_per_pass_incl_host": out["1"], "per_launch_ms_per_pass_incl_host": out["0"],
                  "ranks_agree_pass_kernel": bool(np.array_equal(a[0], a[1])),
                  "rel_diff_pass_vs_per_launch": float(np.abs(a[0] - b[0]).max() / np.abs(b[0]).max())}))
