"""Sweep GEMM pre-wait L2 prefetch / CTAs (device time via the C ABI)."""
import os
import subprocess
import sys

code = r'''
import sys
sys.path.insert(0, ".")
from paper_2503_00784_b200 import SHAPES, Target
t = Target(SHAPES["llama2_7b"], weight_seed=1, plant=None, max_seq=512)
t.prefill(list(range(16)))
out = []
for w in (1, 8, 16):
    ms, n = t.time_gemms(w, trials=5)
    out.append(f"w{w}={ms:.3f}ms/{t.pass_weight_bytes() / ms / 1e6:.0f}GB/s")
print("RESULT", " ".join(out), "pass_w1=%.3f pass_w8=%.3f" % (t.time_pass(1), t.time_pass(8)))
'''
for stages, pf, ctas in [(0, 0, 0), (0, 8, 0), (0, 16, 0), (0, 32, 0), (4, 16, 0), (0, 16, 148)]:
    env = dict(os.environ)
    if stages:
        env["DD_GEMM_STAGES"] = str(stages)
    if ctas:
        env["DD_GEMM_CTAS"] = str(ctas)
    env["DD_GEMM_PREFETCH"] = str(pf)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
    print(f"stages={stages} prefetch={pf} ctas={ctas}:", line[0] if line else r.stderr[-200:], flush=True)
