"""Where an engine iteration's time goes beyond the scored pass (config 2):
per-iteration target_ms / verify_ms / comm_ms (IterationRecord) against the
pass time at the iteration's width, for duo at the calibrated budget."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Draft, EngineConfig, Target, run_generation  # noqa: E402

tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
drf = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=12, cpus=list(range(2, 14)))
prompt = np.random.default_rng(1).integers(0, 32000, 128).tolist()
bud = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = EngineConfig(mode="duo", budget=bud, max_sequences=4, max_new_tokens=128, greedy=True)
for rep in range(3):
    r = run_generation(tgt, drf, prompt, cfg)
its = r.iterations[1:]
widths = sorted({it.width for it in its})
tgt.truncate(0)
tgt.prefill(prompt)
pass_ms = {w: tgt.time_pass(w, trials=10) for w in widths}
tot = sum(it.target_ms for it in its)
passes = sum(pass_ms[it.width] for it in its)
print(f"iterations {len(its)}  tps {r.tps:.1f}  decode sum target_ms {tot:.2f}  sum pass_ms(width) {passes:.2f}  "
      f"overhead/iter {(tot - passes) / len(its) * 1e3:.1f} us")
print(f"mean verify_ms {np.mean([it.verify_ms for it in its]) * 1e3:.1f} us  mean comm_ms "
      f"{np.mean([it.comm_ms for it in its]) * 1e3:.1f} us  mean draft_ms {np.mean([it.draft_ms for it in its]):.3f}")
for w in widths:
    sel = [it for it in its if it.width == w]
    print(f"  width {w:3d}: n={len(sel):3d} target_ms {np.mean([it.target_ms for it in sel]):.3f} pass {pass_ms[w]:.3f} "
          f"comm {np.mean([it.comm_ms for it in sel]):.3f} verify {np.mean([it.verify_ms for it in sel]):.3f} "
          f"draft {np.mean([it.draft_ms for it in sel]):.3f}")

# the same pass + verify + truncate cycle without the draft: host/launch overhead alone
import time  # noqa: E402
for w in (1, 16):
    tgt.truncate(0)
    tgt.prefill(prompt)
    n0 = len(prompt)
    ts = []
    for i in range(30):
        t0 = time.perf_counter()
        tgt.score([(13 * i + j) % 32000 for j in range(w)])
        tgt.verify(0, tail_len=w - 1, firsts=[5], seed=2, counter=0, q_onehot=True)
        ts.append((time.perf_counter() - t0) * 1e3)
        tgt.truncate(n0)
    print(f"no draft: width {w}: pass+verify wall {np.median(ts):.3f} ms (pass {pass_ms.get(w, tgt.time_pass(w)):.3f})")
