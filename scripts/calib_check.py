"""calibrate() on the 7B target and the 68M draft pinned to 12 host cores: c and the budget."""
import sys, os
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target, Draft, calibrate
t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
cpus = sorted(os.sched_getaffinity(0))[1:13]
d = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=len(cpus), cpus=cpus)
print("calibrate", calibrate(t, d, probe_len=8, trials=12))
print("draft token ms", d.time_token(12))
for n in (8, 128):
    t.truncate(0); t.prefill(list(range(n)))
    print("n", n, "pass(8) ms", t.time_pass(8, 12), "pass(1)", t.time_pass(1, 12))
