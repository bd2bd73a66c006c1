"""Is per-CTA streaming speed tied to the SM, and stable across launches?"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target, _lib  # noqa: E402

t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
t.prefill(list(range(128)))
lib = _lib.lib()
runs = []
for rep in range(3):
    cap = 148 * 200 * 12 + 200 * 512 + 148 * 200 * 4
    buf = (C.c_uint64 * cap)()
    n = C.c_int()
    assert lib.dd_debug_pass_timeline(t.h, 8, buf, C.c_size_t(cap), C.byref(n)) == 0
    a = np.frombuffer(buf, dtype=np.uint64)[: 148 * n.value * 12].reshape(148, n.value, 12).astype(np.float64)
    smid = a[:, 0, 10].astype(int)
    # GU phases, layers 1..30: MMA span per CTA
    d = np.array([(a[:, 1 + 5 * l + 3, 2] - a[:, 1 + 5 * l + 3, 1]) / 1e3 for l in range(1, 31)]).mean(0)
    runs.append((smid, d))
    print(f"run {rep}: span min/med/max {d.min():.1f} {np.median(d):.1f} {d.max():.1f}; smid of CTA 0..7 {smid[:8]}")
for i in range(1, 3):
    s0, d0 = runs[0]
    s1, d1 = runs[i]
    by_sm0 = np.zeros(148); by_sm0[s0] = d0
    by_sm1 = np.zeros(148); by_sm1[s1] = d1
    print(f"run0 vs run{i}: corr by CTA {np.corrcoef(d0, d1)[0,1]:.2f}, by SM {np.corrcoef(by_sm0, by_sm1)[0,1]:.2f}, same mapping {np.mean(s0 == s1):.2f}")
by = np.zeros(148); by[runs[0][0]] = runs[0][1]
print("per-SM span (us), smid order:", np.round(by, 1).tolist())
