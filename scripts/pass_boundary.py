"""Where does a GEMM phase's tail go?  Per-CTA stamps of one phase (o1 by
default): last weight k-block issued (2), accumulator ready (4), reducer saw
all partials (5), partials summed (8), epilogue done (9), flag published (6)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target, _lib  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 8
t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
t.prefill([(7 * i) % 32000 for i in range(128)])
lib = _lib.lib()
cap = 148 * 200 * 12
buf = (C.c_uint64 * cap)()
n = C.c_int()
rc = lib.dd_debug_pass_timeline(t.h, w, buf, C.c_size_t(cap), C.byref(n))
assert rc == 0, lib.dd_last_error(t.h)
a = np.frombuffer(buf, dtype=np.uint64)[: 148 * n.value * 12].reshape(148, n.value, 12).astype(np.float64)
t0 = a[:, :, 0][a[:, :, 0] > 0].min()
a = np.where((a > 0) & (a > t0 - 1e9), (a - t0) / 1e3, np.nan)
names = ["embed"] + [x for l in range(32) for x in (f"qkv{l}", f"attn{l}", f"o{l}", f"gu{l}", f"dn{l}")] + ["head"]
for ph in (7, 8, 9, 10, 11):
    r = a[:, ph, :]
    print(f"== {names[ph]}: inputs {np.nanmin(r[:,1]):.1f}/{np.nanmax(r[:,1]):.1f}  issue-done {np.nanmin(r[:,2]):.1f}/{np.nanmax(r[:,2]):.1f}"
          f"  acc-ready {np.nanmin(r[:,4]):.1f}/{np.nanmax(r[:,4]):.1f}  publish {np.nanmin(r[:,6]):.1f}/{np.nanmax(r[:,6]):.1f}"
          f"  epi-done {np.nanmin(r[:,3]):.1f}/{np.nanmax(r[:,3]):.1f}")
    red = ~np.isnan(r[:, 5])
    if red.any():
        print(f"   reducers {red.sum()}: acc-ready->all-partials {np.nanmedian(r[red,5]-r[red,4]):.2f} (max {np.nanmax(r[red,5]-r[red,4]):.2f})"
              f"  ->summed {np.nanmedian(r[red,8]-r[red,5]):.2f}  ->epi {np.nanmedian(r[red,9]-r[red,8]):.2f}"
              f"  ->publish {np.nanmedian(r[red,6]-r[red,9]):.2f}  issue-done->acc-ready {np.nanmedian(r[red,4]-r[red,2]):.2f}")
    for cta in (0, 1, 2, 37, 74, 111, 147):
        print(f"   cta {cta:3d}: " + " ".join(f"{k}:{r[cta,k]:.1f}" for k in (1, 2, 4, 5, 8, 9, 6, 3) if not np.isnan(r[cta, k])))
