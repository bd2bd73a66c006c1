"""Per-CTA timeline of the wide (prefill) GEMM launches of one pass."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target, _lib  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 127
t = Target(SHAPES["llama2_7b"], weight_seed=1, plant=DEFAULT_PLANT, max_seq=1024)
t.prefill(list(range(16)))
N = 129 * 8 * 148
buf = (C.c_uint64 * N)()
nl = C.c_int()
rc = _lib.lib().dd_debug_prefill_trace(t.h, w, buf, N, C.byref(nl))
assert rc == 0, _lib.lib().dd_last_error(t.h)
a = np.frombuffer(buf, dtype=np.uint64).reshape(129, 148, 8).astype(np.float64)
names = ["qkv", "o", "gu", "down"]
for k, nm in enumerate(names):
    rows = []
    for l in range(1, 31):
        v = a[4 * l + k]
        v = v[v[:, 0] > 0]
        st, wt, mm, ep, en, ld = (v[:, i] for i in (0, 2, 3, 4, 5, 6))
        rows.append(((wt.max() - st.min()), (mm.max() - wt.min()), (ld.max() - mm.max()), (ep.max() - ld.max()),
                     (en.max() - st.min()), np.median(ep - ld)))
    r = np.array(rows).mean(0) / 1e3
    print(f"{nm:5s}: start->waitpass {r[0]:6.1f}  stream(wait->last MMA issued) {r[1]:6.1f}  mma drain {r[2]:6.1f}  "
          f"epi tail {r[3]:6.1f} (median CTA {r[5]:5.1f})  total {r[4]:6.1f} us")
