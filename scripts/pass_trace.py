"""Timeline of all GEMM launches of one pass (globaltimer per CTA)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, Target, _lib  # noqa: E402

t = Target(SHAPES["llama2_7b"], weight_seed=1, max_seq=512)
t.prefill(list(range(16)))
for w in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,16").split(",")]:
    N = 8 * 400 * 200
    buf = (C.c_uint64 * N)()
    nl, cpl = C.c_int(), C.c_int()
    rc = _lib.lib().dd_debug_pass_trace(t.h, w, buf, N, C.byref(nl), C.byref(cpl))
    assert rc == 0, _lib.lib().dd_last_error(t.h)
    a = np.frombuffer(buf, dtype=np.uint64)[: nl.value * 8 * cpl.value].reshape(nl.value, cpl.value, 8).astype(np.int64)
    t0 = a[0, :, 0][a[0, :, 0] > 0].min()
    names = ["qkv", "o", "gu", "down"] * 32 + ["head"]
    rows = []
    for i in range(nl.value):
        v = a[i][a[i, :, 0] > 0]
        st = (v[:, 0] - t0) / 1e3
        wt = (v[:, 2] - t0) / 1e3   # producer passed griddep wait
        mm = (v[:, 3] - t0) / 1e3   # last MMA issued
        ep = (v[:, 4] - t0) / 1e3   # epilogue done
        en = (v[:, 5] - t0) / 1e3   # CTA end
        ld = (v[:, 6] - t0) / 1e3   # last accumulator landed
        rows.append((names[i], st.min(), np.median(st), wt.min(), wt.max(), mm.max(), ep.max(), en.max(), ld.max(), np.median(ep - ld), (ep - ld).max()))
    tot = rows[-1][-1] - rows[0][1]
    print(f"w={w} total {tot:.1f} us over {nl.value} launches")
    for r in rows[:10] + rows[-6:]:
        print("  %-5s start[min,med]=%8.1f %8.1f waitpass[min,max]=%8.1f %8.1f lastmma=%8.1f epi_end=%8.1f end=%8.1f acc_landed=%8.1f epi_after_land[med,max]=%6.1f %6.1f" % r)
    # averages per layer position
    for k, nm in enumerate(["qkv", "o", "gu", "down"]):
        rr = [rows[4 * l + k] for l in range(32)]
        stream = np.mean([r[5] - r[4] for r in rr])
        tail = np.mean([r[7] - r[5] for r in rr])
        gap = np.mean([rows[4 * l + k + 1][4] - r[7] for l, r in enumerate(rr) if 4 * l + k + 1 < len(rows)])
        span = np.mean([r[7] - r[3] for r in rr])
        print(f"  {nm:5s}: waitpass->lastmma {stream:6.1f} us, lastmma->end {tail:5.1f} us, wait span {span:6.1f}, end->next wait max {gap:5.1f}")
