"""Per-CTA timeline of the layer-0 GEMMs (globaltimer), summarised."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, Target, _lib  # noqa: E402

t = Target(SHAPES["llama2_7b"], weight_seed=1, max_seq=512)
t.prefill(list(range(64)))  # context
names = ["qkv", "o", "gate_up", "down", "head"]
for which in range(5):
    for w in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,16").split(",")]:
        buf = (C.c_uint64 * (8 * 4096))()
        n = C.c_int()
        rc = _lib.lib().dd_debug_gemm_trace(t.h, which, w, buf, 4096, C.byref(n))
        assert rc == 0, _lib.lib().dd_last_error(t.h)
        a = np.frombuffer(buf, dtype=np.uint64)[: 8 * n.value].reshape(n.value, 8).astype(np.int64)
        t0 = a[:, 0].min()
        rel = (a[:, :6] - t0) / 1000.0  # us
        span = rel[:, 5].max()
        setup = rel[:, 1] - rel[:, 0]
        first = rel[:, 2] - rel[:, 1]
        stream = rel[:, 3] - rel[:, 2]
        drain = rel[:, 4] - rel[:, 3]
        epi = rel[:, 5] - rel[:, 4]
        starts = np.sort(rel[:, 0])
        print(f"{names[which]:8s} w={w:2d} ctas={n.value:4d} span={span:7.2f}us  start[p50,p90,max]="
              f"{np.percentile(starts,50):.2f},{np.percentile(starts,90):.2f},{starts.max():.2f}  "
              f"setup={setup.mean():.2f} first_stage={first.mean():.2f} stream={stream.mean():.2f} "
              f"(max {stream.max():.2f}) drain={drain.mean():.2f} epi={epi.mean():.2f}(max {epi.max():.2f}) "
              f"smids={len(set(a[:,7]))}", flush=True)
