"""Run one tiny (or 7B) pass with the persistent kernel under a watchdog that
dumps per-CTA progress words if the pass does not finish (debug only)."""
import ctypes as C
import os
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2503_00784_b200 import SHAPES, Target, _lib  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "tiny"
lib = _lib.lib()
lib.dd_debug_pass_progress.restype = C.c_void_p
ptr = lib.dd_debug_pass_progress()
prog = (C.c_int * (148 * 8)).from_address(ptr)


def dump():
    a = np.array(prog[:], dtype=np.int64).reshape(148, 8)
    names = ["wprod_phase", "xprod_pre_empty", "xprod_pre_flag", "mma_tile", "epi_phase",
             "epi_tile", "attn_item", "done"]
    for j, n in enumerate(names):
        col = a[:, j]
        vals, cnt = np.unique(col, return_counts=True)
        order = np.argsort(-cnt)[:6]
        print(f"{n:16s}", " ".join(f"{vals[i]}x{cnt[i]}" for i in order), "| min", col.min(), flush=True)


def watchdog(tag, secs):
    time.sleep(secs)
    print("WATCHDOG", tag, flush=True)
    dump()
    os._exit(3)


t = Target(SHAPES[shape], weight_seed=5, max_seq=512)
wd = threading.Thread(target=watchdog, args=("prefill", 20), daemon=True)
wd.start()
t.prefill(list(range(1, 40)))
print("prefill ok", flush=True)
dump()
t.score([5, 6, 7])
g = t.logits(0, 3)
print("score ok", np.abs(g).max(), flush=True)
os._exit(0)
