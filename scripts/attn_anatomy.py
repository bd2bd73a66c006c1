"""Anatomy of the decode attention phase inside the persistent pass kernel:
per layer, QKV tile publishes -> attention item stamps (entered, flags seen,
first chunk staged, chunks done, o stored, published) -> O-phase activation
inputs.  Averages over layers 1..30 (us relative to the layer's last QKV MMA)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target, _lib  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 9
n_ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 128
t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
t.prefill([(7 * i) % 32000 for i in range(n_ctx)])
lib = _lib.lib()
cap = 148 * 200 * 12
rows = []
for rep in range(3):
    buf = (C.c_uint64 * cap)()
    n = C.c_int()
    rc = lib.dd_debug_pass_timeline(t.h, w, buf, C.c_size_t(cap), C.byref(n))
    assert rc == 0, lib.dd_last_error(t.h)
    a = np.frombuffer(buf, dtype=np.uint64)[: 148 * n.value * 12].reshape(148, n.value, 12).astype(np.float64)
    a = np.where(a > 0, a / 1e3, np.nan)
    for l in range(1, 31):
        pq, pa, po = 1 + 5 * l, 2 + 5 * l, 3 + 5 * l
        ref = np.nanmax(a[:, pq, 2])  # last QKV MMA done
        r = {"qkv_mma_done_min": np.nanmin(a[:, pq, 2]) - ref,
             "qkv_publish_max": np.nanmax(a[:, pq, 6]) - ref}
        for k, nm in ((0, "entered"), (1, "flags"), (2, "chunk0"), (4, "chunks_done"), (5, "stored"),
                      (6, "published"), (3, "phase_end")):
            col = a[:, pa, k] - ref
            r[f"attn_{nm}_min"] = np.nanmin(col)
            r[f"attn_{nm}_max"] = np.nanmax(col)
        A = a[:, pa, :]
        ok = ~np.isnan(A[:, 0]) & ~np.isnan(A[:, 4])
        for nm, k1, k0 in (("d_entry_to_flags", 1, 0), ("d_flags_to_chunk0", 2, 1),
                           ("d_chunk0_to_done", 4, 2), ("d_done_to_phase_end", 3, 4)):
            r[nm] = np.nanmean(A[ok, k1] - A[ok, k0])
        r["o_inputs_min"] = np.nanmin(a[:, po, 1]) - ref
        r["o_inputs_max"] = np.nanmax(a[:, po, 1]) - ref
        r["o_mma_done_max"] = np.nanmax(a[:, po, 2]) - ref
        rows.append(r)
print(f"W={w} ctx={n_ctx}: us relative to the layer's last QKV MMA completion (mean over layers 1..30, 3 passes)")
for k in rows[0]:
    print(f"  {k:24s} {np.mean([r[k] for r in rows]):7.2f}")
