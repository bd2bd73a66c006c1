"""Per-phase timeline of one persistent-kernel pass (globaltimer stamps per CTA)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Target, _lib  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n_ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 128
t = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
t.prefill([(7 * i) % 32000 for i in range(n_ctx)])
lib = _lib.lib()
cap = 148 * 200 * 12
buf = (C.c_uint64 * cap)()
n = C.c_int()
rc = lib.dd_debug_pass_timeline(t.h, w, buf, C.c_size_t(cap), C.byref(n))
assert rc == 0, lib.dd_last_error(t.h)
a = np.frombuffer(buf, dtype=np.uint64)[: 148 * n.value * 12].reshape(148, n.value, 12).astype(np.float64)
if len(sys.argv) > 3:
    np.save(sys.argv[3] + ".raw.npy", a[:, :, 10])
t0 = a[:, :, 0][a[:, :, 0] > 0].min()
a = np.where(a > 0, (a - t0) / 1e3, np.nan)
if len(sys.argv) > 3:
    np.save(sys.argv[3], a)
names = ["embed"] + [x for l in range(32) for x in (f"qkv{l}", f"attn{l}", f"o{l}", f"gu{l}", f"dn{l}")] + ["head"]
print("phase      wstart(min/max)   inputs(min/max)    mma_done(min/max)   epi_done(min/max)  -  -  publish  enter-poll  wend")
for p in range(n.value):
    if not (p <= 1 or 6 <= p <= 11 or p >= n.value - 2):
        continue
    r = a[:, p, :]
    def mm(k):
        col = r[:, k]
        col = col[~np.isnan(col)]
        return f"{col.min():8.1f}/{col.max():8.1f}" if len(col) else "      -/-      "
    print(f"{names[p]:8s} {mm(0)} {mm(1)} {mm(2)} {mm(3)} {mm(6)} {mm(7)} {mm(11)}")
end = np.nanmax(a)
print("total span us", round(end, 1))
# per-layer averages of (epi_done max of dn) deltas
dn = [np.nanmax(a[:, 1 + 5 * l + 4, 3]) for l in range(32)]
print("per-layer us", np.round(np.diff(dn).mean(), 2))
for k, nm in ((0, "qkv"), (1, "attn"), (2, "o"), (3, "gu"), (4, "dn")):
    # average over layers of (epi_done max) - (previous phase epi_done max)
    d = [np.nanmax(a[:, 1 + 5 * l + k, 3]) - np.nanmax(a[:, 1 + 5 * l + k - 1, 3]) for l in range(1, 32)]
    print(f"  {nm}: +{np.mean(d):.2f} us (epi_done max to epi_done max)")

# per-CTA detail for gu1 (phase 9) inputs vs o1 (phase 8) publishes
po = a[:, 8, 6]
print("o1 publish: sorted last 8", np.round(np.sort(po[~np.isnan(po)])[-8:], 1))
for cta in range(0, 148, 21):
    r = a[cta, 9]
    print(f"cta {cta}: gu1 enter-poll {r[7]:.1f} polled {r[4]:.1f} fenced {r[5]:.1f} wstart {r[0]:.1f} | o1 mma_done {a[cta, 8, 2]:.1f} epi_done {a[cta, 8, 3]:.1f}")

# per-CTA streaming speed consistency across layers (GU phases)
d = np.array([a[:, 1 + 5 * l + 3, 2] - a[:, 1 + 5 * l + 3, 1] for l in range(1, 31)])  # [layer, cta]
m = d.mean(0)
print("GU mma span per CTA: mean over layers min/median/max", np.round(m.min(), 1), np.round(np.median(m), 1), np.round(m.max(), 1))
print("layer-to-layer corr of per-CTA span:", np.round(np.corrcoef(d[0], d[1])[0, 1], 2), np.round(np.corrcoef(d[5], d[20])[0, 1], 2))
order = np.argsort(m)
print("slowest CTAs:", order[-12:], "fastest:", order[:12])
sm = np.round(m, 1)
print("even/odd CTA mean:", sm[::2].mean(), sm[1::2].mean(), " first/second half:", sm[:74].mean(), sm[74:].mean())
for k, nm in ((0, "qkv"), (2, "o"), (3, "gu"), (4, "dn")):
    sp = [np.nanmax(a[:, 1 + 5 * l + k, 2]) - np.nanmin(a[:, 1 + 5 * l + k, 1]) for l in range(1, 31)]
    print(f"  {nm} inputs(min)->mma_done(max) {np.mean(sp):.1f} us")
