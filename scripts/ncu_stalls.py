"""Stall-reason breakdown of an ncu --set full capture over a SASS index range
(from `ncu --page source --csv --print-source sass`):
python scripts/ncu_stalls.py REPORT.ncu-rep [first_idx last_idx | auto-hmma]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, data = rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
else:  # the HMMA-dense region (attention), widened
    hm = [k for k, r in enumerate(data) if "HMMA" in r[1]]
    lo, hi = hm[0] - 300, hm[len(hm) // 2] + 200
num = lambda r, h: int(r[col[h]]) if r[col[h]].isdigit() else 0
tot = {h: sum(num(r, h) for r in data[lo:hi]) for h in reasons}
alls = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
reg = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data[lo:hi])
ins = sum(num(r, "Instructions Executed") for r in data[lo:hi])
print(f"range [{lo}, {hi}): {reg} of {alls} samples, {ins} warp instructions executed")
for h, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v:
        print(f"  {h:24s} {v:8d}  {v / max(reg, 1):.1%}")
print("top instructions:")
top = sorted(range(lo, hi), key=lambda k: -num(data[k], "Warp Stall Sampling (All Samples)"))[:25]
for k in sorted(top):
    r = data[k]
    main = max(reasons, key=lambda h: num(r, h))
    print(f"  {k:6d} {num(r, 'Warp Stall Sampling (All Samples)'):6d} {main[6:]:14s} "
          f"x{num(r, 'Instructions Executed'):8d}  {r[1].strip()[:80]}")
