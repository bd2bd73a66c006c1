"""profiles/pass_traffic.json from ncu launch lists of scripts/one_pass.py
(one CSV per width, dram bytes + duration of the pass_kernel launches):
python scripts/traffic_json.py CTX W1:csv1 W2:csv2 ..."""
import csv
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
ctx = int(sys.argv[1])
WEIGHTS = 13214154752
out = {"kernel": "pass_kernel", "context": ctx,
       "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 "--clock-control none -k regex:pass_kernel python scripts/one_pass.py W CTX "
                 "(three scored passes of width W after a CTX-token prefill; scripts/profile_refresh.sh)",
       "algorithmic_weight_bytes_per_pass": WEIGHTS, "widths": {}}
for arg in sys.argv[2:]:
    w, path = arg.split(":", 1)
    lines = [l for l in open(path) if not l.startswith("==")]
    per = {}
    for r in csv.DictReader(io.StringIO("".join(lines))):
        v = float(r["Metric Value"].replace(",", ""))
        per.setdefault(r["ID"], {})[r["Metric Name"]] = v
    rows = list(per.values())
    rd = sum(x["dram__bytes_read.sum"] for x in rows) / len(rows)
    wr = sum(x["dram__bytes_write.sum"] for x in rows) / len(rows)
    us = sum(x["gpu__time_duration.sum"] for x in rows) / len(rows) / 1e3
    out["widths"][w] = {"launches": len(rows), "dram_bytes_per_pass": int(rd + wr),
                        "dram_read_bytes_per_pass": int(rd), "dram_write_bytes_per_pass": int(wr),
                        "ratio_read_to_weights": round(rd / WEIGHTS, 4),
                        "duration_us_per_launch_ncu": round(us, 1)}
(ROOT / "profiles" / "pass_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
