"""Summarise an ncu --metrics launch list (CSV) of scripts/one_pass.py into a
per-kernel table of the LAST scored pass: serialised cold-cache times (shares),
DRAM bytes, and the GEMM DRAM traffic per pass (profiles/gemm_traffic.json)."""
import csv
import io
import json
import sys
from collections import OrderedDict

src, out_launch, out_traffic = sys.argv[1], sys.argv[2], sys.argv[3]
lines = [l for l in open(src) if not l.startswith("==")]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
launches = OrderedDict()
for r in rows:
    key = r["ID"]
    d = launches.setdefault(key, {"name": r["Kernel Name"].split("(")[0]})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    m = r["Metric Name"]
    if m == "gpu__time_duration.sum":
        d["us"] = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
    else:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
        d[m] = v * scale
L = list(launches.values())
# the last pass: from the last embed_norm_kernel to the end (minus the accept etc.)
last = max(i for i, d in enumerate(L) if d["name"].endswith("embed_norm_kernel"))
p = L[last:]
tot = sum(d["us"] for d in p)
per = OrderedDict()
for d in p:
    k = d["name"].split("::")[-1]
    e = per.setdefault(k, {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
    e["launches"] += 1
    e["us"] += d["us"]
    e["dram_bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
for k, e in per.items():
    e["share"] = round(e["us"] / tot, 4)
    e["us"] = round(e["us"], 1)
json.dump({"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                     "dram__bytes_write.sum --clock-control none python scripts/one_pass.py 8 "
                     "(serialised, cold cache: compare shares)",
           "pass_total_us_serialised": round(tot, 1), "kernels": per}, open(out_launch, "w"),
          indent=1)
g = [d for d in p if "gemm" in d["name"]]
gb = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in g)
alg = 13214154752
json.dump({"launches": len(g), "dram_bytes_per_pass": int(gb), "algorithmic_bytes_per_pass": alg,
           "ratio": round(gb / alg, 4), "width": 8}, open(out_traffic, "w"), indent=1)
print(json.dumps(per, indent=1))
print("gemm dram", gb, gb / alg)
