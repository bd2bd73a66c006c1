"""Summarise an ncu --set full report into profiles/ JSON:
python scripts/ncu_summary.py REPORT.ncu-rep OUT.json "capture command" [launch index]"""
import csv
import io
import json
import subprocess
import sys

rep, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
idx = sys.argv[4] if len(sys.argv) > 4 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.DictReader(io.StringIO(txt)))
ids = sorted({r["ID"] for r in rows}, key=int)
sel = idx if idx is not None else ids[0]
res = {"kernel": None, "capture": cmd, "metrics": {}, "rules": []}
for r in rows:
    if r["ID"] != sel:
        continue
    res["kernel"] = r["Kernel Name"].split("(")[0]
    if r["Metric Name"]:
        res["metrics"][f'{r["Section Name"]} / {r["Metric Name"]}'] = \
            f'{r["Metric Value"]} {r["Metric Unit"]}'.strip()
    if r.get("Rule Name") and r.get("Rule Description"):
        res["rules"].append({"rule": r["Rule Name"], "speedup": r.get("Estimated Speedup"),
                             "text": r["Rule Description"][:400]})
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                      "lts__t_sector_hit_rate.pct,sm__pipe_tensor_op_umma_cycles_active.avg.pct_of_peak_sustained_active"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    hdr, units = rr[0], rr[1]
    for row in rr[2:]:
        if row[0] == sel:
            for h, u, v in zip(hdr, units, row):
                if "__" in h:
                    res["metrics"]["raw / " + h] = f"{v} {u}".strip()
json.dump(res, open(out, "w"), indent=1)
for k, v in res["metrics"].items():
    if any(s in k for s in ("Duration", "DRAM Throughput", "Memory Throughput", "Issued Warp",
                            "No Eligible", "Registers", "raw /")):
        print(k, v)
