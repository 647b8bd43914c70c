"""DRAM traffic per launch from an ncu metrics CSV (--csv --log-file) into a
profiles/ summary bench.py reads as roofline.traffic.

usage: ncu_traffic.py <metrics.csv> <out.json> <kernel-substring>
(the capture: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
 --clock-control none -k regex:<kernel> --csv --log-file <metrics.csv> <command>)
"""
import csv
import json
import sys

src, out, pat = sys.argv[1:4]
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
hdr = rows[0]
ix = {k: i for i, k in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
launches = {}
for r in rows[1:]:
    name = r[ix["Kernel Name"]]
    if pat not in name:
        continue
    key = (r[ix["ID"]], name)
    rec = launches.setdefault(key, {"kernel": name[:120]})
    unit = r[ix["Metric Unit"]]
    val = float(r[ix["Metric Value"]].replace(",", ""))
    rec[r[ix["Metric Name"]]] = val * scale.get(unit, 1) if "bytes" in r[ix["Metric Name"]] else val
recs = list(launches.values())
summary = {"source": src, "kernel_filter": pat, "launches": recs}
if recs:
    summary["solver_dram_bytes_per_launch"] = recs[0].get("dram__bytes_read.sum", 0) + recs[0].get(
        "dram__bytes_write.sum", 0)
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1)[:800])
