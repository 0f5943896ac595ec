"""Parse an ncu --csv metrics log (dram__bytes_read.sum, dram__bytes_write.sum,
gpu__time_duration.sum per launch) and write profiles/traffic_<workload>.json: measured DRAM
bytes per launch of the dominant kernel class (bench.py's roofline "traffic")."""
import csv
import json
import sys
from collections import defaultdict

log, workload, kernel = sys.argv[1], sys.argv[2], (sys.argv[3] if len(sys.argv) > 3 else "conv_tc_kernel")
lines = open(log).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[start:]))
per = defaultdict(dict)
for r in rows:
    if kernel not in r["Kernel Name"]:
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
    per[r["ID"]][r["Metric Name"]] = v * scale
    per[r["ID"]]["name"] = r["Kernel Name"][:80]
launches = []
for i, d in per.items():
    launches.append({"id": int(i), "kernel": d["name"], "dram_read": d.get("dram__bytes_read.sum", 0.0),
                     "dram_write": d.get("dram__bytes_write.sum", 0.0), "ns": d.get("gpu__time_duration.sum", 0.0)})
launches.sort(key=lambda x: x["id"])
tot = sum(l["dram_read"] + l["dram_write"] for l in launches)
out = {"workload": workload, "kernel": kernel, "launches": len(launches),
       "bytes_per_launch": tot / max(len(launches), 1), "bytes_total": tot,
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 "--clock-control none (cold caches, serialized; one forward of tools/prof_step.py)",
       "per_launch": launches}
json.dump(out, open(f"profiles/traffic_{workload}.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "per_launch"}))
