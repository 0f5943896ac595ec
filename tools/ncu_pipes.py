"""Summarise an ncu --csv metrics log of one forward (one row per launch): duration, tensor
pipe (HMMA/UTCHMMA subpipe) % of peak, DRAM % of peak and GB/s, per launch and per class."""
import csv
import sys
from collections import OrderedDict, defaultdict

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[start:]))
per = OrderedDict()
for r in rows:
    d = per.setdefault(r["ID"], {"name": r["Kernel Name"]})
    v = r["Metric Value"].replace(",", "")
    try:
        v = float(v)
    except ValueError:
        continue
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
    d[r["Metric Name"]] = v * scale
print(f"{'id':>3} {'us':>8} {'tensor%':>8} {'tc%':>6} {'dram%':>6} {'GB/s':>7}  kernel")
cls = defaultdict(lambda: [0.0, 0.0, 0.0, 0])
for i, d in per.items():
    ns = d.get("gpu__time_duration.sum", 0.0)
    by = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    t = d.get("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
    tc = d.get("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
    dr = d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0.0)
    name = d["name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:48]
    print(f"{i:>3} {ns / 1e3:8.1f} {t:8.1f} {tc:6.1f} {dr:6.1f} {by / max(ns, 1):7.0f}  {name}")
    c = cls[name.split("<")[0]]
    c[0] += ns; c[1] += t * ns; c[2] += by; c[3] += 1
print()
tot = sum(c[0] for c in cls.values())
print(f"{'class':<28} {'launches':>8} {'share':>6} {'tensor% (time-wtd)':>19} {'GB/s':>7}")
for k, c in sorted(cls.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:<28} {c[3]:8d} {c[0] / tot:6.1%} {c[1] / max(c[0], 1):19.1f} {c[2] / max(c[0], 1):7.0f}")
