"""Summarize an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel.

Usage: python tools/ncu_summarize.py launches.csv out.json [--last-frame]
--last-frame keeps only the launches from the last k_prologue on (one steady frame).
"""
import csv
import json
import sys
from collections import OrderedDict, defaultdict

src, dst = sys.argv[1], sys.argv[2]
last = "--last-frame" in sys.argv
rows = []
with open(src) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    rows.append(r)
by_id = OrderedDict()
for r in rows:
    d = by_id.setdefault(r["ID"], {"name": r["Kernel Name"], "m": {}})
    try:
        d["m"][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    except ValueError:
        pass
launches = list(by_id.values())
if last:
    idx = [i for i, d in enumerate(launches) if "k_prologue" in d["name"]]
    if idx:
        launches = launches[idx[-1]:]
agg = defaultdict(lambda: {"launches": 0, "sum_us": 0.0, "sum_dram": 0.0})
for d in launches:
    key = d["name"].split("(")[0]
    a = agg[key]
    a["launches"] += 1
    a["sum_us"] += d["m"].get("gpu__time_duration.sum", 0.0) / 1e3
    a["sum_dram"] += d["m"].get("dram__bytes_read.sum", 0.0) + d["m"].get("dram__bytes_write.sum", 0.0)
out = {}
total = sum(a["sum_us"] for a in agg.values())
for k, a in agg.items():
    out[k] = {"launches": a["launches"], "mean_us": a["sum_us"] / a["launches"], "total_us": a["sum_us"],
              "share_of_frame": a["sum_us"] / total if total else None,
              "dram_bytes_per_launch": a["sum_dram"] / a["launches"]}
json.dump({"source": src, "last_frame_only": last, "kernels": out, "frame_sum_us": total}, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
