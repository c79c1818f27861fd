"""Summarise an ncu --csv launch list: per-kernel device time (and DRAM bytes if captured)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
per = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    key = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0])
    per.setdefault(key, {})[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
tot = 0.0
for (i, name), m in per.items():
    t = m.get("gpu__time_duration.sum", ("0", ""))
    tv = float(t[0].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(t[1], 1.0)
    tot += tv
    extra = "  ".join(f"{k.split('__')[1].split('.')[0]}={v[0]} {v[1]}" for k, v in m.items()
                      if k != "gpu__time_duration.sum")
    print(f"{i:>4} {name:<40} {tv:9.1f} us  {extra}")
print(f"total {tot:.1f} us over {len(per)} launches")
