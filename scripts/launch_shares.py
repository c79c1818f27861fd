"""Per-kernel totals and shares of an ncu launch list (gpu__time_duration.sum [+ dram bytes]).

  python scripts/launch_shares.py profiles/r01/launches_evict.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
per = {}
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    key = (int(r[ix["ID"]]), r[ix["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0])
    per.setdefault(key, {})[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
unit = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot, allus = {}, 0.0
for (i, n), m in per.items():
    t = m["gpu__time_duration.sum"]
    us = float(t[0].replace(",", "")) * unit[t[1]]
    b = sum(float(m[k][0].replace(",", "")) * scale.get(m[k][1], 1)
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
    e = tot.setdefault(n, [0.0, 0, 0.0])
    e[0] += us; e[1] += 1; e[2] += b
    allus += us
print(f"{'kernel':40s} {'launches':>8s} {'us':>9s} {'share':>6s} {'DRAM MB':>9s}")
for n, (us, c, b) in sorted(tot.items(), key=lambda x: -x[1][0]):
    print(f"{n:40s} {c:8d} {us:9.1f} {100 * us / allus:5.1f}% {b / 1e6:9.1f}")
print(f"{'total':40s} {'':8s} {allus:9.1f}")
