"""Per-kernel summary (µs, DRAM bytes) of an ncu launch list -> profiles/latest_ncu.json.

  python scripts/ncu_json.py gpurun_out/launches.csv profiles/r02/launches_c2.csv [commit] > profiles/latest_ncu.json

The Activator section of the previous profiles/latest_ncu.json is carried over (its kernels are
profiled by scripts/profile_activator.sh).

Only launches of the second bench step are kept (the first step includes one-time setup)."""
import csv
import json
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
    key = (int(r[ix["ID"]]), r[ix["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0])
    per.setdefault(key, {})[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
launches = [(i, n, m) for (i, n), m in per.items()]
hashes = [k for k, (i, n, m) in enumerate(launches) if n == "k_hash_register"]
second = launches[hashes[1]:] if len(hashes) > 1 else launches
unit = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
commit = sys.argv[3] if len(sys.argv) > 3 else "unknown"
out = {"source": f"{sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]} (commit {commit}): ncu --metrics "
                 "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                 "lts__t_sector_hit_rate.pct,smsp__inst_executed.sum "
                 "--clock-control none, bench.py --profile --steps 1 --warmup 1 (C2, second step)",
       "kernels": OrderedDict()}
for i, n, m in second:
    t = m["gpu__time_duration.sum"]
    d = {"us": round(float(t[0].replace(",", "")) * unit.get(t[1], 1.0), 1)}
    for k, name in [("dram__bytes_read.sum", "dram_read"), ("dram__bytes_write.sum", "dram_write")]:
        if k in m:
            d[name] = int(float(m[k][0].replace(",", "")) * scale.get(m[k][1], 1))
    if "smsp__inst_executed.sum" in m:
        d["warp_instructions"] = int(float(m["smsp__inst_executed.sum"][0].replace(",", "")))
    if "lts__t_sector_hit_rate.pct" in m:
        d["l2_hit_pct"] = round(float(m["lts__t_sector_hit_rate.pct"][0].replace(",", "")), 1)
    if "dram_read" in d and "dram_write" in d:
        d["traffic"] = d["dram_read"] + d["dram_write"]
    out["kernels"].setdefault(n, []).append(d)
try:
    prev = json.load(open("profiles/latest_ncu.json"))
    if "activator" in prev:
        out["activator"] = prev["activator"]
except (OSError, ValueError):
    pass
print(json.dumps(out, indent=1))
