"""Key metrics of `ncu --set full` reports -> JSON (profiles/rNN/ncu_full_summary.json).

  python scripts/ncu_full_summary.py COMMIT gpurun_out/full_k_*.ncu-rep > profiles/r02/ncu_full_summary.json
"""
import csv
import json
import os
import subprocess
import sys

WANT = {"Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Compute (SM) Throughput", "Mem Busy", "Max Bandwidth",
        "Block Limit Registers", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "No Eligible", "Active Warps Per Scheduler"}
out = {"commit": sys.argv[1], "command": "ncu --set full --clock-control none --import-source on "
       "-k regex:^K -s 1 -c 1 python bench.py --profile --steps 1 --warmup 1 --no-cpu "
       "(scripts/r2_profile.sh; C2 bench step, second launch of each kernel)", "kernels": {}}
for rep in sys.argv[2:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if not rows:
        continue
    ix = {k: i for i, k in enumerate(rows[0])}
    m = {}
    for r in rows[1:]:
        name = r[ix["Metric Name"]]
        if name in WANT and name not in m:
            m[name] = f"{r[ix['Metric Value']]} {r[ix['Metric Unit']]}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) >= 3:
        h = rr[0]
        for k in ["dram__bytes_read.sum", "dram__bytes_write.sum"]:
            if k in h:
                m[k] = f"{rr[2][h.index(k)]} {rr[1][h.index(k)]}"
    out["kernels"][os.path.basename(rep).replace("full_", "").replace(".ncu-rep", "")] = m
print(json.dumps(out, indent=1))
