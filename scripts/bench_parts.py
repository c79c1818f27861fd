"""Run single sub-measurements of bench.py (quick iteration / ncu captures).

  python scripts/bench_parts.py evict|policy|hash2 [--steps K] [--warmup W] [--no-cpu]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
ap = argparse.ArgumentParser()
ap.add_argument("part", choices=["evict", "policy", "hash2", "configs", "btab"])
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--no-cpu", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
if a.part == "evict":
    r = bench.measure_evict(dev, a)
elif a.part == "configs":
    r = bench.measure_configs(dev, a)
elif a.part == "policy":
    r = bench.measure_policy_eval(dev, a)
else:
    import paper_2603_10726_b200 as P
    s, _ = bench._workload("c2", 0)
    fn = bench.measure_hash2 if a.part == "hash2" else bench.measure_block_table
    r = fn(dev, a, P.to_device(s, dev), s)
print(json.dumps(r, indent=1))
