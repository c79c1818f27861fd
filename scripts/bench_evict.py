"""Only the evict-mode measurement of bench.py (quick iteration)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--no-cpu", action="store_true")
a = ap.parse_args()
print(json.dumps(bench.measure_evict(torch.device("cuda", 0), a), indent=1))
if os.environ.get("POLICY_EVAL"):
    print(json.dumps(bench.measure_policy_eval(torch.device("cuda", 0), a), indent=1))
