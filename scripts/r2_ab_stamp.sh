#!/bin/bash
# A/B of the resolver's inserter-stamp rule (SOLID_STAMP=1 default vs 0): parity suites, then
# C2/C3/C4 bench lines with per-round times
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hardening.py tests/test_gpu_fuzz.py tests/test_gpu_hash2.py -m gpu -x -q > gpurun_out/tests_stamp.log 2>&1
for ST in 1 0 1 0; do
  SOLID_STAMP=$ST timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu --no-activator --no-evict --no-policy-eval --no-c5 --e2e-steps 0 > gpurun_out/ab_$ST.json 2> gpurun_out/ab_$ST.err
  python - <<PY >> gpurun_out/ab_stamp.txt
import json
d=json.loads(open("gpurun_out/ab_$ST.json").read().strip().splitlines()[-1])
oc=d["other_configs"]
print("stamp=$ST", round(d["ms_per_step"],4), d["phases_ms_median"]["resolve"], d["resolver_round_us"][:6], "c3", round(oc["c3"]["ms_per_batch"],3), oc["c3"]["resolver_round_us"], "c4", round(oc["c4"]["ms_per_batch"],3), oc["c4"]["resolver_round_us"])
PY
done
