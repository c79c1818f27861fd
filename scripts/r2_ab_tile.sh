#!/bin/bash
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hardening.py tests/test_gpu_fuzz.py tests/test_gpu_hash2.py -m gpu -x -q > gpurun_out/tests16.log 2>&1
for TW in auto 32 auto 32; do
  SOLID_RESOLVE_TILE=$TW timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu --no-activator --no-evict --no-policy-eval --no-c5 --e2e-steps 0 > gpurun_out/ab_$TW.json 2> gpurun_out/ab_$TW.err
  python - <<PY >> gpurun_out/ab.txt
import json
d=json.loads(open("gpurun_out/ab_$TW.json").read().strip().splitlines()[-1])
oc=d["other_configs"]
print("$TW", round(d["ms_per_step"],4), d["phases_ms_median"]["resolve"], d["resolver_round_us"][:5], "c3", round(oc["c3"]["ms_per_batch"],3), oc["c3"]["phases_ms"]["resolve"], "c4", round(oc["c4"]["ms_per_batch"],3), oc["c4"]["phases_ms"]["resolve"])
PY
done
