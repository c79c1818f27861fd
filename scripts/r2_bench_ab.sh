#!/bin/bash
# bench lines (pipelined C2 + C3/C4 legs) for SOLID_STAMP=1 and 0, alternating
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hardening.py -m gpu -x -q > gpurun_out/tests_ab.log 2>&1
for ST in ${VARIANTS:-1 0 1 0}; do
  env $ST timeout 900 python bench.py --steps 20 --warmup 3 --no-activator --no-evict --no-policy-eval --no-c5 --e2e-steps 0 > gpurun_out/ab_${ST//[=,]/_}.json 2> gpurun_out/ab_${ST//[=,]/_}.err
  python - <<PY >> gpurun_out/ab_stamp.txt
import json
d=json.loads(open("gpurun_out/ab_${ST//[=,]/_}.json").read().strip().splitlines()[-1])
oc=d["other_configs"]
print("$ST", round(d["ms_per_step"],4), d["phases_ms_median"]["resolve"], d["resolver_round_us"][:6], d["parity"]["status"], "c3", round(oc["c3"]["ms_per_batch"],3), oc["c3"]["resolver_round_us"], "c4", round(oc["c4"]["ms_per_batch"],3), oc["c4"]["resolver_round_us"])
PY
done
