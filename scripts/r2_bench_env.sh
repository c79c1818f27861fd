#!/bin/bash
# default C2 bench line (no sub-measurements) under environment-variable variants, alternating
mkdir -p gpurun_out
rm -f gpurun_out/bench_env.txt
for rep in 1 2 3; do
  for V in "$@"; do
    env $V timeout 600 python bench.py --steps 20 --warmup 5 --no-activator --no-policy-eval --no-evict --no-c5 --no-configs --no-cpu --e2e-steps 0 > gpurun_out/bench_env.json 2> gpurun_out/bench_env.err
    python - <<PY >> gpurun_out/bench_env.txt
import json
d=json.loads(open("gpurun_out/bench_env.json").read().strip().splitlines()[-1])
print("$V", round(d["ms_per_step"],4), {k: round(v, 4) for k, v in d["phases_ms_median"].items()})
PY
  done
done
