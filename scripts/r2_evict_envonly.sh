#!/bin/bash
# the bench's LRU leg alternating environment-variable variants (no test suites)
mkdir -p gpurun_out
rm -f gpurun_out/evict_env_ab.txt
for rep in 1 2; do
  for V in "$@"; do
    env $V timeout 900 python bench.py --no-configs --no-c5 --no-activator --no-policy-eval --no-cpu --e2e-steps 0 --steps 10 --warmup 2 > gpurun_out/evict_env.json 2> gpurun_out/evict_env.err
    python - <<PY >> gpurun_out/evict_env_ab.txt
import json
d=json.loads(open("gpurun_out/evict_env.json").read().strip().splitlines()[-1]); e=d["lru_eviction"]
print("$V", round(e["ms_per_batch"],4), {k: round(v, 4) for k, v in e["phases_ms"].items()}, e.get("evict_iterations"), e.get("resolver_rounds"))
PY
  done
done
