#!/bin/bash
# evict-mode variants chosen by environment variables: the evict / pin / pool suites under the
# first variant, then the bench's LRU leg alternating all variants
mkdir -p gpurun_out
env $1 timeout 1500 python -m pytest tests/test_gpu_evict.py tests/test_gpu_pins.py tests/test_gpu_pool.py -m gpu -x -q > gpurun_out/tests_evict_env.log 2>&1
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
