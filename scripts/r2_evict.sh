#!/bin/bash
# evict-mode suites + the bench's LRU leg (bucket sort vs radix-sort fallback)
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_evict.py tests/test_gpu_pins.py tests/test_gpu_pool.py -m gpu -x -q > gpurun_out/tests_evict.log 2>&1
for V in SOLID_EVICT_NONE=1 SOLID_EVICT_NONE=2; do
  env $V timeout 900 python bench.py --no-configs --no-c5 --no-activator --no-policy-eval --no-cpu --e2e-steps 0 --steps 10 --warmup 2 > gpurun_out/evict_$V.json 2> gpurun_out/evict_$V.err
  python - <<PY >> gpurun_out/evict_ab.txt
import json
d=json.loads(open("gpurun_out/evict_$V.json").read().strip().splitlines()[-1]); e=d["lru_eviction"]
print("$V", round(e["ms_per_batch"],4), e["phases_ms"], e["evict_iterations"], e["resolver_rounds"])
PY
done
