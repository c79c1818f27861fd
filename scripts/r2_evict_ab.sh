#!/bin/bash
# evict / pin / pool suites with the in-tree library, then the bench's LRU leg alternating two
# library builds (lib/libsolid_base.so vs lib/libsolid.so)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_evict.py tests/test_gpu_pins.py tests/test_gpu_pool.py -m gpu -x -q > gpurun_out/tests_evict.log 2>&1
rm -f gpurun_out/evict_ab.txt
for L in base new base new; do
  if [ $L = base ]; then export SOLID_LIB=paper_2603_10726_b200/lib/libsolid_base.so; else unset SOLID_LIB; fi
  timeout 900 python bench.py --no-configs --no-c5 --no-activator --no-policy-eval --no-cpu --e2e-steps 0 --steps 10 --warmup 2 > gpurun_out/evict_$L.json 2> gpurun_out/evict_$L.err
  python - <<PY >> gpurun_out/evict_ab.txt
import json
d=json.loads(open("gpurun_out/evict_$L.json").read().strip().splitlines()[-1]); e=d["lru_eviction"]
print("$L", round(e["ms_per_batch"],4), e["phases_ms"], e.get("evict_iterations"), e.get("resolver_rounds"), "c2", round(d["ms_per_step"],4))
PY
done
