#!/bin/bash
# round 2: new hardening tests, core parity, then a default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_hardening.py tests/test_gpu_hash2.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/tests_a.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/tests_all.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
