#!/bin/bash
# core GPU suites + one bench line (C2 + C3/C4 legs)
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hardening.py tests/test_gpu_fuzz.py tests/test_gpu_hash2.py tests/test_gpu_pool.py -m gpu -x -q > gpurun_out/tests_quick.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 --no-activator --no-evict --no-policy-eval --no-c5 --e2e-steps 0 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
