#!/bin/bash
# parity suites + resolver A/B (scripts/ab_resolve.py) of the variants given as arguments
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hardening.py tests/test_gpu_fuzz.py tests/test_gpu_hash2.py -m gpu -x -q > gpurun_out/tests_ab.log 2>&1
timeout 1200 python scripts/ab_resolve.py "$@" > gpurun_out/ab_resolve.txt 2>&1
