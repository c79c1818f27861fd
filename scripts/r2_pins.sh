#!/bin/bash
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_pins.py tests/test_gpu_evict.py tests/test_gpu_pool.py -m gpu -x -q > gpurun_out/tests_pins.log 2>&1
