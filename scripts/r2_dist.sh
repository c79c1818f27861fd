#!/bin/bash
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_dist_procs.py -m gpu -x -q > gpurun_out/tests_dist.log 2>&1
timeout 900 python -m pytest tests/test_gpu_c5.py -m gpu -x -q -k sharded > gpurun_out/tests_c5_sharded.log 2>&1
