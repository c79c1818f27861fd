#!/bin/bash
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi --query-gpu=name,memory.total --format=csv) > gpurun_out/box.txt 2>&1
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hardening.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/tests_a.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_c5.py -m gpu -q -s > gpurun_out/tests_c5.log 2>&1
MEM=$(free -g | awk '/Mem:/{print $7}')
if [ "$MEM" -gt 70 ]; then SOLID_C5_ORACLE=1 timeout 1800 python -m pytest tests/test_gpu_c5.py -m gpu -q -k oracle_parity > gpurun_out/tests_c5_oracle.log 2>&1; fi
timeout 1500 python bench.py --steps 20 --warmup 5 --no-policy-eval > gpurun_out/bench.json 2> gpurun_out/bench.err
