#!/bin/bash
# resolver A/B under environment-variable variants (scripts/ab_resolve.py), no parity suites
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 1200 python scripts/ab_resolve.py "$@" > gpurun_out/ab_env.txt 2>&1
