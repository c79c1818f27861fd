#!/bin/bash
# commit-kernel A/B: parity suites with the in-tree library, C2/C3/C4 timings of two builds,
# and the C5 batch (scripts/c5_profile.py) with each build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hardening.py tests/test_gpu_pool.py -m gpu -x -q > gpurun_out/tests_commit.log 2>&1
bash scripts/r2_ab_libs.sh base commit
for L in base commit base commit; do
  echo "$L $(SOLID_LIB=paper_2603_10726_b200/lib/libsolid_$L.so python scripts/c5_profile.py 2>&1 | tail -1)" >> gpurun_out/ab_libs.txt
done
