#!/bin/bash
# A/B of two library builds (lib/libsolid_base.so vs lib/libsolid.so) on C2/C3/C4 + parity suites
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hardening.py tests/test_gpu_fuzz.py tests/test_gpu_hash2.py -m gpu -x -q > gpurun_out/tests_ab.log 2>&1
rm -f gpurun_out/ab_lib.txt
for L in base new base new; do
  if [ $L = base ]; then export SOLID_LIB=paper_2603_10726_b200/lib/libsolid_base.so; else unset SOLID_LIB; fi
  timeout 900 python scripts/ab_resolve.py "lib=$L" --reps 5 >> gpurun_out/ab_lib.txt 2>&1
done
