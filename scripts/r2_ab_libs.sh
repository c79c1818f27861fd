#!/bin/bash
# A/B of several library builds: lib/libsolid_<name>.so for each name given (C2/C3/C4 timings)
mkdir -p gpurun_out
rm -f gpurun_out/ab_libs.txt
for rep in 1 2; do
  for L in "$@"; do
    SOLID_LIB=paper_2603_10726_b200/lib/libsolid_$L.so timeout 900 python scripts/ab_resolve.py "lib=$L" --reps 5 >> gpurun_out/ab_libs.txt 2>&1
  done
done
