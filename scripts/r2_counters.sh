#!/bin/bash
# per-round resolver counters (profiling build) on C2 and C4
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build --counters > gpurun_out/build_c.log 2>&1
for C in c2 c4; do for V in "SOLID_STAMP=1" "SOLID_STAMP=0"; do
  echo "== $C $V" >> gpurun_out/counters.txt
  env $V SOLID_LIB=paper_2603_10726_b200/lib/libsolid_counters.so timeout 600 python scripts/counters.py $C >> gpurun_out/counters.txt 2>&1
done; done
