#!/bin/bash
# ncu --set full of the evict-mode resolver (CTA per request) and the window kernel, LRU bench leg
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
for K in k_resolve_evict_cta k_window k_touch; do
  SOLID_PROFILE_EVICT=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"^$K" -c 1 \
    -o gpurun_out/full_$K -f python bench.py --no-configs --no-c5 --no-activator --no-policy-eval --no-cpu --e2e-steps 0 --steps 3 --warmup 1 > gpurun_out/full_$K.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
