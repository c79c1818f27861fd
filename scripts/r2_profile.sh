#!/bin/bash
# round 2 profiles of the C2 bench step: launch list (per-kernel time, DRAM, L2 hit, instructions)
# and one `ncu --set full` capture of each of the four kernels of the step (second bench step)
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/launches_run.log 2>&1
for K in ${KERNELS:-k_hash_register k_resolve k_commit k_stats}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 1 -c 1 \
    -o gpurun_out/full_$K -f python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/full_$K.log 2>&1
done
ls -la gpurun_out/
