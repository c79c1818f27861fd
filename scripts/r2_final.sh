#!/bin/bash
# end-of-round evidence: smoke, the whole -m gpu suite, the default bench line, the ncu launch
# list of the C2 step and --set full captures of its four kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/tests_all.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/launches_run.log 2>&1
for K in k_hash_register k_resolve k_commit k_stats; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 1 -c 1 \
    -o gpurun_out/full_$K -f python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/full_$K.log 2>&1
done
ls -la gpurun_out/
