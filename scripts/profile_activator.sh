# fp64 peak micro-benchmark + full ncu capture of the Activator's window kernel (one GPU)
OUT=${OUT:-gpurun_out}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64 scripts/micro/fp64.cu && /tmp/fp64 | tee $OUT/fp64_peak.json
cat > /tmp/act_prof.py <<'PY'
import sys; sys.path.insert(0, ".")
import argparse, torch
import bench
a = argparse.Namespace(no_cpu=True)
print(bench.measure_activator(torch.device("cuda", 0), a)["ms_per_call"])
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_act_window -s 1 -c 1 \
  -o $OUT/prof_act_window -f python /tmp/act_prof.py > $OUT/prof_act_window.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $OUT/launches_act.csv python /tmp/act_prof.py > /dev/null 2>&1
python scripts/launches.py $OUT/launches_act.csv | tail -8
