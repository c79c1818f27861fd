# one iteration on the GPU box: build, parity tests, bench, ncu launch list
set -x
OUT=${OUT:-gpurun_out}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-sample 20000 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --profile --steps 1 --warmup 1 --no-cpu > $OUT/launches_bench.log 2>&1
python scripts/launches.py $OUT/launches.csv
