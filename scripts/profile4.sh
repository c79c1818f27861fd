OUT=${OUT:-gpurun_out}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_resolve -s 1 -c 1 \
    -o $OUT/prof_resolve -f python bench.py --profile --steps 1 --warmup 1 --no-cpu > $OUT/prof_resolve.log 2>&1
ls -la $OUT/prof_resolve.ncu-rep
