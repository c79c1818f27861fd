# full ncu captures (source-level) of the two top kernels of the bench step; one GPU only
OUT=${OUT:-gpurun_out}
TAG=${TAG:-cur}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for K in ${KERNELS:-k_hash_chain k_register k_resolve}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
    -o $OUT/prof_${K}_$TAG -f python bench.py --profile --steps 1 --warmup 1 --no-cpu > $OUT/prof_${K}_$TAG.log 2>&1
done
ls -la $OUT/*_$TAG.ncu-rep
