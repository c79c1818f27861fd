# build kernel variants (-D flags) as separate libraries and time them under the bench (ncu launch list)
# usage: VARIANTS="name1:-DFOO=1 name2:-DBAR=2" bash scripts/variants.sh
OUT=${OUT:-gpurun_out}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in $VARIANTS; do
  name=${v%%:*}; flags=${v#*:}; flags=${flags//,/ }
  lib=paper_2603_10726_b200/lib/libsolid_$name.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -diag-suppress 186 $flags -I include -o $lib paper_2603_10726_b200/csrc/solid.cu || continue
  SOLID_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 0 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', 'ms/step', round(d['ms_per_step'],4), 'phases', {k: round(v,4) for k,v in d['phases_ms_median'].items()})"
  SOLID_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$name.csv \
    python bench.py --profile --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
  echo "== $name"; python scripts/launches.py $OUT/launches_$name.csv | tail -8
done
