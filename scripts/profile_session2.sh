# ncu evidence for the session-2 kernels (one GPU): evict-mode launch list + full captures of
# its top kernels, and the two-component hash kernel.  Outputs under gpurun_out/.
set -x
OUT=${OUT:-gpurun_out}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SOLID_PROFILE_EVICT=1 timeout 900 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $OUT/launches_evict.csv python scripts/bench_parts.py evict --no-cpu --steps 1 --warmup 1 > $OUT/launches_evict.log 2>&1
for K in k_window k_resolve_evict; do
  SOLID_PROFILE_EVICT=1 timeout 900 ncu --profile-from-start off --set full --clock-control none \
    --import-source on -k regex:$K -c 1 -o $OUT/prof_$K -f \
    python scripts/bench_parts.py evict --no-cpu --steps 1 --warmup 1 > $OUT/prof_$K.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_register -s 2 -c 1 \
  -o $OUT/prof_k_hash_register_nc2 -f python scripts/bench_parts.py hash2 --steps 1 --warmup 1 > $OUT/prof_hash2.log 2>&1
ls -la $OUT/*.ncu-rep
