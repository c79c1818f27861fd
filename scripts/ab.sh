# A/B timing of two library builds on the C2 bench step (alternating, same box)
for r in 1 2 3; do
  for v in A B; do
    if [ $v = A ]; then export SOLID_LIB=paper_2603_10726_b200/lib/libsolid_A.so; else unset SOLID_LIB; fi
    timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu --no-evict --no-policy-eval --no-activator --no-configs --e2e-steps 0 > gpurun_out/ab_$v$r.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v$r.json').read().strip().splitlines()[-1]); print('$v', $r, round(d['ms_per_step'],4), round(d['phases_ms_median']['commit'],4))"
  done
done
