# k_resolve occupancy sweep: build variants with __launch_bounds__(256, C) and time the C2 step.
set -e
for c in 4 5 6 8; do
  sed "s/__global__ void __launch_bounds__(256, 4) k_resolve(KParams kp, uint32_t t_max) {/__global__ void __launch_bounds__(256, $c) k_resolve(KParams kp, uint32_t t_max) {/" \
    paper_2603_10726_b200/csrc/solid.cu > paper_2603_10726_b200/csrc/solid_occ.cu
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -diag-suppress 186 -I include -o paper_2603_10726_b200/lib/libsolid_occ$c.so \
    paper_2603_10726_b200/csrc/solid_occ.cu paper_2603_10726_b200/csrc/solid_activator.cu
done
rm -f paper_2603_10726_b200/csrc/solid_occ.cu
for c in 4 5 6 8; do
  SOLID_LIB=paper_2603_10726_b200/lib/libsolid_occ$c.so timeout 300 python bench.py --steps 10 --warmup 3 \
    --no-cpu --no-evict --no-policy-eval --no-activator --e2e-steps 0 > gpurun_out/occ$c.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/occ$c.json').read().strip().splitlines()[-1]); print($c, round(d['ms_per_step'],4), round(d['phases_ms_median']['resolve'],4), d['resolver_round_us'][:4])"
done
