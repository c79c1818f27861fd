# k_hash_register occupancy sweep: __launch_bounds__(256, C), C2 step timing.
set -e
for c in 3 4 5 6; do
  sed "s/__global__ void __launch_bounds__(256, 4) k_hash_register(KParams kp) {/__global__ void __launch_bounds__(256, $c) k_hash_register(KParams kp) {/" \
    paper_2603_10726_b200/csrc/solid.cu > paper_2603_10726_b200/csrc/solid_occ.cu
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -diag-suppress 186 -Xptxas -v -I include -o paper_2603_10726_b200/lib/libsolid_ka$c.so \
    paper_2603_10726_b200/csrc/solid_occ.cu paper_2603_10726_b200/csrc/solid_activator.cu 2>&1 | \
    grep -A2 "k_hash_registerILi2ELi1E" | grep "Used\|spill" | sed "s/^/C=$c /"
done
rm -f paper_2603_10726_b200/csrc/solid_occ.cu
for c in 3 4 5 6; do
  SOLID_LIB=paper_2603_10726_b200/lib/libsolid_ka$c.so timeout 300 python bench.py --steps 20 --warmup 3 \
    --no-cpu --no-evict --no-policy-eval --no-activator --no-configs --e2e-steps 0 > gpurun_out/ka$c.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ka$c.json').read().strip().splitlines()[-1]); print($c, round(d['ms_per_step'],4), round(d['phases_ms_median']['hash_kernel'],4))"
done
