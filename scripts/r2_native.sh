#!/bin/bash
# solid_dist_admit: multi-process GPU tests, the existing sharded suites, and 2-rank bench lines
# (both ranks on this box's one GPU, gloo for torch.distributed, native vs python-driven p2p)
mkdir -p gpurun_out
python -m paper_2603_10726_b200.build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_dist_admit.py -m gpu -x -q > gpurun_out/tests_native.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_dist_procs.py -m gpu -x -q > gpurun_out/tests_dist.log 2>&1
for X in native p2p-dev; do
  SOLID_DIST_BACKEND=gloo SOLID_DIST_EXCHANGE=$X timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 2 --e2e-steps 0 > gpurun_out/bench2_$X.json 2> gpurun_out/bench2_$X.err
done
