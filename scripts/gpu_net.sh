#!/bin/bash
# network: multi-GPU parity (2 GPUs) + whole-network training-step bench (N=1 and N=2)
set -u
TAG=${1:-net}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k network -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --network --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
python scripts/show_bench.py gpurun_out/bench_$TAG.json | head -4
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 \
  bench.py --gpus 2 --network --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_n2.json 2> gpurun_out/bench_${TAG}_n2.err; echo "bench n2 rc=$?"
python scripts/show_bench.py gpurun_out/bench_${TAG}_n2.json | head -2
