#!/bin/bash
# weak-scaling bench at N = 2 and 4 (layer path and whole network), 4-GPU multi tests
set -u
TAG=${1:-s4}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi_$TAG.log 2>&1; echo "multi pytest rc=$?"; tail -3 gpurun_out/pytest_multi_$TAG.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29633 \
    bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/bench_n${n}_$TAG.json 2> gpurun_out/bench_n${n}_$TAG.err; echo "bench n=$n rc=$?"
  python scripts/show_bench.py gpurun_out/bench_n${n}_$TAG.json 2>/dev/null | head -1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 \
  bench.py --gpus 4 --network --steps 10 --warmup 3 > gpurun_out/bench_net_n4_$TAG.json 2> gpurun_out/bench_net_n4_$TAG.err; echo "bench net n=4 rc=$?"
python scripts/show_bench.py gpurun_out/bench_net_n4_$TAG.json 2>/dev/null | head -1
