#!/bin/bash
# 4-GPU box at HEAD: real NCCL / NVLink multi-GPU parity, then c3 strong scaling at N = 2 and 4 and the
# whole network at N = 4
set -u
O=gpurun_out/r02; mkdir -p $O; TAG=${1:-m}
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu -x > $O/pytest_multi4_$TAG.log 2>&1; echo "multi rc=$?"; tail -3 $O/pytest_multi4_$TAG.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29700 \
    bench.py --gpus $n --steps 20 --warmup 5 > $O/bench_c3_n${n}_$TAG.json 2> $O/bench_c3_n${n}_$TAG.err; echo "bench c3 n=$n rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 \
    bench.py --gpus 4 --network --steps 10 --warmup 3 > $O/bench_net_c3_n4_$TAG.json 2> $O/bench_net_c3_n4_$TAG.err; echo "bench net n=4 rc=$?"
python scripts/show_bench.py $O/bench_c3_n2_$TAG.json $O/bench_c3_n4_$TAG.json $O/bench_net_c3_n4_$TAG.json 2>&1 | grep -E "==|roofline"
