#!/bin/bash
# 4-GPU box, final build: multi-GPU parity suite, c3 strong scaling N = 2 / 4, network step at c3 N = 1 / 4
set -u
O=gpurun_out/r02m4; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_multi4.log 2>&1; echo "multi rc=$?"; tail -2 $O/pytest_multi4.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n \
    bench.py --gpus $n --steps 20 --warmup 5 > $O/bench_c3_n$n.json 2> $O/bench_c3_n$n.err; echo "bench c3 n=$n rc=$?"
done
timeout 600 python bench.py --network --steps 10 --warmup 3 --no-phases > $O/bench_net_c3_n1.json 2> $O/bench_net_c3_n1.err; echo "net n=1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29710 \
    bench.py --gpus 4 --network --steps 10 --warmup 3 --no-phases > $O/bench_net_c3_n4.json 2> $O/bench_net_c3_n4.err; echo "net n=4 rc=$?"
python scripts/show_bench.py $O/bench_c3_n2.json $O/bench_c3_n4.json $O/bench_net_c3_n1.json $O/bench_net_c3_n4.json 2>&1 | grep -E "==|step roofline"
