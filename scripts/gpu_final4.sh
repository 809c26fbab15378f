#!/bin/bash
# 4-GPU evidence: all gpu tests, smoke, bench N=1 (default), N=2, N=4, network N=1/4
set -u
TAG=${1:-f4}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_all_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_all_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_n1_$TAG.json 2> gpurun_out/bench_n1_$TAG.err; echo "bench n1 rc=$?"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29633 \
    bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/bench_n${n}_$TAG.json 2> gpurun_out/bench_n${n}_$TAG.err; echo "bench n=$n rc=$?"
done
timeout 600 python bench.py --network --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_net1_$TAG.json 2>/dev/null; echo "net n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 \
  bench.py --gpus 4 --network --steps 10 --warmup 3 > gpurun_out/bench_net4_$TAG.json 2>/dev/null; echo "net n4 rc=$?"
for f in n1 n2 n4 net1 net4; do python scripts/show_bench.py gpurun_out/bench_${f}_$TAG.json 2>/dev/null | head -1; done
