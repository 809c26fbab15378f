#!/bin/bash
# multi-GPU: parity tests + weak-scaling bench at N = 2..$1
set -u
N=${1:-4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_multi${N}.log 2>&1; echo "multi pytest rc=$?"; tail -3 gpurun_out/pytest_multi${N}.log
for n in 2 4 8; do
  if [ $n -le $N ]; then
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29633 \
      bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo "bench n=$n rc=$?"
    tail -2 gpurun_out/bench_n$n.err
  fi
done
