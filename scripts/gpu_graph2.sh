#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 \
  bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err; echo "graph n2 rc=$?"; tail -3 gpurun_out/bench_g2.err
python scripts/show_bench.py gpurun_out/bench_g2.json 2>/dev/null | head -1
