#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g1.json 2> gpurun_out/bench_g1.err; echo "graph n1 rc=$?"; tail -2 gpurun_out/bench_g1.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/bench_e1.json 2> /dev/null; echo "eager n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 \
  bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err; echo "graph n2 rc=$?"; tail -2 gpurun_out/bench_g2.err
for f in g1 e1 g2; do python scripts/show_bench.py gpurun_out/bench_$f.json 2>/dev/null | head -1; done
