#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "decomposed_matches" > gpurun_out/pytest_yinv.log 2>&1; echo "multi rc=$?"; tail -2 gpurun_out/pytest_yinv.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_y1.json 2>/dev/null; echo "n1 rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 \
  bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_y2.json 2> /dev/null; echo "n2 rc=$?"
for f in y1 y2; do python scripts/show_bench.py gpurun_out/bench_$f.json 2>/dev/null | grep -E "value|b_y_inv|pass_a"; done
