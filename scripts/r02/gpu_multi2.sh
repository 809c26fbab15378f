#!/bin/bash
# 2-GPU box: multi-GPU parity (peer + NCCL transports) and c3 at N = 2
set -u
O=gpurun_out/r02m; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -m gpu -x -k "decomposed_matches or network" > $O/pytest_multi2.log 2>&1; echo "multi rc=$?"; tail -3 $O/pytest_multi2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29700 \
    bench.py --gpus 2 --steps 20 --warmup 5 --no-phases > $O/bench_c3_n2.json 2> $O/bench_c3_n2.err; echo "bench c3 n=2 rc=$?"
python scripts/show_bench.py $O/bench_c3_n2.json 2>&1 | grep -E "==|exchange|b_y_inv|pass_c"
