#!/bin/bash
# 4-GPU box: real NCCL / NVLink multi-GPU parity, then c3 strong scaling at N = 2 and 4 (+ c4 weak at N = 4),
# NVLink byte counters around one bench run
set -u
O=gpurun_out/r02; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu -x > $O/pytest_multi4.log 2>&1; echo "multi rc=$?"; tail -3 $O/pytest_multi4.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29700 \
    bench.py --gpus $n --steps 20 --warmup 5 > $O/bench_c3_n$n.json 2> $O/bench_c3_n$n.err; echo "bench c3 n=$n rc=$?"
done
nvidia-smi nvlink -gt d > $O/nvlink_before.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 \
    bench.py --gpus 2 --steps 20 --warmup 5 --no-phases > $O/bench_c3_n2_nvl.json 2> $O/bench_c3_n2_nvl.err; echo "bench nvl rc=$?"
nvidia-smi nvlink -gt d > $O/nvlink_after.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29702 \
    bench.py --gpus 4 --config c4 --steps 10 --warmup 3 > $O/bench_c4_n4.json 2> $O/bench_c4_n4.err; echo "bench c4 n=4 rc=$?"
python scripts/show_bench.py $O/bench_c3_n2.json $O/bench_c3_n4.json $O/bench_c4_n4.json 2>&1 | grep -E "==|roofline|exchange|b_y_inv|pass_c"
