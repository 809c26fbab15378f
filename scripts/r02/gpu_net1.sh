#!/bin/bash
# whole network at N = 1 (c3) and the c4 layer line at N = 1
set -u
O=gpurun_out/r02; mkdir -p $O; TAG=${1:-n1}
timeout 600 python bench.py --network --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_net_c3_n1_$TAG.json 2> $O/bench_net_c3_n1_$TAG.err; echo "net rc=$?"
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4_n1_$TAG.json 2> $O/bench_c4_n1_$TAG.err; echo "c4 rc=$?"
python scripts/show_bench.py $O/bench_net_c3_n1_$TAG.json $O/bench_c4_n1_$TAG.json 2>&1 | grep -E "==|roofline"
