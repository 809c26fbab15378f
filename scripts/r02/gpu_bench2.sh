#!/bin/bash
O=gpurun_out/r02s; mkdir -p $O; TAG=${1:-x}
for cfg in c3 c2; do
timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-phases --layers 2 > $O/bench_${cfg}_$TAG.json 2> $O/bench_${cfg}_$TAG.err; echo "bench $cfg rc=$?"
python scripts/show_bench.py $O/bench_${cfg}_$TAG.json 2>&1 | grep -E "==|b_"
done
