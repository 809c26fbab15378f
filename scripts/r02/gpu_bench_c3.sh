#!/bin/bash
O=gpurun_out/r02s; mkdir -p $O; TAG=${1:-x}
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-phases --layers 2 > $O/bench_c3_$TAG.json 2> $O/bench_c3_$TAG.err; echo "bench c3 rc=$?"
python scripts/show_bench.py $O/bench_c3_$TAG.json 2>&1 | grep -E "==|pass_c|mix|pass_a|b_"
