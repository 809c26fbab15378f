#!/bin/bash
# parity + bench (default path) + the same bench with the pass_c2 forward (FNO_PASS_C3=0)
set -u
TAG=${1:-ab}
bash scripts/gpu_iter.sh $TAG
FNO_PASS_C3=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c2.json 2>/dev/null
python scripts/show_bench.py gpurun_out/bench_${TAG}_c2.json | head -5
