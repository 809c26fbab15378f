#!/bin/bash
# quick loop: a parity subset, then c3 / c2 bench lines (no CPU baseline)
set -u
O=gpurun_out/r02; mkdir -p $O; TAG=${1:-q}
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py -x -q -m gpu -k "not full_size and not instantiations" > $O/pytest_$TAG.log 2>&1; echo "parity rc=$?"; tail -2 $O/pytest_$TAG.log
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-phases --layers 2 > $O/bench_c3_$TAG.json 2> $O/bench_c3_$TAG.err; echo "bench c3 rc=$?"
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-phases > $O/bench_c2_$TAG.json 2> $O/bench_c2_$TAG.err; echo "bench c2 rc=$?"
python scripts/show_bench.py $O/bench_c3_$TAG.json $O/bench_c2_$TAG.json 2>&1 | head -40
