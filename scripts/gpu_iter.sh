#!/bin/bash
# quick iteration: parity (single GPU) + short bench with per-stage times
set -u
TAG=${1:-it}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python scripts/show_bench.py gpurun_out/bench_$TAG.json 2>&1 | head -12
