#!/bin/bash
# quick GPU iteration: parity tests (single GPU) + bench (no cpu baseline)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "not multi" > gpurun_out/pytest_quick.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_quick.err
